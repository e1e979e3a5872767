"""Multi-rank host logic on CPU: world_size-2 (and 3) process groups over gloo.

* Every rank plans its slab with the library's own host code (st_plan_layout);
  the gathered slabs must tile the mesh in rank order and match the oracle's
  ownership rule (C-16), with the chunk_cells-plane halo the exchange assumes.
* The migration protocol the NCCL path implements (counts by all-gather, payload
  by point-to-point, kept ++ arrivals by ascending source rank, stable sort by
  bin key) is run across real processes with the oracle's per-particle step and
  must reproduce the single-process R-rank emulation exactly (order, ids, M).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _entry(rank, world, port, fn_name, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import tests.test_multirank_gloo as me
        res = getattr(me, fn_name)(rank, world)
        q.put((rank, "ok", res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, "err", traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def run_ranks(fn_name, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_entry, args=(r, world, port, fn_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    for _ in range(world):
        r, status, res = q.get(timeout=300)
        assert status == "ok", res
        out[r] = res
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


# ---------------------------------------------------------------- layout
MESHES = [((192, 192, 144), 8, 0), ((20, 13, 75), 8, 1), ((16, 16, 48), 4, 0)]


def layout_worker(rank, world):
    from paper_2603_26691_b200 import Config, plan_layout
    res = []
    for dims, cc, bcz in MESHES:
        cfg = Config(dims=dims, chunk_cells=cc, bc=(1, 1, bcz), rank=rank, nranks=world, capacity=10)
        lay = plan_layout(cfg)
        mine = (lay.z0, lay.z1, lay.kz0, lay.kz1, lay.halo_cells, lay.local_cells)
        allv = [None] * world
        dist.all_gather_object(allv, mine)
        res.append(allv)
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_slab_layout_tiles_the_mesh(world):
    import oracle
    out = run_ranks("layout_worker", world)
    for m, (dims, cc, bcz) in enumerate(MESHES):
        views = [out[r][m] for r in range(world)]
        assert all(v == views[0] for v in views)          # every rank agrees
        slabs = views[0]
        assert slabs[0][0] == 0 and slabs[-1][1] == dims[2]
        for r in range(world - 1):
            assert slabs[r][1] == slabs[r + 1][0]            # contiguous, rank order
            assert slabs[r][3] == slabs[r + 1][2]
        sim = oracle.Sim(oracle.Mesh(dims=dims, chunk_cells=cc), nranks=world)
        for r in range(world):
            z0, z1, kz0, kz1, H, cells = slabs[r]
            assert (kz0, kz1) == sim.plane_range(r)
            assert H == cc and cells == dims[0] * dims[1] * (z1 - z0)
            assert z1 - z0 >= H + 1                           # the field halo fits in one slab


# ---------------------------------------------------------------- migration protocol
def _mesh():
    import oracle
    return oracle.Mesh(dims=(16, 16, 32), cell_size=(1 / 16,) * 3, chunk_cells=4,
                       bc=(oracle.BC_PERIODIC, oracle.BC_PERIODIC, oracle.BC_REFLECT))


def _inputs(world):
    rng = np.random.default_rng(31)
    parts = []
    for r in range(world):
        n = 400 + 37 * r
        x = rng.random((3, n)) * np.array([[1.0], [1.0], [2.0]])
        parts.append((x.astype(np.float32), np.zeros((3, n), np.float32), np.full(n, 30e-6, np.float32)))
    F = (rng.normal(size=(3, 32, 16, 16)) * 0.4).astype(np.float32)
    return parts, F


def migrate_worker(rank, world):
    """One rank of the distributed protocol (mirrors st_comm.cu comm_migrate)."""
    import oracle
    mesh = _mesh()
    parts, F = _inputs(world)
    sim = oracle.Sim(mesh, oracle.Physics(coupling=oracle.ONE_WAY), precision="f32", rebin_interval=10 ** 9)
    x, u, d = parts[rank]
    sim.inject(x, u, d, rank=0, ids=(np.uint64(rank) << np.uint64(40)) + np.arange(x.shape[1], dtype=np.uint64))
    sim.set_fluid_field(F)
    ncz = mesh.nchunk[2]
    bases = [(q * ncz) // world for q in range(world + 1)]
    history = []
    for step in range(4):
        sim.advance(0.02, 1)                              # per-particle physics (rank-local)
        s = sim.stores[0]
        _, chunk = sim.locate(s.x)
        kz = chunk // (mesh.nchunk[0] * mesh.nchunk[1])
        owner = np.searchsorted(np.array(bases[1:]), kz, side="right")
        # 1) stable sort by chunk -> owner segments in rank order
        perm, _ = oracle.stable_order(chunk.astype(np.int64), mesh.n_chunks)
        own_sorted = owner[perm]
        cnt = np.array([(own_sorted == q).sum() for q in range(world)], np.int64)
        # 2) counts by all-gather (ncclAllGather)
        M = [torch.zeros(world, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(M, torch.from_numpy(cnt))
        M = torch.stack(M).numpy()
        # 3) payload by point-to-point (ncclSend/ncclRecv in a group)
        reqs, recv = [], {}
        for q in range(world):
            if q == rank or cnt[q] == 0:
                continue
            idx = perm[own_sorted == q]
            buf = np.concatenate([s.x[:, idx].ravel(), s.u[:, idx].ravel(), s.d[idx], s.w[idx]]).astype(np.float32)
            reqs.append(dist.isend(torch.from_numpy(buf), q))
            reqs.append(dist.isend(torch.from_numpy(s.id[idx].astype(np.int64)), q))
        for src in range(world):
            m = int(M[src, rank])
            if src == rank or m == 0:
                continue
            fb = torch.empty(8 * m, dtype=torch.float32)
            ib = torch.empty(m, dtype=torch.int64)
            dist.recv(fb, src)
            dist.recv(ib, src)
            recv[src] = (fb.numpy(), ib.numpy().astype(np.uint64))
        for r_ in reqs:
            r_.wait()
        # 4) kept ++ arrivals (ascending source rank), then stable sort by bin key
        kept = perm[own_sorted == rank]
        xs, us, ds, ws, ids = [s.x[:, kept]], [s.u[:, kept]], [s.d[kept]], [s.w[kept]], [s.id[kept]]
        for src in sorted(recv):
            fb, ib = recv[src]
            m = ib.size
            xs.append(fb[:3 * m].reshape(3, m)); us.append(fb[3 * m:6 * m].reshape(3, m))
            ds.append(fb[6 * m:7 * m]); ws.append(fb[7 * m:8 * m]); ids.append(ib)
        X = np.concatenate(xs, 1)
        order, _ = oracle.stable_order(sim.bin_key(X), mesh.n_bins)
        st = oracle._Store(np.ascontiguousarray(X[:, order]), np.ascontiguousarray(np.concatenate(us, 1)[:, order]),
                           np.concatenate(ds)[order], np.concatenate(ws)[order], np.concatenate(ids)[order])
        sim.stores[0] = st
        history.append((M[rank].tolist(), st.id.tolist(), st.x.tolist()))
    return history


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_migration_matches_emulation(world):
    import oracle
    out = run_ranks("migrate_worker", world)
    mesh = _mesh()
    parts, F = _inputs(world)
    emu = oracle.Sim(mesh, oracle.Physics(coupling=oracle.ONE_WAY), precision="f32", rebin_interval=1,
                     nranks=world)
    for r in range(world):
        x, u, d = parts[r]
        emu.inject(x, u, d, rank=r)
    emu.set_fluid_field(F)
    for step in range(4):
        emu.advance(0.02, 1)
        for r in range(world):
            M_row, ids, xs = out[r][step]
            assert M_row == emu.M[r].tolist()
            assert ids == emu.stores[r].id.tolist()
            assert np.array_equal(np.array(xs, np.float32), emu.stores[r].x)
    assert emu.M.sum() > 0 and np.trace(emu.M) < emu.M.sum()   # migration happened
