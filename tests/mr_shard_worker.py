"""torchrun worker for the particle-sharded decomposition (ST_DECOMP_SHARDED, SURVEY
§8(f2), PAPER Fig. 1c): the Eulerian side stays partitioned (rank r feeds the field of
its z-slab and reads the sources of its z-slab), while every rank holds the whole
field (broadcast from the owners) and its own particles (drawn anywhere); the sources
are reduced onto their owners.  Rank 0 joins the slabs' sources of every step and
compares them and every particle with ONE oracle run holding all ranks' particles (the
physics of a particle does not depend on which rank holds it): sources 1e-5 relative
L2, positions / velocities 1e-5."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import oracle
    import synth
    from paper_2603_26691_b200 import DECOMP_SHARDED, Config, ScaleTrack, nccl_unique_id

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    K = int(os.environ.get("MR_K", "2"))
    steps = int(os.environ.get("MR_STEPS", "6"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)

    dims, h = (32, 24, int(os.environ.get("MR_DZ", "40"))), 1 / 16   # 16 * world: equal slabs (all-gather path)
    L = [d * h for d in dims]
    cfg = Config(dims=dims, cell_size=(h, h, h), chunk_cells=8, bc=(1, 1, 1), gravity=(0, 0, -9.81),
                 rebin_interval=K, capacity=100_000, device=local, rank=rank, nranks=world,
                 decomposition=DECOMP_SHARDED)
    st = ScaleTrack(cfg, unique_id=uid[0])
    lay = st.layout
    ncz = dims[2] // 8
    assert (lay.z0, lay.z1) == (rank * ncz // world * 8, (rank + 1) * ncz // world * 8) and lay.halo_cells == 0
    parts = [synth.particles_np(15_000 + 2000 * r, (0, 0, 0), tuple(L), (5e-6, 40e-6), seed=300 + r)
             for r in range(world)]
    wl_f = synth.Workload("shard", dims, (0, 0, 0), (h, h, h), (1, 1, 1), 8, 0, (0, 0), "uniform", 1.0,
                          (0, 0, -9.81), 1, 1, 2e-3, steps, "fourier", {"u_rms": 0.3, "modes": 64, "kmax": 6}, 9, 0)
    F = synth.make_field(wl_f)                               # whole field, every rank
    x, u, d, w = parts[rank]
    st.inject(x, u, d, w)
    st.set_fluid_field(np.ascontiguousarray(F[:, lay.z0:lay.z1]))   # this rank's Eulerian partition
    Ss = []
    rebalance = os.environ.get("MR_REBALANCE") == "1"
    moved = (0, 0)
    for s in range(steps):
        st.advance(2e-3, 1)
        S, T = st.get_sources()
        Ss.append(S)
        if rebalance and s == 1:      # f4: equalise the counts (15000 + 2000 r injected)
            moved = st.rebalance(0.0)
    p = st.get_particles()
    gathered = [None] * world
    dist.all_gather_object(gathered, {"p": p, "S": Ss, "z": (lay.z0, lay.z1), "moved": moved})
    ok = True
    if rank == 0:
        mesh = oracle.Mesh(dims=dims, cell_size=(h, h, h), chunk_cells=8, bc=(1, 1, 1))
        o = oracle.Sim(mesh, oracle.Physics(gravity=(0, 0, -9.81)), rebin_interval=K, precision="f32")
        for r in range(world):
            xr, ur, dr, wr = parts[r]
            o.inject(xr, ur, dr, wr, ids=(np.uint64(r) << np.uint64(40)) + np.arange(dr.size, dtype=np.uint64))
        o.set_fluid_field(F)
        worst_s = 0.0
        same_all = [gathered[r]["z"] for r in range(world)] == [
            (r * (dims[2] // 8) // world * 8, (r + 1) * (dims[2] // 8) // world * 8) for r in range(world)]
        for s in range(steps):
            o.advance(2e-3, 1)
            So, _ = o.get_sources()
            Sg = np.concatenate([gathered[r]["S"][s] for r in range(world)], axis=1).astype(np.float64)
            worst_s = max(worst_s, float(np.linalg.norm(Sg - So) / max(np.linalg.norm(So), 1e-300)))
        po = o.particles()
        oid = po["id"].astype(np.uint64)
        worst_x = worst_u = 0.0
        ids_ok = True
        for r in range(world):
            pg = gathered[r]["p"]
            gid = pg["id"].astype(np.uint64)
            if not rebalance:
                ids_ok &= bool(np.all((gid >> np.uint64(40)) == r)) and gid.size == parts[r][2].size
            idx = np.searchsorted(oid, gid, sorter=np.argsort(oid))
            oi = np.argsort(oid)[idx]
            ids_ok &= bool(np.array_equal(oid[oi], gid))
            dx = np.abs(pg["x"].astype(np.float64) - po["x"][:, oi])
            for a in range(3):
                dx[a] = np.minimum(dx[a], L[a] - dx[a])
            worst_x = max(worst_x, float(dx.max() / max(L)))
            worst_u = max(worst_u, float(np.abs(pg["u"].astype(np.float64) - po["u"][:, oi]).max()))
            ok &= bool(np.all(np.diff(mesh_bins := o.bin_key(pg["x"])) >= 0))
        counts = [int(gathered[r]["p"]["id"].size) for r in range(world)]
        all_ids = np.sort(np.concatenate([gathered[r]["p"]["id"] for r in range(world)]).astype(np.uint64))
        ids_ok &= bool(np.array_equal(all_ids, np.sort(oid)))
        if rebalance:
            tot = sum(counts)
            ids_ok &= counts == [tot // world + (1 if r < tot % world else 0) for r in range(world)]
            ids_ok &= sum(gathered[r]["moved"][0] for r in range(world)) == sum(
                gathered[r]["moved"][1] for r in range(world)) > 0
        report = dict(counts=counts, moved=[gathered[r]["moved"] for r in range(world)],
                      source_rel_l2=worst_s, eulerian_slabs_ok=same_all, ids_ok=ids_ok,
                      worst_x=worst_x, worst_u=worst_u)
        ok &= worst_s <= 1e-5 and same_all and ids_ok and worst_x <= 1e-5 and worst_u <= 1e-5
        print("MR_REPORT " + json.dumps(report), flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
