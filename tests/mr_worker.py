"""torchrun worker for the multi-GPU parity test (tests/test_gpu_multirank.py).

Every rank runs the CUDA path on its z-slab (NCCL migration + halo exchange);
rank 0 gathers particles, migration rows and sources and compares them with the
oracle's R-rank emulation on the same seeded inputs (C-16): per-rank order and
ids bit-exact given positions, migration counts exact, positions/velocities
1e-5, sources 1e-5 relative L2.
"""
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
    from paper_2603_26691_b200 import Config, ScaleTrack, nccl_unique_id, plan_partition

    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    K = int(os.environ.get("MR_K", "1"))
    bcz = int(os.environ.get("MR_BCZ", "1"))
    steps = int(os.environ.get("MR_STEPS", "6"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uid = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)

    dims, h = (32, 24, 32 * world), 1 / 16
    wl = synth.workload("C4", n_particles=0)
    cfg = Config(dims=dims, cell_size=(h, h, h), chunk_cells=8, bc=(1, 1, bcz), gravity=(0, 0, -9.81),
                 rebin_interval=K, capacity=200_000, device=local, rank=rank, nranks=world)
    split = None
    if os.environ.get("MR_SPLIT") == "weighted":   # count-balanced slabs for a bottom-heavy load (f4)
        split = plan_partition(cfg, np.exp(-np.arange(dims[2] // 8) / 2.0) * 1e5)
        cfg.slab_planes = split
    st = ScaleTrack(cfg, unique_id=uid[0])
    lay = st.layout
    # inputs: every rank injects particles drawn over its own slab, seed per rank
    L = [d * h for d in dims]
    L_x = L[0]
    slabs = [(r * (dims[2] // 8) // world * 8, (r + 1) * (dims[2] // 8) // world * 8) for r in range(world)]
    if split is not None:
        slabs = [(split[r] * 8, split[r + 1] * 8) for r in range(world)]
    parts = [synth.particles_np(20_000 + 1000 * r, (0, 0, slabs[r][0] * h), (L[0], L[1], slabs[r][1] * h),
                                (5e-6, 40e-6), seed=100 + r) for r in range(world)]
    assert (lay.z0, lay.z1) == slabs[rank]
    wl_f = synth.Workload("mr", dims, (0, 0, 0), (h, h, h), (1, 1, bcz), 8, 0, (0, 0), "uniform", 1.0,
                          (0, 0, -9.81), 1, 1, 2e-3, steps, "fourier", {"u_rms": 0.3, "modes": 64, "kmax": 6}, 9, 0)
    F = synth.make_field(wl_f)                               # global field [3][nz][ny][nx]
    if os.environ.get("MR_FIELD") == "xcross":
        # fast along x everywhere and 2 m/s upwards: far particles (C-15b) also cross the
        # slab boundaries, so far tails receive far particles from the neighbour ranks
        F = np.zeros_like(F)
        F[0] = 20.0
        F[2] = 2.0
        F = F.astype(np.float32)
    if os.environ.get("MR_FIELD") == "xshear":
        # fast along x (20 m/s: ~1.3 cells per 4 calls, far particles of C-15b) in the
        # planes from 2 above a slab boundary to 2 below the next, still along x in the
        # two planes on either side of a boundary, and 2 m/s upwards everywhere: the
        # boundary bins of plane z0 get local runs, arrivals from below (slow in x, so
        # near) and far particles from their own upper half (trilinear u_x rises to the
        # next plane) in the same rebin; no far particle changes rank (that would take
        # the general path)
        slab = dims[2] // world
        F = np.zeros_like(F)
        zl = np.arange(dims[2]) % slab
        F[0] = np.where((zl >= 2) & (zl <= slab - 3), 20.0, 0.0)[:, None, None]
        F[2] = 2.0
        F = F.astype(np.float32)
    x, u, d, w = parts[rank]
    st.inject(x, u, d, w)
    st.set_fluid_field(np.ascontiguousarray(F[:, lay.z0:lay.z1]))
    rows, Ss = [], []
    observe = os.environ.get("MR_OBSERVE", "each")   # "end": no per-call migration_counts (it
    for s in range(steps):                             # flushes a due rebin), so rebins run fused
        st.advance(2e-3, 1)
        if observe == "each" or s == steps - 1:
            rows.append(st.migration_counts().tolist())
        S, T = st.get_sources()
        Ss.append((S, T))
    p = st.get_particles()
    gathered = [None] * world
    stt = st.stats()
    dist.all_gather_object(gathered, {"p": p, "rows": rows, "S": [s for s, _ in Ss], "T": [t for _, t in Ss],
                                      "z": (lay.z0, lay.z1), "far": stt["last_far"],
                                      "general": stt["general_rebins"]})
    ok = True
    report = {}
    if rank == 0:
        mesh = oracle.Mesh(dims=dims, cell_size=(h, h, h), chunk_cells=8, bc=(1, 1, bcz))
        emu = oracle.Sim(mesh, oracle.Physics(gravity=(0, 0, -9.81)), rebin_interval=K, precision="f32", nranks=world,
                         plane_split=split)
        for r in range(world):
            xr, ur, dr, wr = parts[r]
            emu.inject(xr, ur, dr, wr, rank=r)
        emu.set_fluid_field(F)
        worst_s = 0.0
        for s in range(steps):
            emu.advance(2e-3, 1)
            So, To = emu.get_sources()
            Sg = np.concatenate([gathered[r]["S"][s] for r in range(world)], axis=1)
            err = float(np.linalg.norm(Sg.astype(np.float64) - So) / max(np.linalg.norm(So), 1e-300))
            worst_s = max(worst_s, err)
        report["source_rel_l2"] = worst_s
        ok &= worst_s <= 1e-5
        # migration rows of the last rebin
        last_rows = [gathered[r]["rows"][-1] for r in range(world)]
        if steps % K == 0:
            report["M_gpu"] = last_rows
            report["M_oracle"] = emu.M.tolist()
            ok &= last_rows == emu.M.tolist()
        worst_x = worst_u = 0.0
        order_ok = True
        for r in range(world):
            pg = gathered[r]["p"]
            po = emu.particles(r)
            same_set = sorted(pg["id"].tolist()) == sorted(po["id"].tolist())
            order_ok &= same_set and pg["id"].tolist() == po["id"].tolist()
            if same_set:
                og, oo = np.argsort(pg["id"]), np.argsort(po["id"])
                worst_x = max(worst_x, float(np.max(np.abs(pg["x"][:, og].astype(np.float64) - po["x"][:, oo])) / max(L)))
                U = max(1.0, float(np.max(np.abs(F))))       # velocities relative to the field's speed
                worst_u = max(worst_u, float(np.max(np.abs(pg["u"][:, og].astype(np.float64) - po["u"][:, oo]))) / U)
            # the last call ended with a rebin (flushed by the observation): the store is
            # sorted by the bin key of its own positions and owned (else it is sorted by
            # the positions of the previous rebin and advanced since: nothing to check)
            if steps % K == 0:
                bins = emu.bin_key(pg["x"])
                order_ok &= bool(np.all(np.diff(bins) >= 0))
                kz = pg["chunk"] // (mesh.nchunk[0] * mesh.nchunk[1])
                lo, hi = emu.plane_range(r)
                order_ok &= bool(np.all((kz >= lo) & (kz < hi)))
            if not (same_set and pg["id"].tolist() == po["id"].tolist()):
                k = next((i for i, (a, b) in enumerate(zip(pg["id"].tolist(), po["id"].tolist())) if a != b), -1)
                report.setdefault("first_mismatch", []).append((r, k))
        report.update(order_ok=bool(order_ok), worst_x=worst_x, worst_u=worst_u, oracle_last_far=int(emu.last_far),
                      gpu_last_far=[int(gathered[r]["far"]) for r in range(world)],
                      gpu_general=[int(gathered[r]["general"]) for r in range(world)])
        if os.environ.get("MR_FIELD") in ("xshear", "xcross"):
            ok &= emu.last_far > 0 and sum(report["gpu_last_far"]) == emu.last_far
            ok &= all(gg == 1 for gg in report["gpu_general"])   # every later rebin fused
        ok &= order_ok and worst_x <= 1e-5 and worst_u <= 1e-5
        print("MR_REPORT " + json.dumps(report), flush=True)
    st.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 3)


if __name__ == "__main__":
    main()
