#!/usr/bin/env python
"""Small end-to-end case for compute-sanitizer (memcheck / racecheck / synccheck): every
step-kernel flavour of the library at a size the sanitizers finish in minutes.

  compute-sanitizer --tool racecheck python scripts/sanitize_case.py

Covers: the unbinned first step and the general radix rebin (after injection), k_ip
(in place, with and without the slot count), k_fs (fused scatter + advance), the
standalone scatter (a flush by observation), far tails + k_far_order (fast flow at
K = 4), several sub-steps per call, 4^3 chunks (the generic k_step path), the source
readout and the droplet step k_micro; then checks the run against the oracle so a
silent corruption cannot pass as "no sanitizer report"."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def run_case(name, dims, chunk, K, n, calls, nsub=1, scale=1.0, seed=3):
    import oracle
    import synth
    from paper_2603_26691_b200 import Config, ScaleTrack
    wl = synth.workload("C5", n_particles=n)
    wl.dims, wl.origin, wl.chunk_cells = dims, (1.0, 1.0, 1.0), chunk
    wl.field_args = {"u_rms": 0.3, "modes": 32, "kmax": 2}
    lo, hi = synth.domain_box(wl)
    x, u, d, w = synth.particles_np(n, lo, hi, wl.d_range, wl.d_dist, wl.w, seed)
    F = (synth.make_field(wl) * scale).astype(np.float32)
    cfg = Config(dims=dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=chunk, bc=wl.bc,
                 gravity=wl.gravity, coupling=1, rebin_interval=K, capacity=n)
    g = ScaleTrack(cfg)
    mesh = oracle.Mesh(dims=dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=chunk, bc=wl.bc)
    o = oracle.Sim(mesh, oracle.Physics(gravity=wl.gravity, coupling=1), rebin_interval=K, precision="f32")
    for s in (g, o):
        s.inject(x, u, d, w)
        s.set_fluid_field(F)
    for c in range(calls):
        g.advance(wl.dt / nsub, nsub)
        o.advance(wl.dt / nsub, nsub)
        if c == calls // 2:
            g.get_particles()          # a flush by observation (standalone scatter)
    Sg, _ = g.get_sources()
    So, _ = o.get_sources()
    pg, po = g.get_particles(), o.particles()
    ig, io = np.argsort(pg["id"]), np.argsort(po["id"])
    dx = float(np.max(np.abs(pg["x"][:, ig].astype(np.float64) - po["x"][:, io])))
    st = g.stats()
    err = float(np.linalg.norm(Sg.astype(np.float64) - So) / max(np.linalg.norm(So), 1e-300))
    print(f"{name}: n={n} calls={calls} K={K} fused={st['fused_rebins']} general={st['general_rebins']} "
          f"far={st['last_far']} max|dx|={dx:.2e} S_relL2(free-running)={err:.2e}", flush=True)
    assert dx < 1e-4
    g.close()


def main():
    run_case("binned K=2 (k_ip, k_fs)", (24, 24, 24), 8, 2, 60_000, 7)
    run_case("K=4 fast (far tails)", (24, 24, 24), 8, 4, 40_000, 9, scale=8.0)
    run_case("sub-steps", (16, 16, 24), 8, 1, 30_000, 4, nsub=3)
    run_case("4^3 chunks (generic k_step)", (20, 16, 12), 4, 2, 30_000, 5)
    # droplet microphysics
    import torch

    import synth
    from oracle import microphysics as M
    from paper_2603_26691_b200 import MicroConfig, micro_advance
    dims, h = (16, 12, 8), 0.125
    F = synth.micro_field(dims, (0.0, 0.0, 0.0), (h,) * 3, seed=2)
    x, u, d, T, w = synth.droplets_np(5000, (0, 0, 0), (2.0, 1.5, 1.0), seed=3)
    dev = torch.device("cuda", 0)
    t = [torch.from_numpy(np.ascontiguousarray(v)).to(dev) for v in (x, u, d, T, w, F)]
    acc = torch.zeros((5, 8, 12, 16), dtype=torch.float64, device=dev)
    micro_advance(MicroConfig(dims=dims, cell_size=(h,) * 3, bc=(0, 0, 1)), *t, 5e-3, 3, acc)
    mesh = M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=(0, 0, 1))
    xo = M.micro_advance(mesh, M.MicroProps(), x, u, d, T, w, F, 5e-3, 3)[0]
    print(f"micro: max|dx|={np.max(np.abs(t[0].cpu().numpy() - xo)):.2e}", flush=True)
    print("SANITIZE_CASE_OK")


if __name__ == "__main__":
    main()
