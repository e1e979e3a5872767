#!/usr/bin/env python
"""Timeline of the asynchronous coupling buffer:
field copies in and source readouts out must run under the particle step, not between
steps.  Drives C3 (BASELINE.json configs[2]: 1e8 particles, 256^3 periodic, two-way,
a new field every step) through the C-ABI with pinned host buffers in the paper's
one-step-skew pattern and reads the st_trace event ring after the run: CUDA-event intervals on
the copy-in stream, the compute stream and the readout stream.

  python scripts/coupling_timeline.py [--workload C3] [--particles 1e8] [--steps 12] [--out f.json]

Prints one line per step (ms on the context's clock) and the fraction of copy-in /
readout time that lies inside some step's interval."""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def overlap(iv, steps):
    """Length of interval iv covered by the union of the step intervals."""
    a, b = iv
    tot = 0.0
    for s0, s1 in steps:
        lo, hi = max(a, s0), min(b, s1)
        if hi > lo:
            tot += hi - lo
    return tot


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="C3")
    ap.add_argument("--particles", type=float, default=None)
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--rebin-interval", type=int, default=4)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch

    import synth
    from paper_2603_26691_b200 import Config, ScaleTrack
    wl = synth.workload(a.workload)
    n = int(a.particles) if a.particles else wl.n_particles
    dev = torch.device("cuda", 0)
    cfg = Config(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells, bc=wl.bc,
                 rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity, drag_law=wl.drag_law,
                 coupling=wl.coupling, rebin_interval=a.rebin_interval, capacity=n)
    st = ScaleTrack(cfg)
    lo, hi = synth.domain_box(wl)
    for b0 in range(0, n, 100_000_000):
        nb = min(100_000_000, n - b0)
        x, u, d, w = synth.particles_torch(nb, lo, hi, wl.d_range, wl.d_dist, wl.w, seed=wl.seed_particles + b0,
                                           device=dev)
        st.inject(x, u, d, w)
        del x, u, d, w
    torch.cuda.synchronize()
    # a new field every step (C3: omega = |k| u_rms), two pinned host buffers alternating
    Fh = [synth.make_field(wl, t=s * wl.dt, device=dev).cpu().pin_memory() for s in range(2)]
    nx, ny, nz = wl.dims
    Sh = torch.empty((3, nz, ny, nx), dtype=torch.float32).pin_memory()
    rows = []
    for s in range(a.steps + 4):
        st.set_fluid_field(Fh[s % 2])
        st.advance(wl.dt, 1)
        if s > 0:
            st.wait_sources(Sh)
        st.request_sources()
    st.wait_sources(Sh)
    # read the event ring after the run (reading it inside the loop would block the host)
    for s in range(4, a.steps + 4):   # after the first sort and a full rebin cycle
        ci, sp, ro = st.trace(s), st.trace(s), st.trace(s - 1)
        rows.append({"step": s - 4, "copy_in": [ci[0], ci[1]], "step_ms": [sp[2], sp[3]],
                     "readout_prev": [ro[4], ro[5]]})
    t0 = rows[0]["copy_in"][0]
    steps = [r["step_ms"] for r in rows]
    cov_in = cov_out = len_in = len_out = 0.0
    print(f"{'step':>4} {'copy-in [ms]':>22} {'step [ms]':>22} {'readout of prev [ms]':>24}")
    for r in rows:
        ci, sp, ro = r["copy_in"], r["step_ms"], r["readout_prev"]
        print(f"{r['step']:4d} {ci[0]-t0:10.3f}-{ci[1]-t0:10.3f} {sp[0]-t0:10.3f}-{sp[1]-t0:10.3f} "
              f"{ro[0]-t0:11.3f}-{ro[1]-t0:11.3f}")
        len_in += ci[1] - ci[0]
        len_out += ro[1] - ro[0]
        cov_in += overlap(ci, steps)
        cov_out += overlap(ro, steps)
    gaps = [steps[k + 1][0] - steps[k][1] for k in range(len(steps) - 1)]
    summ = {"workload": f"{wl.name}: {n:.3g} particles, grid {list(wl.dims)}", "steps": len(rows),
            "mean_step_ms": float(np.mean([s1 - s0 for s0, s1 in steps])),
            "mean_gap_between_steps_ms": float(np.mean(gaps)),
            "copy_in_ms_per_step": len_in / len(rows), "copy_in_hidden_frac": cov_in / max(len_in, 1e-9),
            "readout_ms_per_step": len_out / len(rows), "readout_hidden_frac": cov_out / max(len_out, 1e-9),
            "h2d_bytes_per_step": int(Fh[0].numel() * 4), "d2h_bytes_per_step": int(Sh.numel() * 4)}
    print(json.dumps(summ))
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summ, "rows": rows}, f, indent=1)
    st.close()


if __name__ == "__main__":
    main()
