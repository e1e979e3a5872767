#!/usr/bin/env python
"""Per-call timings of the C5 loop (debug aid): st_last_timings and host wall time of
each set_fluid_field/advance/get_sources call at rebin interval K.
usage: python scripts/probe_calls.py <particles> <K> <calls>"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2603_26691_b200 import Config, ScaleTrack  # noqa: E402

n, K, calls = float(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
wl = synth.workload("C5", 1, int(n))
dev = torch.device("cuda", 0)
cfg = Config(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells, bc=wl.bc,
             rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity, drag_law=wl.drag_law,
             coupling=wl.coupling, rebin_interval=K, capacity=int(n))
st = ScaleTrack(cfg, stream=torch.cuda.current_stream(dev).cuda_stream)
lo, hi = synth.domain_box(wl, (0, wl.dims[2]))
x, u, d, w = synth.particles_torch(int(n), lo, hi, wl.d_range, wl.d_dist, wl.w, seed=8000, device=dev)
st.inject(x, u, d, w)
del x, u, d, w
fields = [synth.make_field(wl, t=s * wl.dt, z_range=(0, wl.dims[2]), device=dev).contiguous() for s in range(2)]
S = torch.empty((3, wl.dims[2], wl.dims[1], wl.dims[0]), dtype=torch.float32, device=dev)
for c in range(calls):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.set_fluid_field(fields[c % 2])
    st.advance(wl.dt, 1)
    st.get_sources(S)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    a, r = st.last_timings()
    s = st.stats()
    print(f"call {c + 1:3d}  wall {1e3 * (t1 - t0):8.2f} ms  advance {a:7.2f}  rebin {r:7.2f}  "
          f"rebins {s['rebins']} fused {s['fused_rebins']} general {s['general_rebins']} far {s['last_far']}")
