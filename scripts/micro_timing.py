"""Time st_micro_advance at the C5 grid with N droplets resident in HBM:
CUDA events on the launching stream around `calls` calls of `nsteps` sub-steps each,
after warm-up.  Prints one JSON line (droplet-updates/s and the kernel's HBM roofline:
algorithmic bytes = 52 B per droplet per call + 5 x 8 B fp64 reductions per droplet
sub-step)."""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2603_26691_b200 import MicroConfig, micro_advance  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000_000)
ap.add_argument("--nsteps", type=int, default=1)
ap.add_argument("--calls", type=int, default=5)
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--arith", choices=("fp64", "fp32"), default="fp64", help="arithmetic mode (C-28 / C-36)")
ap.add_argument("--dt", type=float, default=1e-3)
ap.add_argument("--unsorted", action="store_true", help="random order instead of the binned (cell-sorted) store")
a = ap.parse_args()

dims, h = (192, 192, 72), 1.0 / 32
dev = torch.device("cuda:0")
F = torch.from_numpy(synth.micro_field(dims, (0.0, 0.0, 0.0), (h,) * 3, seed=4)).to(dev)
g = torch.Generator(device=dev)
g.manual_seed(1)
n = a.n
x = torch.rand((3, n), generator=g, device=dev) * torch.tensor([6.0, 6.0, 2.25], device=dev)[:, None]
x = torch.minimum(x, torch.tensor([6.0, 6.0, 2.25], device=dev)[:, None] * (1 - 1e-7))
if not a.unsorted:     # the binned store (C-15): droplets ordered by their cell
    c = torch.floor(x / h).to(torch.int64)
    key = (c[2] * 192 + c[1]) * 192 + c[0]
    x = x[:, torch.argsort(key)].contiguous()
    del c, key
u = torch.zeros((3, n), device=dev)
d = 10e-6 + 20e-6 * torch.rand(n, generator=g, device=dev)   # dt / tau_T <= 0.71 at dt = 1 ms
T = 281.0 + 4.0 * torch.rand(n, generator=g, device=dev)
w = torch.full((n,), 100.0, device=dev)
acc = torch.zeros((5, 72, 192, 192), dtype=torch.float64, device=dev)
cfg = MicroConfig(dims=dims, cell_size=(h,) * 3, bc=(0, 0, 1), arithmetic=a.arith)
s = torch.cuda.current_stream()
cfg.stream = s.cuda_stream
for _ in range(a.warmup):
    micro_advance(cfg, x, u, d, T, w, F, a.dt, a.nsteps, acc)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.calls + 1)]
ev[0].record(s)
for k in range(a.calls):
    micro_advance(cfg, x, u, d, T, w, F, a.dt, a.nsteps, acc)
    ev[k + 1].record(s)
torch.cuda.synchronize()
per = [ev[k].elapsed_time(ev[k + 1]) for k in range(a.calls)]
ms = ev[0].elapsed_time(ev[-1]) / a.calls
peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))
alg = n * (52 + 40 * a.nsteps)
print(json.dumps({"metric": "droplet-updates/s (microphysics step, f3)", "value": n * a.nsteps / (ms * 1e-3),
                  "n": n, "nsteps": a.nsteps, "arith": a.arith, "dt": a.dt, "binned": not a.unsorted, "ms_per_call": ms, "per_call_ms": per, "alg_bytes_per_call": alg,
                  "achieved_GBs": alg / (ms * 1e-3) / 1e9, "peaks": peaks}))
