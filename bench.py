#!/usr/bin/env python
"""bench.py — particle-updates/s of the two-way-coupled SCALE-TRACK particle step
(arXiv 2603.26691) on N B200s, through the C-ABI (include/scaletrack.h).

One "step" = one pass of the whole hot path over the resident particles:
  st_set_fluid_field (field ingest, a1) -> st_advance(dt, 1) (locate, interpolate,
  drag+gravity, walls, relocate, deposit, rebin at the stated interval K, a2-a8,
  migration/halo when N > 1) -> st_get_sources (readout, a9).
Default workload: C5 (BASELINE.json configs[4]) true weak scaling, 1e9 particles
per GPU on a 192x192x(72 N) reflecting chamber grid, two-way, dt = 5 ms.

  python bench.py --gpus N --steps K --warmup W [--impl reference] [--workload C3|C4|C5]
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "particle-updates/s (two-way coupled) at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "particle-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5", choices=["C3", "C4", "C5"])
    ap.add_argument("--cluster", type=float, default=0.0,
                    help="clustered load: particle density ~ exp(-z / (c Lz)) over the whole job (0 = uniform)")
    ap.add_argument("--partition", default="equal", choices=["equal", "weighted", "hilbert"],
                    help="slab boundaries: equal chunk planes, or count-balanced (st_plan_partition, SURVEY f4); "
                         "hilbert (with --decomp sharded): each rank holds the particles of a count-balanced "
                         "range of chunks along the Hilbert curve (st_plan_hilbert, P:185)")
    ap.add_argument("--decomp", default="slab", choices=["slab", "sharded"],
                    help="slab: z-slabs with migration (north star); sharded: every GPU holds the whole "
                         "domain, particles stay, sources all-reduced (PAPER Fig. 1c, SURVEY f2)")
    ap.add_argument("--particles", type=float, default=None, help="particles per GPU (default: the workload's)")
    ap.add_argument("--rebin-interval", type=int, default=4,
                    help="K: rebin (fused neighbour scatter) every K-th step; particles that moved more than one "
                         "cell in between go to their bin's far tail (C-15b, DESIGN.md section 9)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-micro", action="store_true", help="skip the droplet-microphysics side measurement (f3)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0, help="target oracle CPU time for cpu_baseline")
    return ap.parse_args()


# ---------------------------------------------------------------- helpers
def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle sampler running during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons, pw = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
                pw.append(float(f[3]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_median": statistics.median(pw) if pw else None}


def make_workload(name, G, particles):
    import synth
    if name != "C5" and G > 1:
        raise SystemExit("multi-GPU runs use the C5 weak-scaling workload")
    wl = synth.workload(name, nranks=G)
    n_per = int(particles) if particles else (wl.n_particles // G if name == "C5" else wl.n_particles)
    return wl, n_per


def algorithmic_bytes_per_update(two_way=True):
    """read + write x,u (48 B) + read d (4) + read w (4, two-way)."""
    return 48 + 4 + (4 if two_way else 0)


# ---------------------------------------------------------------- oracle (CPU) legs
def _oracle_sim(wl, n_sample, K, F=None):
    import oracle
    import synth
    mesh = oracle.Mesh(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells, bc=wl.bc)
    phys = oracle.Physics(rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity,
                          drag_law=wl.drag_law, coupling=wl.coupling)
    sim = oracle.Sim(mesh, phys, rebin_interval=K, precision="f32")
    lo, hi = synth.domain_box(wl)
    x, u, d, w = synth.particles_np(n_sample, lo, hi, wl.d_range, wl.d_dist, wl.w, wl.seed_particles)
    sim.inject(x, u, d, w)
    F = synth.make_field(wl) if F is None else F
    sim.set_fluid_field(F)
    return sim, F


def run_oracle_sample(wl, n_sample, steps, z_range=None, K=4, F=None, barrier=None):
    """Time the oracle (fp32, single-threaded, as it stands) on a bounded sample of the
    workload: same grid and field recipe, n_sample particles, `steps` calls."""
    sim, F = _oracle_sim(wl, n_sample, K, F)
    if barrier is not None:
        barrier.wait()
    t0 = time.perf_counter()
    for _ in range(steps):
        sim.set_fluid_field(F)
        sim.advance(wl.dt, 1)
        sim.get_sources()
    return time.perf_counter() - t0


_SHARD = {}


def _shard_init(F, barrier):
    _SHARD["F"], _SHARD["barrier"] = F, barrier


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def _oracle_shard(args):
    """One independent oracle process of the all-core figure: its own
    shard of particles (seed per shard) on the full grid and field, `steps` calls, timed
    from a barrier all shards pass together; returns seconds."""
    name, n, steps, K, shard = args
    import synth
    wl = synth.workload(name)
    wl.seed_particles = 1000 + shard
    return run_oracle_sample(wl, n, steps, K=K, F=_SHARD["F"], barrier=_SHARD["barrier"])


def cpu_baseline(wl, target_s, K):
    """The oracle as it stands on the host: 1 core (one process), then every core
    (os.cpu_count() independent processes on disjoint particle shards),
    each a bounded sample of the workload; pu/s = particles x steps / wall seconds."""
    import multiprocessing as mp

    import synth
    n = 200_000
    F = synth.make_field(wl)
    t1 = run_oracle_sample(wl, n, 1, K=K, F=F)
    steps = max(1, int(target_s / max(t1, 1e-3)))
    steps = min(steps, 200)
    t = run_oracle_sample(wl, n, steps, K=K, F=F)
    cores = os.cpu_count() or 1
    all_core = None
    if cores > 1:
        n_sh = n
        steps_sh = max(1, min(200, int(0.5 * target_s / max(t1, 1e-3))))
        ctx = mp.get_context("spawn")
        barrier = ctx.Barrier(cores)
        with ctx.Pool(cores, initializer=_shard_init, initargs=(F, barrier)) as pool:
            ts = pool.map(_oracle_shard, [(wl.name, n_sh, steps_sh, K, k) for k in range(cores)])
        tw = max(ts)
        all_core = {"value": cores * n_sh * steps_sh / tw, "cores": cores,
                    "sample": f"{cores} independent oracle processes x {n_sh} particles x {steps_sh} steps on "
                              f"disjoint shards, timed from a common barrier, slowest {tw:.1f} s"}
    return {"value": n * steps / t, "unit": UNIT, "cores": 1, "kind": "oracle", "cpu_model": cpu_model(),
            "sample": f"{n} particles x {steps} steps of {wl.name} (full {wl.dims} grid, same field recipe), "
                      f"fp32 oracle, single-threaded, {t:.1f} s",
            "all_core": all_core}


def bench_config(wl, n_per, K, G, decomp):
    """The `config` of the JSON line, identical for both arms."""
    return {"workload": f"{wl.name}: {n_per:.3g} particles/GPU, grid {list(wl.dims)}, "
                        f"{'reflect' if wl.bc[0] else 'periodic'}, random-Fourier field "
                        f"u_rms={wl.field_args.get('u_rms')}, two-way, S-N drag + gravity, dt={wl.dt}",
            "particles_per_gpu": n_per, "grid": list(wl.dims), "chunk_cells": wl.chunk_cells,
            "rebin_interval": K, "substeps_per_step": 1,
            "l2": "inputs larger than L2 (40 B x N resident particle state)",
            "parallelism": f"z-slab x{G}" if decomp == "slab" else f"particle-sharded x{G}"}


def micro_leg(dev, n=200_000_000, calls=5, warmup=3):
    """Side measurement of NEXT f3 (st_micro_advance): n droplets in the
    binned (cell-sorted) order on the C5 grid, 10-30 um, dt = 1 ms (the explicit Eq. 7 /
    Eq. 12 updates stay contractive call after call), one sub-step per call, both
    arithmetic modes (fp64 default C-28, fp32 C-36), CUDA events on the launching stream
    after warm-up.  Not part of the headline step."""
    import torch

    import synth
    from paper_2603_26691_b200 import MicroConfig, micro_advance
    dims, h = (192, 192, 72), 1.0 / 32
    box = torch.tensor([6.0, 6.0, 2.25], device=dev)[:, None]
    F = torch.from_numpy(synth.micro_field(dims, (0.0, 0.0, 0.0), (h,) * 3, seed=4)).to(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(1)
    x = torch.minimum(torch.rand((3, n), generator=g, device=dev) * box, box * (1 - 1e-7))
    c = torch.floor(x / h).to(torch.int64)
    x = x[:, torch.argsort((c[2] * dims[1] + c[1]) * dims[0] + c[0])].contiguous()
    del c
    u = torch.zeros((3, n), device=dev)
    d = 10e-6 + 20e-6 * torch.rand(n, generator=g, device=dev)
    T = 281.0 + 4.0 * torch.rand(n, generator=g, device=dev)
    w = torch.full((n,), 100.0, device=dev)
    acc = torch.zeros((5, dims[2], dims[1], dims[0]), dtype=torch.float64, device=dev)
    s = torch.cuda.current_stream()
    alg = n * (52 + 40)
    out = {"metric": "droplet-updates/s (microphysics sub-step, NEXT f3)", "unit": "droplet-updates/s",
           "droplets": n, "calls": calls, "dt": 1e-3, "d_range_um": [10, 30], "order": "binned (cell-sorted)",
           "alg_bytes_per_call": alg}
    for mode in ("fp64", "fp32"):
        cfg = MicroConfig(dims=dims, cell_size=(h,) * 3, bc=(0, 0, 1), stream=s.cuda_stream, arithmetic=mode)
        for _ in range(warmup):
            micro_advance(cfg, x, u, d, T, w, F, 1e-3, 1, acc)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(calls):
            micro_advance(cfg, x, u, d, T, w, F, 1e-3, 1, acc)
        e1.record(s)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / calls
        out[mode] = {"value": n / (ms * 1e-3), "ms_per_call": ms, "achieved_GBs": alg / (ms * 1e-3) / 1e9}
    assert bool(torch.isfinite(d).all()) and bool(torch.isfinite(T).all())
    out["value"] = out["fp32"]["value"]
    out["ms_per_call"] = out["fp32"]["ms_per_call"]
    out["achieved_GBs"] = out["fp32"]["achieved_GBs"]
    out["bound"] = "fp64: alu (fp64 transcendentals); fp32: see DESIGN.md 9e"
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl, n_per = make_workload(args.workload, args.gpus, args.particles)
    n = 100_000
    t_w = run_oracle_sample(wl, n, max(args.warmup, 0), K=args.rebin_interval) if args.warmup else 0.0
    t = run_oracle_sample(wl, n, args.steps, K=args.rebin_interval)
    v = n * args.steps / t
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": bench_config(wl, n_per, args.rebin_interval, args.gpus, args.decomp),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle",
                             "sample": f"{n} particles x {args.steps} steps of {wl.name} (full {wl.dims} grid, same "
                                       f"field recipe), fp32 oracle, 1 thread, per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- GPU leg
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    from paper_2603_26691_b200 import Config, ScaleTrack, nccl_unique_id

    G = args.gpus
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != G:
        raise SystemExit(f"--gpus {G} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if G > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl, n_per = make_workload(args.workload, G, args.particles)
    K = args.rebin_interval
    uid = None
    if G > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    stream = torch.cuda.current_stream(dev)
    cap = n_per if G == 1 else int(n_per * 1.05) + 1_000_000
    cfg = Config(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells, bc=wl.bc,
                 rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity, drag_law=wl.drag_law,
                 coupling=wl.coupling, rebin_interval=K, capacity=cap, device=local, rank=rank, nranks=G,
                 decomposition=1 if args.decomp == "sharded" else 0)
    n_mine = n_per
    if args.cluster > 0:
        # clustered job: G * n_per particles with density ~ exp(-z / (c Lz)); rank r holds
        # those of its slab (equal planes, or count-balanced boundaries from the planes' counts)
        from paper_2603_26691_b200 import plan_partition
        Lz = wl.dims[2] * wl.cell_size[2]
        lam = args.cluster * Lz
        cc_h = wl.chunk_cells * wl.cell_size[2]
        ncz = (wl.dims[2] + wl.chunk_cells - 1) // wl.chunk_cells
        edges = [min(k * cc_h, Lz) for k in range(ncz + 1)]
        mass = [math.exp(-a / lam) - math.exp(-b / lam) for a, b in zip(edges[:-1], edges[1:])]
        tot_m = sum(mass)
        counts = [G * n_per * m / tot_m for m in mass]
        if args.partition == "weighted" and G > 1:
            cfg.slab_planes = plan_partition(cfg, counts)
        lay0 = __import__("paper_2603_26691_b200").plan_layout(cfg)
        if args.decomp == "slab":
            n_mine = int(round(sum(counts[lay0.kz0:lay0.kz1])))
            cfg.capacity = cap = int(n_mine * 1.1) + 1_000_000
    hil = None
    if args.decomp == "sharded" and args.partition == "hilbert":
        # f4: expected particles per chunk of the job's distribution (uniform, or the
        # clustered z-profile), chunk ranges along the Hilbert curve balanced by count
        from paper_2603_26691_b200 import plan_hilbert
        cc = wl.chunk_cells
        NC = [(d + cc - 1) // cc for d in wl.dims]
        L = [d * h for d, h in zip(wl.dims, wl.cell_size)]
        ze = [min(k * cc * wl.cell_size[2], L[2]) for k in range(NC[2] + 1)]
        if args.cluster > 0:
            lam_h = args.cluster * L[2]
            pm = np.array([math.exp(-a / lam_h) - math.exp(-b / lam_h) for a, b in zip(ze[:-1], ze[1:])])
        else:
            pm = np.diff(np.array(ze))
        cw = np.repeat(pm / pm.sum() / (NC[0] * NC[1]), NC[0] * NC[1])   # chunk ids z-major
        # ragged chunks at the x / y edges hold proportionally fewer cells
        fx = np.array([min(cc, wl.dims[0] - k * cc) / cc for k in range(NC[0])])
        fy = np.array([min(cc, wl.dims[1] - k * cc) / cc for k in range(NC[1])])
        cw = cw * np.tile(np.outer(fy, fx).ravel(), NC[2])
        cw = cw / cw.sum()
        owner = plan_hilbert(cfg, np.round(cw * G * n_per).astype(np.int64))
        mine = np.nonzero(owner == rank)[0]
        n_mine = int(round(cw[mine].sum() * G * n_per))
        cfg.capacity = cap = int(n_mine * 1.05) + 1_000_000
        hil = (mine, cw[mine], NC, L, ze)
    st = ScaleTrack(cfg, stream=stream.cuda_stream, unique_id=uid)
    lay = st.layout
    z_range = (lay.z0, lay.z1)      # this rank's Eulerian partition (field in, sources out)
    # particles: uniform in this rank's slab (slab decomposition) or anywhere in the domain
    # (particle-sharded: n_per per rank whatever the clustering, Fig. 1c), drawn on the
    # device in batches (seed 8 + rank); clustered: z redrawn from the exponential
    # restricted to that box (inverse CDF)
    lo, hi = synth.domain_box(wl, z_range if args.decomp == "slab" else None)
    batch = 100_000_000
    # st_inject is collective with nranks > 1 (slab decomposition): every rank makes the
    # same number of calls, those with fewer particles pass n = 0
    n_calls = (n_mine + batch - 1) // batch
    if G > 1 and args.decomp == "slab":
        t = torch.tensor([n_calls], dtype=torch.int64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        for _ in range(int(t.item()) - n_calls):
            st.inject(torch.empty((3, 0), device=dev), torch.empty((3, 0), device=dev), torch.empty(0, device=dev))
    for b0 in range(0, n_mine, batch):
        nb = min(batch, n_mine - b0)
        x, u, d, w = synth.particles_torch(nb, lo, hi, wl.d_range, wl.d_dist, wl.w,
                                           seed=wl.seed_particles * 1000 + rank * 100 + b0 // batch, device=dev)
        if hil is not None:
            # positions inside this rank's chunks: chunk by inverse CDF of its weights, then
            # uniform in x, y and (uniform or clustered) z within the chunk
            mine, wts, NC, L, ze = hil
            gen = torch.Generator(device=dev).manual_seed(91 + rank * 1000 + b0 // batch)
            cdf = torch.cumsum(torch.from_numpy(wts / wts.sum()).to(dev), 0)
            pick = torch.searchsorted(cdf, torch.rand(nb, device=dev, dtype=torch.float64, generator=gen)).clamp_(
                max=len(mine) - 1)
            ch = torch.from_numpy(mine).to(dev)[pick]
            kx, ky, kz = ch % NC[0], (ch // NC[0]) % NC[1], ch // (NC[0] * NC[1])
            ext = wl.chunk_cells * torch.tensor(wl.cell_size, dtype=torch.float64, device=dev)
            qs = torch.rand((3, nb), device=dev, dtype=torch.float64, generator=gen)
            xs = [torch.minimum((k + qs[a]) * ext[a], torch.tensor(L[a], dtype=torch.float64, device=dev))
                  for a, k in enumerate((kx, ky))]
            z0 = torch.tensor(ze, dtype=torch.float64, device=dev)[kz]
            z1 = torch.tensor(ze, dtype=torch.float64, device=dev)[kz + 1]
            if args.cluster > 0:
                ea, eb = torch.exp(-z0 / lam), torch.exp(-z1 / lam)
                zz = -lam * torch.log(ea - qs[2] * (ea - eb))
            else:
                zz = z0 + qs[2] * (z1 - z0)
            xs.append(zz)
            for a in range(3):
                hi32 = torch.tensor(L[a], dtype=torch.float32, device=dev)
                x[a] = torch.minimum(xs[a].to(torch.float32), torch.nextafter(hi32, torch.zeros_like(hi32)))
        elif args.cluster > 0:
            qz = torch.rand(nb, device=dev, dtype=torch.float64,
                            generator=torch.Generator(device=dev).manual_seed(77 + rank * 1000 + b0 // batch))
            ea, eb = math.exp(-lo[2] / lam), math.exp(-hi[2] / lam)
            z = -lam * torch.log(ea - qz * (ea - eb))
            z32 = z.to(torch.float32)   # clamp in fp32: the cast must not round onto the slab's top face
            lo32 = torch.tensor(lo[2], dtype=torch.float32, device=dev)
            hi32 = torch.tensor(hi[2], dtype=torch.float32, device=dev)
            x[2] = torch.minimum(torch.maximum(z32, lo32), torch.nextafter(hi32, lo32))
        st.inject(x, u, d, w)
        del x, u, d, w
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # two fields (t = 0, dt) of this rank's owned planes, alternated every step
    fields = [synth.make_field(wl, t=s * wl.dt, z_range=z_range, device=dev).contiguous() for s in range(2)]
    nx, ny, _ = wl.dims
    S = torch.empty((3, lay.z1 - lay.z0, ny, nx), dtype=torch.float32, device=dev)

    def step(s, Fsrc, Sdst):
        st.set_fluid_field(Fsrc[s % 2])
        st.advance(wl.dt, 1)
        st.get_sources(Sdst)

    # setup (untimed): 2K + 1 calls — the first rebin after injection (a full sort of the
    # randomly injected store) at call K, then one whole K-cycle including a fused
    # neighbour-slot rebin, so every kernel has run once — then W warm-up steps
    for s in range(2 * K + 1 + args.warmup):
        step(s, fields, S)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    l0 = st.stats()["kernel_launches"]
    c0 = st.stats()["calls"]          # first timed call in the library's trace ring
    adv, reb = [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for s in range(args.steps):
        step(s, fields, S)
        a, r = st.last_timings()
        adv.append(a)
        reb.append(r)
    e1.record(stream)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    launches = st.stats()["kernel_launches"] - l0
    timeline = None
    try:   # where the step time goes between the step kernels (library event ring, st_trace)
        tr = [st.trace(c0 + k) for k in range(min(args.steps, 60))]
        if all(t[2] >= 0 and t[3] >= 0 for t in tr):
            timeline = {"calls": len(tr),
                        "advance_call_ms": float(np.mean([t[3] - t[2] for t in tr])),
                        "gap_to_next_advance_ms": float(np.mean([tr[k + 1][2] - tr[k][3] for k in range(len(tr) - 1)]))
                        if len(tr) > 1 else 0.0,
                        "field_in_ms": float(np.mean([t[1] - t[0] for t in tr])),
                        "readout_ms": float(np.mean([t[5] - t[4] for t in tr]))}
    except Exception as ex:
        timeline = {"error": str(ex)[:200]}
    ms = e0.elapsed_time(e1)
    n_local = st.count()
    tot = torch.tensor([ms, float(n_local)], dtype=torch.float64, device=dev)
    if G > 1:
        t_max = tot[:1].clone()
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
        n_sum = tot[1:].clone()
        dist.all_reduce(n_sum, op=dist.ReduceOp.SUM)
        ms, n_total = float(t_max.item()), float(n_sum.item())
    else:
        n_total = float(n_local)
    value = n_total * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (per launch, CUDA events on the launching stream):
    # the step kernel (advance, with the rebin scatter fused in every K-th launch)
    adv_ms = statistics.mean(adv)
    reb_list = [r for r in reb if r > 0]
    reb_ms = statistics.mean(reb_list) if reb_list else 0.0
    st_stats = st.stats()
    movers = st_stats["last_movers"]          # chunk movers since the last rebin (one step's worth)
    f_move = movers / max(1, n_local)
    peak, peak_src = peaks()
    cells_win = nx * ny * (lay.z1 - lay.z0 + 2 * lay.halo_cells)
    kname = "step" + (" (advance + fused rebin scatter)" if K == 1 else f" (advance; rebin fused every {K})")
    # 56 B/update + 80 B per chunk mover (per rebin) + 24 B/cell (u_f in, S out)
    alg = algorithmic_bytes_per_update(wl.coupling == 1) * n_local + 80 * movers * (1.0 / K) + 24 * cells_win
    kms = adv_ms
    achieved = alg / (kms / 1e3) / 1e9
    # DRAM bytes per step launch from the committed ncu capture of THESE kernels at this
    # workload (profiles/ncu_traffic.json: per-launch dram__bytes_read + write of the fused
    # k_fs and the in-place k_ip at C5 1e9), mixed as the timed launches are: one fused
    # launch per K; null when no capture matches the workload / particle count
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        try:
            tj = json.load(open(tp))
            if tj.get("workload") == wl.name and abs(tj.get("particles", 0) - n_local) <= 0.01 * n_local:
                traffic = (tj["k_fs"] + (K - 1) * tj["k_ip"]) / K
                traffic_src = tj.get("source")
        except Exception:
            traffic = None

    # e2e: host (pinned) field in, host sources out, through the same C-ABI calls
    e2e = None
    if not args.no_e2e:
        Fh = [f.cpu().pin_memory() for f in fields]
        Sh = torch.empty(S.shape, dtype=torch.float32).pin_memory()
        for s in range(2):
            step(s, Fh, Sh)
        torch.cuda.synchronize()
        if G > 1:
            dist.barrier()
        k_e2e = max(3, min(args.steps, 10))
        h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        # the paper's asynchronous coupling (one-step skew): step s's
        # field goes in (H2D) and step s-1's sources come out (D2H) while step s runs;
        # every step's copies are inside the timed region
        torch.cuda.synchronize()
        k0 = st.stats()["calls"]      # index of the first e2e call in the library's trace ring
        esampler = ClockSampler(local)
        esampler.start()
        time.sleep(0.3)
        t_host0 = time.perf_counter()
        h0.record(stream)
        for s in range(k_e2e):
            st.set_fluid_field(Fh[s % 2])
            st.advance(wl.dt, 1)
            if s > 0:
                st.wait_sources(Sh)
            st.request_sources()
        st.wait_sources(Sh)
        h1.record(stream)
        torch.cuda.synchronize()
        t_host1 = time.perf_counter()
        # the device-resident loop again, right after (same thermal / power state): the
        # e2e gap that is not the copies shows up as a difference of the two step times
        d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        d0.record(stream)
        for s in range(k_e2e):
            step(s, fields, S)
        d1.record(stream)
        torch.cuda.synchronize()
        eclocks = esampler.stop()
        ems = max(h0.elapsed_time(h1), 1e3 * (t_host1 - t_host0))   # host-blocking copies: wall clock bounds it
        if G > 1:
            t = torch.tensor([ems], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": n_total * k_e2e / (ems / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(Fh[0].numel() * 4), "d2h_bytes_per_step": int(Sh.numel() * 4),
               "steps": k_e2e, "ms_per_step": ems / k_e2e, "clocks": eclocks,
               "device_ms_per_step_after": d0.elapsed_time(d1) / k_e2e}
        # the store's cost per step drifts as the particles evolve: compare
        # the e2e steps with the device-resident steps timed just before and just after them
        e2e["vs_device_around"] = (ems / k_e2e) / (0.5 * (ms / args.steps + e2e["device_ms_per_step_after"])) - 1.0
        try:   # where the e2e time goes: the library's CUDA-event ring (st_trace) of these calls
            tr = [st.trace(k0 + k) for k in range(k_e2e)]
            stp = [(t[2], t[3]) for t in tr]
            gaps = [stp[k + 1][0] - stp[k][1] for k in range(k_e2e - 1)]
            cin = [(t[0], t[1]) for t in tr[1:]]
            hid = sum(max(0.0, min(b, stp[k][1]) - max(a, stp[k][0])) for k, (a, b) in enumerate(cin))
            e2e["trace"] = {"steps_ms": float(np.mean([b - a for a, b in stp])),
                            "mean_gap_between_steps_ms": float(np.mean(gaps)) if gaps else 0.0,
                            "first_copy_to_last_step_end_ms": float(stp[-1][1] - tr[0][0]),
                            "copy_in_ms": float(np.mean([b - a for a, b in cin])) if cin else 0.0,
                            "copy_in_under_previous_step_frac": hid / max(1e-9, sum(b - a for a, b in cin))}
        except Exception as ex:      # diagnostics never sink the line
            e2e["trace"] = {"error": str(ex)[:200]}

    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(wl, args.cpu_seconds, K)

    micro = None
    if rank == 0 and G == 1 and not args.no_micro:
        try:
            micro = micro_leg(dev)
        except Exception as e:                      # a side measurement never sinks the bench line
            micro = {"error": f"{type(e).__name__}: {e}"[:300]}
        torch.cuda.empty_cache()

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": dict(bench_config(wl, n_per, K, G, args.decomp),
                           **({"cluster": args.cluster, "partition": args.partition,
                               "slab_planes": list(cfg.slab_planes) if cfg.slab_planes else None}
                              if args.cluster > 0 else {})),
            "roofline": {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "alg_bytes_per_launch": alg, "kernel_ms": kms},
            "timeline": timeline,
            "step_kernel_ms": adv_ms, "step_kernel_ms_series": [round(v, 3) for v in adv], "rebin_prep_ms": reb_ms, "rebins_in_timed_region": len(reb_list),
            "f_move_chunk": f_move, "fused_rebins": st_stats["fused_rebins"],
            "general_rebins": st_stats["general_rebins"], "far_last_rebin": st_stats["last_far"],
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clocks,
            "micro_f3": micro,
        }
        print(json.dumps(line), flush=True)
    st.close()
    if G > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
