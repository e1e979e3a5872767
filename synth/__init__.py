"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

Holds none of the method's arithmetic: it only draws particles and writes fluid
velocity fields (uniform, Taylor-Green, random-Fourier) at cell centres, in the
shapes of the paper's workloads (DESIGN.md §7 "input recipe").  Both the oracle
(`oracle/`) and the product (`paper_2603_26691_b200/`) receive the same arrays.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BC_PERIODIC, BC_REFLECT = 0, 1
RHO_F, NU_F, RHO_P = 1.2, 1.5e-5, 1000.0   # air / water droplets


@dataclass
class Workload:
    """One configuration of BASELINE.json (C1..C5) as concrete numbers."""

    name: str
    dims: tuple
    origin: tuple
    cell_size: tuple
    bc: tuple
    chunk_cells: int
    n_particles: int
    d_range: tuple
    d_dist: str                 # "uniform" | "loguniform"
    w: float
    gravity: tuple
    drag_law: int               # 0 Stokes, 1 Schiller-Naumann
    coupling: int               # 0 one-way, 1 two-way
    dt: float
    steps: int
    field_kind: str             # "uniform" | "taylor_green" | "fourier"
    field_args: dict = field(default_factory=dict)
    seed_field: int = 0
    seed_particles: int = 0
    cite: str = ""

    @property
    def lengths(self):
        return tuple(n * h for n, h in zip(self.dims, self.cell_size))

    @property
    def ncell(self):
        return int(np.prod(self.dims))


def workload(name: str, nranks: int = 1, n_particles: int | None = None) -> Workload:
    """The five BASELINE.json configs."""
    g = (0.0, 0.0, -9.81)
    if name == "C1":   # configs[0]: Stokes settling, closed form
        w = Workload("C1", (16, 16, 16), (0, 0, 0), (1 / 16,) * 3, (BC_PERIODIC,) * 3, 2, 1000, (10e-6, 30e-6),
                     "uniform", 1.0, g, 0, 0, 1e-4, 1000, "uniform", {"v": (0.05, -0.02, 0.0)}, 0, 1,
                     "BJ configs[0]")
    elif name == "C2":  # configs[1]: Taylor-Green, one-way, periodic
        h = 2 * math.pi / 64
        w = Workload("C2", (64, 64, 64), (0, 0, 0), (h,) * 3, (BC_PERIODIC,) * 3, 8, 1_000_000, (50e-6, 1e-3),
                     "loguniform", 1.0, (0.0, 0.0, 0.0), 1, 0, 0.01, 100, "taylor_green", {"U0": 1.0}, 0, 2,
                     "BJ configs[1]")
    elif name == "C3":  # configs[2]: 1e8 two-way 256^3
        w = Workload("C3", (256, 256, 256), (0, 0, 0), (1 / 64,) * 3, (BC_PERIODIC,) * 3, 8, 100_000_000,
                     (5e-6, 25e-6), "uniform", 50.0, g, 1, 1, 5e-3, 100, "fourier",
                     {"u_rms": 0.5, "modes": 256, "kmax": 16}, 3, 4, "BJ configs[2]; w = 50 (P:291)")
    elif name == "C4":  # configs[3]: the paper's chamber, 1.4e9 parcels on one GPU
        w = Workload("C4", (96, 96, 288), (0, 0, 0), (1 / 32,) * 3, (BC_REFLECT,) * 3, 8, 1_400_000_000,
                     (5e-6, 25e-6), "uniform", 50.0, g, 1, 1, 5e-3, 20, "fourier",
                     {"u_rms": 0.3, "modes": 256, "kmax": 16}, 5, 6, "BJ configs[3]; P:289-291")
    elif name == "C5":  # configs[4]: true weak scaling, 1e9 per GPU, slab 192x192x72 per rank
        w = Workload("C5", (192, 192, 72 * nranks), (0, 0, 0), (1 / 64,) * 3, (BC_REFLECT,) * 3, 8,
                     1_000_000_000 * nranks, (5e-6, 25e-6), "uniform", 50.0, g, 1, 1, 5e-3, 20, "fourier",
                     {"u_rms": 0.3, "modes": 256, "kmax": 16}, 7, 8, "BJ configs[4]; P:333 (1e9/GPU)")
    else:
        raise ValueError(name)
    if n_particles is not None:
        w.n_particles = int(n_particles)
    return w


# ---------------------------------------------------------------- fields
def cell_centres(dims, origin, cell_size, z_range=None):
    nx, ny, nz = dims
    z0, z1 = (0, nz) if z_range is None else z_range
    cx = origin[0] + (np.arange(nx) + 0.5) * cell_size[0]
    cy = origin[1] + (np.arange(ny) + 0.5) * cell_size[1]
    cz = origin[2] + (np.arange(z0, z1) + 0.5) * cell_size[2]
    return cx, cy, cz


def uniform_field(dims, v, z_range=None, dtype=np.float32):
    nx, ny, nz = dims
    z0, z1 = (0, nz) if z_range is None else z_range
    F = np.empty((3, z1 - z0, ny, nx), dtype)
    for a in range(3):
        F[a] = v[a]
    return F


def taylor_green(dims, origin, cell_size, U0=1.0, z_range=None, dtype=np.float32):
    """u = U0 sin x cos y cos z, v = -U0 cos x sin y cos z, w = 0 at cell centres."""
    cx, cy, cz = cell_centres(dims, origin, cell_size, z_range)
    X, Y, Z = np.meshgrid(cx, cy, cz, indexing="ij")
    u = U0 * np.sin(X) * np.cos(Y) * np.cos(Z)
    v = -U0 * np.cos(X) * np.sin(Y) * np.cos(Z)
    F = np.zeros((3,) + u.T.shape, np.float64)
    F[0], F[1] = u.T, v.T          # (x,y,z) -> (z,y,x)
    return F.astype(dtype)


def fourier_modes(lengths, modes=256, kmax=16, u_rms=0.3, seed=0):
    """Random divergence-free Fourier modes: k = 2 pi m / L (1 <= |m| <= kmax),
    amplitude ~ |k|^(-11/6) (E ~ k^-5/3), A perpendicular to k, phase phi,
    frequency omega = |k| u_rms; scaled so the per-component rms is u_rms."""
    rng = np.random.default_rng(seed)
    ms = []
    while len(ms) < modes:
        m = rng.integers(-kmax, kmax + 1, 3)
        r = np.linalg.norm(m)
        if 1 <= r <= kmax:
            ms.append(m)
    m = np.array(ms, np.float64)
    k = 2 * np.pi * m / np.array(lengths, np.float64)[None, :]
    kn = np.linalg.norm(k, axis=1)
    e = rng.normal(size=(modes, 3))
    e -= (np.sum(e * k, axis=1) / kn ** 2)[:, None] * k          # project out k
    e /= np.linalg.norm(e, axis=1)[:, None]
    amp = kn ** (-11.0 / 6.0)
    A = e * amp[:, None]
    rms = math.sqrt(np.sum(np.sum(A * A, axis=1)) / 2.0 / 3.0)
    A *= u_rms / rms
    phi = rng.uniform(0, 2 * np.pi, modes)
    omega = kn * u_rms
    return k, A, phi, omega


def fourier_field(dims, origin, cell_size, modes=256, kmax=16, u_rms=0.3, seed=0, t=0.0, z_range=None,
                  device=None):
    """sum_n A_n cos(k_n . x + phi_n + omega_n t) at cell centres -> [3][nz][ny][nx] fp32.
    Evaluated with torch (on `device` if given, else CPU)."""
    import torch
    lengths = tuple(n * h for n, h in zip(dims, cell_size))
    k, A, phi, omega = fourier_modes(lengths, modes, kmax, u_rms, seed)
    cx, cy, cz = cell_centres(dims, origin, cell_size, z_range)
    dev = torch.device(device) if device is not None else torch.device("cpu")
    dt = torch.float32 if dev.type == "cuda" else torch.float64
    X = torch.tensor(cx, dtype=dt, device=dev)[None, None, :]
    Y = torch.tensor(cy, dtype=dt, device=dev)[None, :, None]
    Z = torch.tensor(cz, dtype=dt, device=dev)[:, None, None]
    F = torch.zeros((3, Z.shape[0], Y.shape[1], X.shape[2]), dtype=dt, device=dev)
    for n in range(k.shape[0]):
        arg = float(k[n, 0]) * X + float(k[n, 1]) * Y + float(k[n, 2]) * Z + float(phi[n] + omega[n] * t)
        c = torch.cos(arg)
        for a in range(3):
            F[a] += float(A[n, a]) * c
    return F.to(torch.float32)


def make_field(wl: Workload, t=0.0, z_range=None, device=None):
    """The workload's field (numpy fp32 on CPU, or a torch tensor if device is given)."""
    if wl.field_kind == "uniform":
        F = uniform_field(wl.dims, wl.field_args["v"], z_range)
    elif wl.field_kind == "taylor_green":
        F = taylor_green(wl.dims, wl.origin, wl.cell_size, wl.field_args["U0"], z_range)
    else:
        a = wl.field_args
        F = fourier_field(wl.dims, wl.origin, wl.cell_size, a["modes"], a["kmax"], a["u_rms"], wl.seed_field, t,
                          z_range, device)
        return F if device is not None else F.numpy()
    if device is not None:
        import torch
        return torch.from_numpy(F).to(device)
    return F


# ---------------------------------------------------------------- particles
def particles_np(n, lo, hi, d_range, d_dist="uniform", w=1.0, seed=0, dtype=np.float32):
    """x ~ U[lo, hi) per axis, u = 0, d ~ U or log-U over d_range, constant w."""
    rng = np.random.default_rng(seed)
    lo = np.asarray(lo, np.float64)[:, None]
    hi = np.asarray(hi, np.float64)[:, None]
    x = lo + (hi - lo) * rng.random((3, n))
    x = np.minimum(x.astype(dtype), np.nextafter(hi.astype(dtype), -np.inf))   # stay inside after rounding
    u = np.zeros((3, n), dtype)
    if d_dist == "loguniform":
        d = np.exp(rng.uniform(np.log(d_range[0]), np.log(d_range[1]), n))
    else:
        d = rng.uniform(d_range[0], d_range[1], n)
    return x.astype(dtype), u, d.astype(dtype), np.full(n, w, dtype)


def particles_torch(n, lo, hi, d_range, d_dist="uniform", w=1.0, seed=0, device="cuda"):
    """Same recipe drawn with torch's Philox generator on the device (large N)."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed)
    x = torch.empty((3, n), dtype=torch.float32, device=device)
    for a in range(3):
        x[a].uniform_(float(lo[a]), float(hi[a]), generator=gen)
        x[a].clamp_(max=float(np.nextafter(np.float32(hi[a]), np.float32(-np.inf))))
    u = torch.zeros((3, n), dtype=torch.float32, device=device)
    d = torch.empty(n, dtype=torch.float32, device=device)
    if d_dist == "loguniform":
        d.uniform_(math.log(d_range[0]), math.log(d_range[1]), generator=gen).exp_()
    else:
        d.uniform_(float(d_range[0]), float(d_range[1]), generator=gen)
    wt = torch.full((n,), float(w), dtype=torch.float32, device=device)
    return x, u, d, wt


def domain_box(wl: Workload, z_range=None):
    lo = list(wl.origin)
    hi = [o + n * h for o, n, h in zip(wl.origin, wl.dims, wl.cell_size)]
    if z_range is not None:
        lo[2] = wl.origin[2] + z_range[0] * wl.cell_size[2]
        hi[2] = wl.origin[2] + z_range[1] * wl.cell_size[2]
    return lo, hi


def micro_field(dims, origin, cell_size, seed=0, T0=283.15, dT=1.0, rho_v0=0.0095, rel=0.02,
                u_rms=0.3, dtype=np.float32):
    """5-component cell-centred field (u_x, u_y, u_z, T_f, rho_v) for the droplet
    workload: random-Fourier velocity; temperature
    T0 + dT sin-mode (K); vapour density rho_v0 (1 + rel cos-mode) (kg/m^3; about 1 %
    supersaturated at 283 K).  Plain numbers, no microphysics."""
    U = fourier_field(dims, origin, cell_size, modes=64, kmax=4, u_rms=u_rms, seed=seed).numpy()
    cx, cy, cz = cell_centres(dims, origin, cell_size)
    L = [dims[a] * cell_size[a] for a in range(3)]
    Z, Y, X = np.meshgrid(cz, cy, cx, indexing="ij")
    px, py, pz = (2 * math.pi * (X - origin[0]) / L[0], 2 * math.pi * (Y - origin[1]) / L[1],
                  2 * math.pi * (Z - origin[2]) / L[2])
    T = T0 + dT * np.sin(px) * np.cos(py) * np.cos(pz)
    rv = rho_v0 * (1.0 + rel * np.cos(px + py) * np.sin(pz))
    return np.concatenate([U, T[None], rv[None]]).astype(dtype)


def droplets_np(n, lo, hi, d_range=(5e-6, 30e-6), T_range=(281.0, 285.0), w=100.0, seed=0, dtype=np.float32):
    """Droplet cloud: particles_np positions/diameters, u = 0, T ~ U(T_range), weight w."""
    x, u, d, wv = particles_np(n, lo, hi, d_range, "uniform", w, seed, dtype)
    T = np.random.default_rng(seed + 7919).uniform(T_range[0], T_range[1], n).astype(dtype)
    return x, u, d, T, wv
