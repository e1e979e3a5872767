"""ORACLE — droplet microphysics step, plain numpy, fp64 arithmetic.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` may import this module.  It never imports the product package and
shares no code with it (the product kernel is csrc/st_micro.cu).

What it follows (PAPER.md = P, SPEC.md = S; readings C-28..C-33 in DESIGN.md §3):

* mass transfer, Eq. 7:  dm/dt = 2 pi D_v d rho_v,sat (S_v,f - S_v,p),
  S_v,f = rho_v / rho_v,sat(T_f), S_v,p = 1 by default (C-29);
* saturation vapour density (closure not in the paper, C-30):
  e_s(T) = 610.94 Pa exp(17.625 (T - 273.15) / (T - 273.15 + 243.04))  (Magnus),
  rho_v,sat = e_s / (R_v T), R_v = 461.5 J/(kg K);
* heat transfer, Eq. 12, literal sign (C-31):
  m C_p dT/dt = pi Nu kappa_f d (T_f - T_p) - L dm/dt,  Nu = 2;
* drag, Eq. 9-10 with the Schiller-Naumann factor or Stokes, semi-implicit
  Euler for (u, x), explicit Euler for (m, T);
* sources, Eq. 8, 11, 13, deposited into the cell
  of the sub-step start position (C-10), fluid side = minus the droplet gain (C-8):
  acc_u  += -w (m' u' - m u - m g dt),  acc_rv += -w (m' - m),
  acc_e  += -w C_p (m' T' - m T);   S = acc / (V_cell * dt * nsteps)  (C-13);
* mass floor: m' = max(m + dt dm/dt, 0.01 m), counted (C-32);
* diameter recomputed from the new mass, d' = (6 m' / (pi rho_p))^(1/3) (C-33);
* walls: specular reflection or periodic wrap (C-11, C-12); the C-12
  fix-up is applied to the stored value (a wrap that rounds onto hi is stored as lo).

Storage (C-28): the state (x, u, d, T, w) and the 5-component field are stored in
``store`` precision (float32 for the GPU parity tests, float64 for the pins); every
operation of the step is computed in ``arith`` precision from the stored values —
float64 by default (reading C-28), or float32 (the kernel's fp32 mode, reading C-36:
the same operations in the same order, each rounded to binary32) — and the results are
rounded to ``store`` at the end of each sub-step.  The fluid-side accumulators are
float64 in both modes (each sub-step's deposit is computed in ``arith`` and added in
float64).

Parity status: pinned by tests/test_oracle_micro.py (SPEC worked examples, d^2-law
closed form and first-order convergence, the exact discrete temperature relaxation,
mass / momentum / energy ledgers, equilibrium, interpolation against the C oracle).
Parity unpinned: trajectory values of the coupled step in a non-uniform field beyond
those invariants (no closed form exists); they are checked GPU-vs-oracle only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

BC_PERIODIC, BC_REFLECT = 0, 1
DRAG_STOKES, DRAG_SCHILLER_NAUMANN = 0, 1
R_V = 461.5                     # J/(kg K), water vapour gas constant (C-30)


@dataclass
class MicroProps:
    """Physical constants of the droplet workload (values C-30)."""

    rho_f: float = 1.2          # kg/m^3 air
    nu_f: float = 1.5e-5        # m^2/s
    rho_p: float = 1000.0       # kg/m^3 water
    gravity: tuple = (0.0, 0.0, -9.81)
    drag_law: int = DRAG_SCHILLER_NAUMANN
    D_v: float = 2.5e-5         # m^2/s vapour diffusivity (S:147 example)
    kappa_f: float = 0.025      # W/(m K) air conductivity
    cp_p: float = 4186.0        # J/(kg K) liquid water
    latent: float = 2.45e6      # J/kg latent heat of vaporisation
    nusselt: float = 2.0        # Nu_p
    s_vp: float = 1.0           # S_v,p surface saturation


@dataclass
class MicroMesh:
    dims: tuple                 # (nx, ny, nz)
    origin: tuple
    cell_size: tuple
    bc: tuple = (BC_REFLECT,) * 3


# ---- closures (one function per equation) -------------------------------------------

def saturation_vapor_density(T, arith=np.float64):
    """C-30: Magnus saturation pressure over water, ideal-gas conversion."""
    T = np.asarray(T, dtype=arith)
    tc = T - 273.15
    e_s = 610.94 * np.exp(17.625 * tc / (tc + 243.04))
    return e_s / (R_V * T)


def mass_transfer_rate(d, rho_v, T_f, props: MicroProps, arith=np.float64):
    """Eq. 7: dm/dt = 2 pi D_v d rho_v,sat (S_v,f - S_v,p), kg/s."""
    rs = saturation_vapor_density(T_f, arith)
    s_vf = np.asarray(rho_v, dtype=arith) / rs
    return 2.0 * math.pi * props.D_v * np.asarray(d, dtype=arith) * rs * (s_vf - props.s_vp)


def heat_transfer_rate(d, m, T_p, T_f, dm_dt, props: MicroProps, arith=np.float64):
    """Eq. 12, literal sign (C-31): dT_p/dt in K/s."""
    d = np.asarray(d, dtype=arith)
    q = math.pi * props.nusselt * props.kappa_f * d * (np.asarray(T_f, arith) - T_p)
    return (q - props.latent * np.asarray(dm_dt, arith)) / (np.asarray(m, arith) * props.cp_p)


def drag_factor(Re, law, arith=np.float64):
    """f = C_D Re / 24 (Schiller-Naumann; 0.44 Re/24 above Re = 1000), Stokes f = 1."""
    Re = np.asarray(Re, dtype=arith)
    if law == DRAG_STOKES:
        return np.ones_like(Re)
    return np.where(Re <= 1000.0, 1.0 + 0.15 * np.power(Re, 0.687), 0.44 * Re / 24.0)


def droplet_mass(d, rho_p, arith=np.float64):
    return math.pi / 6.0 * rho_p * np.asarray(d, arith) ** 3


# ---- geometry (C-5, C-6, C-11, C-12) -------------------------------------------------

def cell_index(x, mesh: MicroMesh):
    """C-6: per axis clamp(floor((x - o) / h), 0, n - 1); returns flat cell ids."""
    c = []
    for a in range(3):
        # Python-float constants act as weak scalars: rounded to x's dtype at use
        t = (x[a] - float(mesh.origin[a])) * (1.0 / float(mesh.cell_size[a]))
        f = np.floor(t)
        f = np.where(f >= 0, f, 0)
        f = np.where(f >= mesh.dims[a], mesh.dims[a] - 1, f)
        c.append(f.astype(np.int64))
    nx, ny, _ = mesh.dims
    return (c[2] * ny + c[1]) * nx + c[0]


def _ghost(i, n, bc):
    if bc == BC_PERIODIC:
        return np.mod(i, n)
    return np.clip(i, 0, n - 1)


def trilinear(F, x, mesh: MicroMesh, arith=np.float64):
    """C-5: cell-centred field F[k][nz][ny][nx] at x (3 x n), weights from
    s = (x - o)/h - 1/2, ghost cells by the boundary rule.  Returns k x n (arith)."""
    F = np.asarray(F, dtype=arith)
    K = F.shape[0]
    i0, fr = [], []
    for a in range(3):
        t = (x[a] - float(mesh.origin[a])) * (1.0 / float(mesh.cell_size[a]))
        s = t - 0.5
        fl = np.floor(s)
        i = fl.astype(np.int64)
        f = s - fl
        lowm, highm = i < -1, i > mesh.dims[a] - 1
        i = np.where(lowm, -1, np.where(highm, mesh.dims[a] - 1, i))
        f = np.where(lowm, 0.0, np.where(highm, 1.0, f))
        i0.append(i)
        fr.append(f)
    out = np.zeros((K, x.shape[1]), arith)
    for c in range(2):
        for b in range(2):
            for a in range(2):
                w = (fr[0] if a else 1 - fr[0]) * (fr[1] if b else 1 - fr[1]) * (fr[2] if c else 1 - fr[2])
                ix = _ghost(i0[0] + a, mesh.dims[0], mesh.bc[0])
                iy = _ghost(i0[1] + b, mesh.dims[1], mesh.bc[1])
                iz = _ghost(i0[2] + c, mesh.dims[2], mesh.bc[2])
                out += w * F[:, iz, iy, ix]
    return out


def _apply_bc(xa, ua, lo, hi, bc):
    L = hi - lo
    if bc == BC_PERIODIC:
        xa = np.where(xa < lo, xa + L, np.where(xa >= hi, xa - L, xa))
        return xa, ua
    low, high = xa < lo, xa > hi
    xa = np.where(low, 2 * lo - xa, np.where(high, 2 * hi - xa, xa))
    ua = np.where(low | high, -ua, ua)
    return xa, ua


# ---- the step ------------------------------------------------------------------------

def micro_advance(mesh: MicroMesh, props: MicroProps, x, u, d, T, w, F, dt, nsteps, acc=None,
                  store=np.float32, arith=np.float64):
    """``nsteps`` sub-steps of length dt for every droplet, field F frozen (C-7).

    x, u: 3 x n; d, T, w: n; F: 5 x nz x ny x nx = (u_x, u_y, u_z, T_f, rho_v).
    acc: 5 x ncell float64 fluid-side accumulators (added to; created if None):
    (momentum x, y, z in kg m/s, vapour mass in kg, energy in J).
    Returns (x, u, d, T, acc, n_clamped) with the state rounded to ``store``.
    """
    x = np.array(x, dtype=store)
    u = np.array(u, dtype=store)
    d = np.array(d, dtype=store)
    T = np.array(T, dtype=store)
    w64 = np.asarray(w, dtype=store).astype(arith)
    F = np.asarray(F, dtype=store)
    ncell = int(np.prod(mesh.dims))
    if acc is None:
        acc = np.zeros((5, ncell))
    g = np.asarray(props.gravity, dtype=arith)[:, None]
    dt = arith(dt)
    lo = [float(mesh.origin[a]) for a in range(3)]
    hi = [float(mesh.origin[a] + mesh.dims[a] * mesh.cell_size[a]) for a in range(3)]
    n_clamped = 0
    for _ in range(nsteps):
        xp, up = x.astype(arith), u.astype(arith)
        dp, Tp = d.astype(arith), T.astype(arith)
        # 1 deposit cell = cell of the start position (C-10)
        cell = cell_index(xp, mesh)
        # 2 fluid state at x_p: velocity, temperature, vapour density (C-5)
        f = trilinear(F, xp, mesh, arith)
        uf, Tf, rv = f[0:3], f[3], f[4]
        # 3 drag, semi-implicit Euler (Eq. 9-10)
        slip = uf - up
        Re = np.sqrt(np.sum(slip * slip, axis=0)) * dp / props.nu_f
        tau = props.rho_p * dp * dp / (18.0 * props.rho_f * props.nu_f)
        h = dt / (tau / drag_factor(Re, props.drag_law, arith))
        un = (up + h * uf + dt * g) / (1.0 + h)
        xn = xp + dt * un
        # 4 mass (Eq. 7) and temperature (Eq. 12), explicit Euler from the start state
        m = droplet_mass(dp, props.rho_p, arith)
        mdot = mass_transfer_rate(dp, rv, Tf, props, arith)
        mn = m + dt * mdot
        floor = 0.01 * m
        clamp = mn < floor
        n_clamped += int(np.count_nonzero(clamp))
        mn = np.where(clamp, floor, mn)
        Tn = Tp + dt * heat_transfer_rate(dp, m, Tp, Tf, mdot, props, arith)
        dn = np.cbrt(6.0 * mn / (math.pi * props.rho_p))
        # 5 fluid-side sources into the start cell (Eq. 8, 11, 13; C-8)
        for a in range(3):
            np.add.at(acc[a], cell, -w64 * (mn * un[a] - m * up[a] - m * g[a, 0] * dt))
        np.add.at(acc[3], cell, -w64 * (mn - m))
        np.add.at(acc[4], cell, -w64 * props.cp_p * (mn * Tn - m * Tp))
        # 6 walls / periodic (C-11, C-12), then round the state to storage precision
        for a in range(3):
            xn[a], un[a] = _apply_bc(xn[a], un[a], lo[a], hi[a], mesh.bc[a])
        x, u, d, T = xn.astype(store), un.astype(store), dn.astype(store), Tn.astype(store)
        # C-12 fix-up in storage precision: a wrapped position that rounds onto hi (or
        # below lo) is stored as lo, so the periodic domain stays half-open [lo, hi)
        for a in range(3):
            if mesh.bc[a] == BC_PERIODIC:
                lo_s, hi_s = store(lo[a]), store(hi[a])
                x[a] = np.where((x[a] >= hi_s) | (x[a] < lo_s), lo_s, x[a])
    return x, u, d, T, acc, n_clamped


def sources(acc, mesh: MicroMesh, dt, nsteps):
    """C-13: S = acc / (V_cell * dt * nsteps): N/m^3, kg/(m^3 s), W/m^3."""
    V = mesh.cell_size[0] * mesh.cell_size[1] * mesh.cell_size[2]
    return acc / (V * dt * nsteps)
