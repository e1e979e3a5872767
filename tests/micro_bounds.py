"""Error bounds for the droplet step's fp32 arithmetic mode (reading C-36).
Test infrastructure: uses only oracle/ and numpy.

In fp32 mode every operation of a sub-step rounds to binary32 (unit roundoff
eps32 = 2^-23 relative spacing).  Each droplet's deposit is a difference of products
(w (m'u' - m u - m g dt), w (m' - m), w C_p (m'T' - m T)); along the chain
slip -> Re -> f -> h -> u' -> deposit about twenty roundings reach a term, so per sub-step
and cell the deposit error is bounded by

    |acc32 - acc64| <= C_ACC * eps32 * G,   G = sum over droplets in the cell of w times
    the term magnitudes (|m'u'| + |m u| + |m g dt|, |m'| + |m|, C_p (|m'T'| + |m T|)),

with C_ACC = 64 (observed <= 20 on the 2e4-droplet stable cloud).  The fp32 state
carries about one rounding per sub-step in d and T (STATE_ULPS = 4 per sub-step),
positions an ulp of the domain extent per sub-step, velocities C_ACC eps32 of the
velocity scale.  A droplet whose start position sits within an ulp of a cell face may
deposit into the neighbouring cell in one precision and not the other; the global sums
are immune to such flips, so at most MAX_FLIP_CELLS cells may exceed the bound."""
from __future__ import annotations

import numpy as np

from oracle import microphysics as M

EPS32 = float(np.finfo(np.float32).eps)
C_ACC = 64.0
STATE_ULPS = 4.0
MAX_FLIP_CELLS = 4


def run_with_gross(mesh, props, x, u, d, T, w, F, dt, nsteps, arith=np.float64):
    """Oracle run one sub-step at a time (identical to one nsteps call: the state is
    rounded to fp32 storage every sub-step) that also returns the per-cell gross G."""
    ncell = int(np.prod(mesh.dims))
    G = np.zeros((5, ncell))
    g = np.asarray(props.gravity, np.float64)
    w64 = np.asarray(w, np.float64)
    acc = None
    clamps = 0
    for _ in range(nsteps):
        x1, u1, d1, T1, acc, c = M.micro_advance(mesh, props, x, u, d, T, w, F, dt, 1, acc=acc, arith=arith)
        clamps += c
        cell = M.cell_index(np.asarray(x, np.float64), mesh)
        m0 = M.droplet_mass(np.asarray(d, np.float64), props.rho_p)
        m1 = M.droplet_mass(np.asarray(d1, np.float64), props.rho_p)
        for k in range(3):
            np.add.at(G[k], cell, w64 * (np.abs(m1 * u1[k]) + np.abs(m0 * u[k]) + np.abs(m0 * g[k] * dt)))
        np.add.at(G[3], cell, w64 * (m1 + m0))
        np.add.at(G[4], cell, w64 * props.cp_p * (m1 * np.abs(T1) + m0 * np.abs(T)))
        x, u, d, T = x1, u1, d1, T1
    return x, u, d, T, acc, clamps, G


def check_fp32(got, ref, G, mesh, nsteps, u_scale, tag=""):
    """got / ref = (x, u, d, T, acc[5, ncell], clamps); ref from the fp64 or fp32 oracle."""
    gx, gu, gd, gT, gacc, _ = got
    rx, ru, rd, rT, racc, _ = ref
    L = max(mesh.origin[a] + mesh.dims[a] * mesh.cell_size[a] for a in range(3))
    tol_state = STATE_ULPS * nsteps * EPS32
    f64 = lambda a: np.asarray(a, np.float64)  # noqa: E731
    assert np.max(np.abs(f64(gx) - f64(rx))) <= tol_state * L, tag
    assert np.max(np.abs(f64(gu) - f64(ru))) <= C_ACC * EPS32 * u_scale, tag
    assert np.max(np.abs(f64(gd) / f64(rd) - 1)) <= tol_state, tag
    assert np.max(np.abs(f64(gT) / f64(rT) - 1)) <= tol_state, tag
    for k in range(5):
        err = np.abs(gacc[k] - racc[k])
        bound = C_ACC * EPS32 * G[k]
        assert np.count_nonzero(err > bound) <= MAX_FLIP_CELLS, (tag, k, float(np.max(err / (bound + 1e-300))))
        assert abs(gacc[k].sum() - racc[k].sum()) <= C_ACC * EPS32 * G[k].sum(), (tag, k)
