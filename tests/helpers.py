"""Shared test helpers: build the GPU context and the oracle from one workload."""
from __future__ import annotations

import numpy as np

import synth


def gpu_config(wl: synth.Workload, capacity=None, rebin_interval=1, integrator=0):
    from paper_2603_26691_b200 import Config
    return Config(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells, bc=wl.bc,
                  rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity,
                  drag_law=wl.drag_law, integrator=integrator, coupling=wl.coupling,
                  rebin_interval=rebin_interval, capacity=capacity or max(wl.n_particles, 1))


def oracle_sim(wl: synth.Workload, precision="f32", rebin_interval=1, integrator=0, nranks=1):
    import oracle
    mesh = oracle.Mesh(dims=wl.dims, origin=wl.origin, cell_size=wl.cell_size, chunk_cells=wl.chunk_cells,
                       bc=wl.bc)
    phys = oracle.Physics(rho_f=synth.RHO_F, nu_f=synth.NU_F, rho_p=synth.RHO_P, gravity=wl.gravity,
                          drag_law=wl.drag_law, integrator=integrator, coupling=wl.coupling)
    return oracle.Sim(mesh, phys, rebin_interval=rebin_interval, precision=precision, nranks=nranks)


def by_id(p: dict) -> dict:
    o = np.argsort(p["id"], kind="stable")
    return {k: (v[:, o] if v.ndim == 2 else v[o]) for k, v in p.items()}


def periodic_dist(a, b, L):
    """|a - b| with each axis taken modulo L_axis (columns of [3][n])."""
    L = np.asarray(L, np.float64)[:, None]
    d = np.abs(a.astype(np.float64) - b.astype(np.float64))
    return np.minimum(d, L - d)
