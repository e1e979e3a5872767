"""Pins of the droplet-microphysics oracle (oracle/microphysics.py) against
what the paper, SPEC worked examples, textbook tables and closed forms fix — never against
the oracle's own formulas retyped.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import microphysics as M

P = M.MicroProps()
GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _box(dims=(4, 4, 4), h=0.25, bc=M.BC_PERIODIC):
    return M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=(bc,) * 3)


def _uniform_field(mesh, uf=(0.0, 0.0, 0.0), Tf=283.15, rv=0.0095):
    nx, ny, nz = mesh.dims
    F = np.empty((5, nz, ny, nx))
    F[0], F[1], F[2], F[3], F[4] = uf[0], uf[1], uf[2], Tf, rv
    return F


def _one(x=(0.5, 0.5, 0.5), u=(0.0, 0.0, 0.0), d=2e-5, T=283.15, w=1.0):
    return (np.array(x, np.float64)[:, None], np.array(u, np.float64)[:, None],
            np.array([d]), np.array([T]), np.array([w]))


# ---- closures ------------------------------------------------------------------------

def test_saturation_density_spec_and_table():
    """S:154-156 (293.15 K -> 0.0173, 273.15 K -> 0.00485, +-5 %) and the psychrometric
    table (saturated vapour density 9.40e-3 kg/m^3 at 10 C, 30.4e-3 at 30 C, +-2 %)."""
    rs = M.saturation_vapor_density
    for c in GOLDEN["saturation_vapor_density"]["cases"]:
        assert abs(rs(c["T"]) / c["expect"] - 1) < c["rel"]
    assert abs(rs(283.15) / 9.40e-3 - 1) < 0.02
    assert abs(rs(303.15) / 30.4e-3 - 1) < 0.02
    T = np.linspace(200, 350, 301)
    assert np.all(np.diff(rs(T)) > 0) and np.all(rs(T) > 0)


def test_mass_transfer_spec_example():
    """d=1e-5, D_v=2.5e-5, rho_v,sat=0.01, S_v,f - S_v,p = 0.01 -> 1.5708e-13 kg/s."""
    from scipy.optimize import brentq
    g = GOLDEN["mass_transfer_rate"]
    T = brentq(lambda t: M.saturation_vapor_density(t) - g["rho_v_sat"], 250.0, 320.0, xtol=1e-12)
    r = M.mass_transfer_rate(g["d_p"], g["rho_v_sat"] * (1 + g["dS"]), T, M.MicroProps(D_v=g["D_v"]))
    assert abs(r / g["expect"] - 1) < g["rel"]
    assert M.mass_transfer_rate(1e-5, M.saturation_vapor_density(T), T, P) == 0.0
    assert M.mass_transfer_rate(1e-5, 0.0102, T, P) > 0


def test_heat_transfer_signs_literal_eq12():
    """T_p = T_f, no mass transfer -> 0; warmer fluid -> warms; literal Eq. 12
    sign (C-31): evaporation (dm/dt < 0) at T_p = T_f gives +L|dm/dt|/(m C_p)."""
    m = M.droplet_mass(2e-5, P.rho_p)
    assert M.heat_transfer_rate(2e-5, m, 283.0, 283.0, 0.0, P) == 0.0
    assert M.heat_transfer_rate(2e-5, m, 283.0, 284.0, 0.0, P) > 0
    r = M.heat_transfer_rate(2e-5, m, 283.0, 283.0, -1e-13, P)
    assert r == pytest.approx(2.45e6 * 1e-13 / (m * 4186.0), rel=1e-12)


def test_drag_factor_spec_value():
    """Re = 1 -> C_D = 27.6, i.e. f = C_D Re / 24 = 1.15; continuity gap at 1000."""
    assert M.drag_factor(1.0, M.DRAG_SCHILLER_NAUMANN) == pytest.approx(1.15, rel=1e-12)
    assert M.drag_factor(1000.0, M.DRAG_SCHILLER_NAUMANN) * 24 / 1000 == pytest.approx(18.262006 * 24 / 1000, rel=1e-6)


# ---- the step: closed forms ----------------------------------------------------------

def test_equilibrium_leaves_everything_unchanged():
    """resting droplet, quiescent saturated fluid at the droplet temperature, no
    gravity -> state unchanged, all sources zero."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0))
    Tf = 283.15
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    x, u, d, T, w = _one(T=Tf)
    xn, un, dn, Tn, acc, nc = M.micro_advance(mesh, props, x, u, d, T, w, F, 1e-3, 10, store=np.float64)
    assert np.array_equal(xn, x) and np.array_equal(un, u) and nc == 0
    assert abs(dn[0] / d[0] - 1) < 1e-14 and Tn[0] == T[0]
    assert np.max(np.abs(acc)) < 1e-25


def test_d2_law_closed_form_and_first_order():
    """Eq. 7 with m = rho_p pi d^3/6 at fixed rho_v,sat and S_v,f: d^2(t) = d0^2 +
    8 D_v rho_sat (S_v,f - S_v,p) t / rho_p (the d^2-law); explicit Euler converges to it
    at first order."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0))
    Tf = 283.15
    rs = 9.40e-3 * 1.0                                    # table value only sets the scale
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)) * 0.9)   # 10 % subsaturated
    d0, t_end = 10e-6, 0.1
    rsat = float(M.saturation_vapor_density(Tf))
    exact = math.sqrt(d0 ** 2 + 8 * props.D_v * rsat * (-0.1) * t_end / props.rho_p)
    assert 0.5 * d0 < exact < d0 and rs > 0
    errs = []
    for n in (50, 100, 200, 400):
        x, u, d, T, w = _one(d=d0, T=Tf)
        _, _, dn, _, _, nc = M.micro_advance(mesh, props, x, u, d, T, w, F, t_end / n, n, store=np.float64)
        errs.append(abs(dn[0] - exact) / exact)
        assert nc == 0
    assert errs[-1] < 2e-3
    for a, b in zip(errs, errs[1:]):
        assert 1.7 < a / b < 2.3


def test_temperature_relaxation_exact_discrete():
    """Eq. 12 with dm/dt = 0 (saturated fluid): explicit Euler gives exactly
    T_n - T_f = (1 - dt/tau_T)^n (T_0 - T_f), tau_T = m C_p / (pi Nu kappa d)."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0))
    Tf, T0, d0, dt, n = 285.0, 281.0, 20e-6, 2e-3, 25
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    m = math.pi / 6 * props.rho_p * d0 ** 3
    tau_T = m * props.cp_p / (math.pi * 2.0 * props.kappa_f * d0)
    x, u, d, T, w = _one(d=d0, T=T0)
    _, _, _, Tn, acc, _ = M.micro_advance(mesh, props, x, u, d, T, w, F, dt, n, store=np.float64)
    want = Tf + (1 - dt / tau_T) ** n * (T0 - Tf)
    assert Tn[0] == pytest.approx(want, rel=1e-12)
    # energy handed to the fluid = minus the droplet's enthalpy gain (Eq. 13)
    assert acc[4].sum() == pytest.approx(-props.cp_p * m * (Tn[0] - T0), rel=1e-9)


def test_stokes_relaxation_spec():
    """uniform u_f, Stokes drag, no exchange -> u(t) = u_f + (u0 - u_f) exp(-t/tau_p),
    first-order convergence of the semi-implicit step."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0), drag_law=M.DRAG_STOKES)
    Tf = 283.15
    F = _uniform_field(mesh, uf=(0.2, 0.0, 0.0), Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    d0 = 20e-6
    tau = props.rho_p * d0 ** 2 / (18 * props.rho_f * props.nu_f)
    t_end = 2 * tau
    exact = 0.2 + (0.0 - 0.2) * math.exp(-t_end / tau)
    errs = []
    for n in (20, 40, 80, 160):
        x, u, d, T, w = _one(d=d0, T=Tf)
        _, un, _, _, _, _ = M.micro_advance(mesh, props, x, u, d, T, w, F, t_end / n, n, store=np.float64)
        errs.append(abs(un[0, 0] - exact))
    for a, b in zip(errs, errs[1:]):
        assert 1.7 < a / b < 2.3


def test_mass_floor_clamps():
    """S:199 (C-32): a step that would remove more than 99 % of the mass stops at 1 %."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0))
    F = _uniform_field(mesh, Tf=300.0, rv=0.0)          # bone-dry, warm
    x, u, d, T, w = _one(d=1e-6, T=300.0)
    _, _, dn, _, acc, nc = M.micro_advance(mesh, props, x, u, d, T, w, F, 1.0, 1, store=np.float64)
    assert nc == 1
    assert dn[0] == pytest.approx(1e-6 * 0.01 ** (1 / 3), rel=1e-12)
    assert acc[3].sum() == pytest.approx(0.99 * M.droplet_mass(1e-6, props.rho_p), rel=1e-12)


def test_reflection_conserves_speed():
    """a droplet crossing x = 0 with u = (-1, 0, 0) comes back mirrored."""
    mesh = _box(bc=M.BC_REFLECT)
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0), drag_law=M.DRAG_STOKES, rho_p=1e12)   # ballistic
    Tf = 283.15
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    x, u, d, T, w = _one(x=(0.001, 0.5, 0.5), u=(-1.0, 0.0, 0.0), T=Tf)
    xn, un, _, _, _, _ = M.micro_advance(mesh, props, x, u, d, T, w, F, 0.002, 1, store=np.float64)
    # interior twin moving the other way: same drag, no wall -> same speed, exactly
    x2, u2, d2, T2, w2 = _one(x=(0.5, 0.5, 0.5), u=(1.0, 0.0, 0.0), T=Tf)
    _, un2, _, _, _, _ = M.micro_advance(mesh, props, x2, u2, d2, T2, w2, F, 0.002, 1, store=np.float64)
    assert un[0, 0] > 0 and un[0, 0] == un2[0, 0]
    assert xn[0, 0] == pytest.approx(0.002 * un[0, 0] - 0.001, rel=1e-9)


# ---- ledgers and interpolation -------------------------------------------------------

def test_ledgers_close_random_cloud():
    """in a periodic box the droplet mass gain plus the vapour source is 0; the
    momentum change plus the momentum source equals the gravity impulse; the enthalpy
    change plus the energy source is 0 (all to 1e-10 relative)."""
    mesh = M.MicroMesh(dims=(16, 12, 8), origin=(0.0, 0.0, 0.0), cell_size=(0.25,) * 3, bc=(M.BC_PERIODIC,) * 3)
    F = synth.micro_field(mesh.dims, mesh.origin, mesh.cell_size, seed=3, dtype=np.float64)
    x, u, d, T, w = synth.droplets_np(3000, (0, 0, 0), (4.0, 3.0, 2.0), seed=5, dtype=np.float64)
    dt, n = 5e-3, 4
    xn, un, dn, Tn, acc, _ = M.micro_advance(mesh, P, x, u, d, T, w, F, dt, n, store=np.float64)
    m0, m1 = M.droplet_mass(d, P.rho_p), M.droplet_mass(dn, P.rho_p)
    dM = np.sum(w * (m1 - m0))
    assert abs(dM + acc[3].sum()) <= 1e-10 * np.sum(w * m0) * 1e-3 + 1e-10 * abs(dM)
    assert np.sign(dM) != 0
    E0, E1 = np.sum(w * m0 * T) * P.cp_p, np.sum(w * m1 * Tn) * P.cp_p
    assert abs((E1 - E0) + acc[4].sum()) <= 1e-10 * abs(E1 - E0) + 1e-6 * 1e-10 * E0
    # momentum: per sub-step gravity impulse uses that sub-step's start mass, so rebuild it
    g = np.array(P.gravity)
    imp = np.zeros(3)
    xs, us, ds, Ts = x, u, d, T
    for _ in range(n):
        imp += g * dt * np.sum(w * M.droplet_mass(ds, P.rho_p))
        xs, us, ds, Ts, _, _ = M.micro_advance(mesh, P, xs, us, ds, Ts, w, F, dt, 1, store=np.float64)
    p0, p1 = (w * m0 * u).sum(axis=1), (w * m1 * un).sum(axis=1)
    scale = np.abs(imp).max()
    assert np.all(np.abs((p1 - p0) + acc[:3].sum(axis=1) - imp) <= 1e-10 * scale)


def test_trilinear_matches_pinned_c_oracle():
    """The 5-component interpolation follows the same C-5 rule as the pinned C oracle
    (test_oracle_pins): components (0,1,2) and (3,4,0) through orc_interpolate_f64."""
    for bc in (M.BC_PERIODIC, M.BC_REFLECT):
        mesh = M.MicroMesh(dims=(16, 12, 8), origin=(-1.0, 0.5, 0.0), cell_size=(0.25,) * 3, bc=(bc,) * 3)
        F = synth.micro_field(mesh.dims, mesh.origin, mesh.cell_size, seed=1, dtype=np.float64)
        x, *_ = synth.droplets_np(2000, (-1.0, 0.5, 0.0), (3.0, 3.5, 2.0), seed=2, dtype=np.float64)
        got = M.trilinear(F, x, mesh)
        sim = oracle.Sim(oracle.Mesh(dims=mesh.dims, origin=mesh.origin, cell_size=mesh.cell_size,
                                     chunk_cells=4, bc=mesh.bc), oracle.Physics(), precision="f64")
        a = sim.interpolate(x, F[0:3])
        b = sim.interpolate(x, np.stack([F[3], F[4], F[0]]))
        np.testing.assert_allclose(got[0:3], a, rtol=0, atol=1e-13)
        np.testing.assert_allclose(got[3], b[0], rtol=1e-14)
        np.testing.assert_allclose(got[4], b[1], rtol=1e-13)


# ---- deposit cell (C-10) and periodic wrap (C-12) ------------------------------------

def test_deposit_goes_to_start_cell():
    """C-10 ("the Eulerian grid cell containing the particle"; Eq. 8, 11, 13): a
    droplet that crosses a face during the sub-step deposits all five fluid-side sources
    into the cell of the sub-step START position; the end cell receives nothing.  The
    vapour source is minus the droplet's mass gain, read from its new diameter."""
    mesh = _box(dims=(4, 4, 4), h=0.25, bc=M.BC_REFLECT)
    props = M.MicroProps(gravity=(0.0, 0.0, -9.81), drag_law=M.DRAG_STOKES)
    F = _uniform_field(mesh, uf=(0.0, 0.0, 0.0), Tf=290.0, rv=0.006)        # sub-saturated: evaporates
    x, u, d, T, w = _one(x=(0.499, 0.6, 0.3), u=(2.0, 0.0, 0.0), d=4e-4, T=285.0, w=3.0)
    dt = 2e-3
    xn, un, dn, Tn, acc, _ = M.micro_advance(mesh, props, x, u, d, T, w, F, dt, 1, store=np.float64)
    assert xn[0, 0] > 0.5                                   # crossed x = 0.5 into cell ix = 2
    start = (1 * 4 + 2) * 4 + 1                             # (iz, iy, ix) = (1, 2, 1)
    end = (1 * 4 + 2) * 4 + 2
    for k in range(5):
        nz = np.flatnonzero(acc[k])
        assert nz.tolist() == ([] if k == 1 else [start]), (k, nz)     # no y motion: S_u,y = 0
    assert acc[:, end].tolist() == [0.0] * 5
    m0, m1 = M.droplet_mass(d, props.rho_p), M.droplet_mass(dn, props.rho_p)
    assert m1[0] < m0[0]
    assert acc[3, start] == pytest.approx(-3.0 * (m1[0] - m0[0]), rel=1e-9)


@pytest.mark.parametrize("side", ["lo", "hi"])
def test_periodic_wrap_stays_half_open_fp32(side):
    """C-12 (the main oracle's P-8 fix-up): after a periodic wrap the STORED fp32
    position lies in [lo, hi).  A droplet 1e-9 m below lo wraps to lo + L - 1e-9, which
    rounds to hi in fp32; C-12 maps it to lo.  From just below hi the wrap lands at lo
    exactly.  Without the fix-up the stored x would equal hi (outside [lo, hi))."""
    mesh = _box(dims=(4, 4, 4), h=0.25, bc=M.BC_PERIODIC)
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0), drag_law=M.DRAG_STOKES, rho_p=1e9)   # ballistic
    Tf = 283.15
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    if side == "lo":
        x, u, d, T, w = _one(x=(1e-9, 0.5, 0.5), u=(-1.0, 0.0, 0.0), T=Tf)
    else:
        x, u, d, T, w = _one(x=(float(np.nextafter(np.float32(1.0), np.float32(0.0))), 0.5, 0.5),
                             u=(1.0, 0.0, 0.0), T=Tf)
    xn, un, *_ = M.micro_advance(mesh, props, x, u, d, T, w, F, 2e-9, 1, store=np.float32)
    assert xn.dtype == np.float32
    assert 0.0 <= xn[0, 0] < 1.0
    if side == "lo":
        assert xn[0, 0] == np.float32(0.0)
    assert un[0, 0] == np.float32(u[0, 0])                 # a wrap keeps the velocity


# ---- fp32 arithmetic mode (reading C-36) ----------------------------------------------

def _stable_cloud(n=20_000):
    """Droplets of 10-30 um with dt = 1 ms: dt / tau_T <= 0.71 and dt / tau_p <= 3.3 under
    the semi-implicit drag, so the explicit Eq. 7 / Eq. 12 updates are contractive and an
    fp32 rounding is not amplified from step to step."""
    dims, h = (24, 20, 12), 0.125
    mesh = M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=(0, 0, 1))
    F = synth.micro_field(dims, mesh.origin, mesh.cell_size, seed=11)
    x, u, d, T, w = synth.droplets_np(n, (0.0, 0.0, 0.0), (3.0, 2.5, 1.5), seed=12, d_range=(10e-6, 30e-6))
    return mesh, F, x, u, d, T, w


def test_fp32_mode_rounds_every_operation_to_binary32():
    """C-36: the closures and the interpolation compute in float32 (no silent promotion
    through a float64 constant), and the fp32 step is not the fp64 step."""
    d = np.array([12e-6, 25e-6], np.float32)
    Tf = np.array([282.0, 284.5], np.float32)
    rv = np.array([9e-3, 8e-3], np.float32)
    f32 = np.float32
    assert M.saturation_vapor_density(Tf, f32).dtype == f32
    assert M.mass_transfer_rate(d, rv, Tf, P, f32).dtype == f32
    assert M.droplet_mass(d, P.rho_p, f32).dtype == f32
    assert M.drag_factor(np.array([0.0, 3.0, 2e3], f32), M.DRAG_SCHILLER_NAUMANN, f32).dtype == f32
    m = M.droplet_mass(d, P.rho_p, f32)
    assert M.heat_transfer_rate(d, m, Tf, Tf, m, P, f32).dtype == f32
    mesh, F, x, u, d, T, w = _stable_cloud(2000)
    assert M.trilinear(F, x, mesh, f32).dtype == f32
    r64 = M.micro_advance(mesh, P, x, u, d, T, w, F, 1e-3, 3)
    r32 = M.micro_advance(mesh, P, x, u, d, T, w, F, 1e-3, 3, arith=f32)
    assert np.mean(r32[2] == r64[2]) < 0.9           # d: the modes really differ
    assert r32[4].dtype == np.float64                # accumulators stay fp64


@pytest.mark.parametrize("nsteps", [1, 5, 20])
def test_fp32_mode_within_rounding_bound_of_fp64(nsteps):
    """The fp32 oracle stays within the binary32 rounding bound of the fp64 oracle
    (tests/micro_bounds.py) on a 2e4-droplet stable cloud."""
    from tests.micro_bounds import check_fp32, run_with_gross
    mesh, F, x, u, d, T, w = _stable_cloud()
    ref = run_with_gross(mesh, P, x, u, d, T, w, F, 1e-3, nsteps)
    got = M.micro_advance(mesh, P, x, u, d, T, w, F, 1e-3, nsteps, arith=np.float32)
    u_scale = float(np.max(np.abs(F[:3]))) + 9.81 * 1e-3 * nsteps
    check_fp32(got, ref[:6], ref[6], mesh, nsteps, u_scale, f"n={nsteps}")
    assert got[5] == ref[5]


def test_fp32_temperature_relaxation_closed_form():
    """Eq. 12 closed form (test_temperature_relaxation_exact_discrete) in fp32 mode:
    T_n - T_f = (1 - dt/tau_T)^n (T_0 - T_f) to the binary32 rounding of 25 sub-steps."""
    mesh = _box()
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0))
    Tf, T0, d0, dt, n = 285.0, 281.0, 20e-6, 2e-3, 25
    F = _uniform_field(mesh, Tf=Tf, rv=float(M.saturation_vapor_density(Tf)))
    m = math.pi / 6 * props.rho_p * d0 ** 3
    tau_T = m * props.cp_p / (math.pi * 2.0 * props.kappa_f * d0)
    x, u, d, T, w = _one(d=d0, T=T0)
    _, _, _, Tn, _, _ = M.micro_advance(mesh, props, x, u, d, T, w, F, dt, n, arith=np.float32)
    want = Tf + (1 - dt / tau_T) ** n * (T0 - Tf)
    assert abs(float(Tn[0]) - want) <= 4 * n * np.finfo(np.float32).eps * Tf
    assert float(Tn[0]) != pytest.approx(T0, abs=0.5)


def test_fp32_vapour_ledger_closes():
    """S:186 in fp32 mode: the droplets' mass gain plus the vapour source is zero to the
    binary32 rounding of the per-droplet mass differences."""
    from tests.micro_bounds import C_ACC, EPS32
    mesh, F, x, u, d, T, w = _stable_cloud(5000)
    _, _, dn, _, acc, _ = M.micro_advance(mesh, P, x, u, d, T, w, F, 1e-3, 4, arith=np.float32)
    m0 = M.droplet_mass(d.astype(np.float64), P.rho_p)
    m1 = M.droplet_mass(dn.astype(np.float64), P.rho_p)
    dM = np.sum(w * (m1 - m0))
    assert dM != 0
    assert abs(dM + acc[3].sum()) <= C_ACC * EPS32 * np.sum(w * (m0 + m1)) * 4
