"""GPU parity of the droplet-microphysics step (st_micro_advance) against
the fp64-arithmetic / fp32-storage oracle (oracle/microphysics.py, reading C-28), through
the C-ABI.  Tolerances: both sides round the same fp64 operations in the
same order, so the fp32 state agrees to within one fp32 ulp of a rare last-bit flip
(libm exp/pow/cbrt may differ by one fp64 ulp); sources differ only by the fp64
summation order plus those flips: 1e-6 of the largest cell magnitude per component."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402
from oracle import microphysics as M  # noqa: E402


def _setup(n, dims=(24, 20, 12), h=0.125, bc=(0, 0, 1), seed=11, field_kw=None, drop_kw=None):
    mesh = M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=bc)
    F = synth.micro_field(dims, mesh.origin, mesh.cell_size, seed=seed, **(field_kw or {}))
    hi = tuple(dims[a] * h for a in range(3))
    x, u, d, T, w = synth.droplets_np(n, (0.0, 0.0, 0.0), hi, seed=seed + 1, **(drop_kw or {}))
    return mesh, F, x, u, d, T, w


def _gpu_run(mesh, props, F, x, u, d, T, w, dt, calls, arithmetic="fp64"):
    from paper_2603_26691_b200 import MicroConfig, micro_advance
    cfg = MicroConfig(dims=mesh.dims, origin=mesh.origin, cell_size=mesh.cell_size, bc=mesh.bc,
                      rho_f=props.rho_f, nu_f=props.nu_f, rho_p=props.rho_p, gravity=props.gravity,
                      drag_law=props.drag_law, D_v=props.D_v, kappa_f=props.kappa_f, cp_p=props.cp_p,
                      latent=props.latent, nusselt=props.nusselt, s_vp=props.s_vp, arithmetic=arithmetic)
    dev = torch.device("cuda:0")
    tx, tu, td, tT, tw = (torch.from_numpy(np.ascontiguousarray(a)).to(dev) for a in (x, u, d, T, w))
    tF = torch.from_numpy(np.ascontiguousarray(F)).to(dev)
    acc = torch.zeros((5,) + tuple(reversed(mesh.dims)), dtype=torch.float64, device=dev)
    clamps = 0
    for k in calls:
        clamps += micro_advance(cfg, tx, tu, td, tT, tw, tF, dt, k, acc)
    return (tx.cpu().numpy(), tu.cpu().numpy(), td.cpu().numpy(), tT.cpu().numpy(),
            acc.cpu().numpy().reshape(5, -1), clamps)


def _oracle_run(mesh, props, F, x, u, d, T, w, dt, calls):
    acc, clamps = None, 0
    for k in calls:
        x, u, d, T, acc, c = M.micro_advance(mesh, props, x, u, d, T, w, F, dt, k, acc=acc)
        clamps += c
    return x, u, d, T, acc, clamps


def _compare(g, o, mesh, tag=""):
    gx, gu, gd, gT, gacc, gc = g
    ox, ou, od, oT, oacc, oc = o
    L = max(mesh.dims[a] * mesh.cell_size[a] for a in range(3))
    assert gc == oc, tag
    np.testing.assert_allclose(gx, ox, rtol=0, atol=2e-7 * L, err_msg=tag)
    np.testing.assert_allclose(gu, ou, rtol=1e-5, atol=1e-6, err_msg=tag)
    np.testing.assert_allclose(gd, od, rtol=1e-6, atol=0, err_msg=tag)
    np.testing.assert_allclose(gT, oT, rtol=1e-6, atol=0, err_msg=tag)
    assert np.mean(gx == ox) > 0.999 and np.mean(gd == od) > 0.999 and np.mean(gT == oT) > 0.999, tag
    for k in range(5):
        scale = np.max(np.abs(oacc[k])) + 1e-300
        assert np.max(np.abs(gacc[k] - oacc[k])) <= 1e-6 * scale, (tag, k)


@pytest.mark.parametrize("n,calls,bc", [
    (20_000, (3, 2), (0, 0, 1)),        # many tiles + ragged tail, two calls accumulate
    (257, (4,), (1, 1, 1)),             # one full CTA + 1, all walls reflecting
    (1, (6,), (0, 0, 0)),               # a single droplet, fully periodic
])
def test_micro_parity(n, calls, bc):
    mesh, F, x, u, d, T, w = _setup(n, bc=bc)
    props = M.MicroProps()
    dt = 5e-3
    g = _gpu_run(mesh, props, F, x, u, d, T, w, dt, calls)
    o = _oracle_run(mesh, props, F, x, u, d, T, w, dt, calls)
    _compare(g, o, mesh, f"n={n}")


def test_micro_parity_binned_store():
    """Droplets ordered by cell (the binned store of C-15): long runs of lanes share a start
    cell, so the segmented warp reduction of the deposits is exercised; 8 droplets/cell."""
    mesh, F, x, u, d, T, w = _setup(8 * 24 * 20 * 12 + 77)
    c = np.floor(x.astype(np.float64) / 0.125).astype(np.int64)
    order = np.lexsort((c[0], c[1], c[2]))
    x, u, d, T, w = x[:, order].copy(), u[:, order].copy(), d[order].copy(), T[order].copy(), w[order].copy()
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 5e-3, (2, 3))
    o = _oracle_run(mesh, props, F, x, u, d, T, w, 5e-3, (2, 3))
    _compare(g, o, mesh, "binned")


def test_micro_parity_stokes_fast_flow_walls():
    """Stokes drag, u_rms = 2 m/s field so droplets cross cells and hit the z walls."""
    mesh, F, x, u, d, T, w = _setup(5000, field_kw={"u_rms": 2.0}, drop_kw={"d_range": (20e-6, 60e-6)})
    props = M.MicroProps(drag_law=M.DRAG_STOKES)
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 5e-3, (8,))
    o = _oracle_run(mesh, props, F, x, u, d, T, w, 5e-3, (8,))
    _compare(g, o, mesh, "stokes")


def test_micro_mass_floor_clamps_match():
    """Dry, warm field with tiny droplets and a long step: the C-32 floor engages."""
    mesh, F, x, u, d, T, w = _setup(3000, field_kw={"T0": 300.0, "rho_v0": 1e-4},
                                    drop_kw={"d_range": (0.5e-6, 3e-6)})
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 0.2, (2,))
    o = _oracle_run(mesh, props, F, x, u, d, T, w, 0.2, (2,))
    assert o[5] > 0
    _compare(g, o, mesh, "floor")


def test_micro_empty_and_errors():
    from paper_2603_26691_b200 import MicroConfig, StError, micro_advance
    cfg = MicroConfig(dims=(4, 4, 4), cell_size=(0.25,) * 3)
    dev = torch.device("cuda:0")
    e3 = torch.empty((3, 0), device=dev)
    e1 = torch.empty(0, device=dev)
    F = torch.zeros((5, 4, 4, 4), device=dev)
    acc = torch.zeros((5, 4, 4, 4), dtype=torch.float64, device=dev)
    assert micro_advance(cfg, e3, e3.clone(), e1, e1.clone(), e1.clone(), F, 1e-3, 3, acc) == 0
    x = torch.full((3, 4), 0.5)                     # host and device arrays mixed -> rejected
    with pytest.raises(StError):
        micro_advance(cfg, x, x.clone(), torch.ones(4), torch.ones(4), torch.ones(4), F, 1e-3, 1, acc)


def test_micro_host_arrays_equal_device_arrays():
    """All-host arrays are staged through the device: the same results as device arrays."""
    from paper_2603_26691_b200 import MicroConfig, micro_advance
    mesh, F, x, u, d, T, w = _setup(3000)
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 5e-3, (2,))
    cfg = MicroConfig(dims=mesh.dims, origin=mesh.origin, cell_size=mesh.cell_size, bc=mesh.bc)
    hx, hu, hd, hT = (np.ascontiguousarray(a).copy() for a in (x, u, d, T))
    acc = np.zeros((5,) + tuple(reversed(mesh.dims)), np.float64)
    micro_advance(cfg, hx, hu, hd, hT, np.ascontiguousarray(w), np.ascontiguousarray(F), 5e-3, 2, acc)
    assert np.array_equal(hx, g[0]) and np.array_equal(hd, g[2]) and np.array_equal(hT, g[3])
    assert np.allclose(acc.reshape(5, -1), g[4], rtol=1e-12, atol=1e-300 + 1e-9 * np.abs(g[4]).max())


def test_micro_full_size_sampled():
    """2e7 droplets on the bench grid (192 x 192 x 72, h = 1/32): droplets are independent
    given the frozen field, so the oracle run on a 2000-droplet sample gives exactly their
    states; the vapour ledger of the whole field closes in fp64."""
    from paper_2603_26691_b200 import MicroConfig, micro_advance
    dims, h = (192, 192, 72), 1.0 / 32
    mesh = M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=(0, 0, 1))
    F = synth.micro_field(dims, mesh.origin, mesh.cell_size, seed=4)
    n = 20_000_000
    hi = (6.0, 6.0, 2.25)
    x, u, d, T, w = synth.droplets_np(n, (0.0, 0.0, 0.0), hi, seed=9)
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 5e-3, (2,))
    idx = np.random.default_rng(0).choice(n, 2000, replace=False)
    o = M.micro_advance(mesh, props, x[:, idx], u[:, idx], d[idx], T[idx], w[idx], F, 5e-3, 2)
    np.testing.assert_allclose(g[0][:, idx], o[0], rtol=0, atol=2e-7 * 6.0)
    np.testing.assert_allclose(g[2][idx], o[2], rtol=1e-6)
    np.testing.assert_allclose(g[3][idx], o[3], rtol=1e-6)
    m0 = M.droplet_mass(d, props.rho_p)
    m1 = M.droplet_mass(g[2], props.rho_p)
    dM = np.sum(w.astype(np.float64) * (m1 - m0))
    # fp32 storage of d limits the droplet-side sum, not the GPU accumulation
    assert abs(g[4][3].sum() + dM) <= 1e-4 * abs(dM) + 1e-6 * np.sum(w * m0) * 1e-6


@pytest.mark.parametrize("side", ["lo", "hi"])
def test_micro_periodic_wrap_fixup_gpu(side):
    """C-12 on the GPU: the stored fp32 position after a periodic wrap is in [lo, hi);
    a wrap that rounds onto hi is stored as lo, exactly as the oracle pin fixes it."""
    mesh = M.MicroMesh(dims=(4, 4, 4), origin=(0.0, 0.0, 0.0), cell_size=(0.25,) * 3, bc=(0, 0, 0))
    props = M.MicroProps(gravity=(0.0, 0.0, 0.0), drag_law=M.DRAG_STOKES, rho_p=1e9)
    Tf = 283.15
    F = np.empty((5, 4, 4, 4), np.float32)
    F[:3], F[3], F[4] = 0.0, Tf, float(M.saturation_vapor_density(Tf))
    x0 = 1e-9 if side == "lo" else float(np.nextafter(np.float32(1.0), np.float32(0.0)))
    u0 = -1.0 if side == "lo" else 1.0
    x = np.array([[x0], [0.5], [0.5]], np.float32)
    u = np.array([[u0], [0.0], [0.0]], np.float32)
    d, T, w = np.array([2e-5], np.float32), np.array([Tf], np.float32), np.ones(1, np.float32)
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 2e-9, (1,))
    o = _oracle_run(mesh, props, F, x, u, d, T, w, 2e-9, (1,))
    assert 0.0 <= g[0][0, 0] < 1.0
    assert g[0][0, 0] == o[0][0, 0]
    if side == "lo":
        assert g[0][0, 0] == np.float32(0.0)


def test_micro_deposit_start_cell_gpu():
    """C-10 on the GPU: a droplet crossing a face deposits into its start cell only."""
    mesh = M.MicroMesh(dims=(4, 4, 4), origin=(0.0, 0.0, 0.0), cell_size=(0.25,) * 3, bc=(1, 1, 1))
    props = M.MicroProps(gravity=(0.0, 0.0, -9.81), drag_law=M.DRAG_STOKES)
    F = np.empty((5, 4, 4, 4), np.float32)
    F[:3], F[3], F[4] = 0.0, 290.0, 0.006
    x = np.array([[0.499], [0.6], [0.3]], np.float32)
    u = np.array([[2.0], [0.0], [0.0]], np.float32)
    d, T, w = np.array([4e-4], np.float32), np.array([285.0], np.float32), np.array([3.0], np.float32)
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 2e-3, (1,))
    o = _oracle_run(mesh, props, F, x, u, d, T, w, 2e-3, (1,))
    assert g[0][0, 0] > 0.5
    start = (1 * 4 + 2) * 4 + 1
    for k in (0, 2, 3, 4):
        assert np.flatnonzero(g[4][k]).tolist() == [start], k
    _compare(g, o, mesh, "start-cell")


# ---- fp32 arithmetic mode (reading C-36; bounds in tests/micro_bounds.py) -------------

def _stable(n, bc=(0, 0, 1), seed=11, binned=False):
    mesh, F, x, u, d, T, w = _setup(n, bc=bc, seed=seed, drop_kw={"d_range": (10e-6, 30e-6)})
    if binned:
        c = np.floor(x.astype(np.float64) / 0.125).astype(np.int64)
        o = np.lexsort((c[0], c[1], c[2]))
        x, u, d, T, w = x[:, o].copy(), u[:, o].copy(), d[o].copy(), T[o].copy(), w[o].copy()
    return mesh, F, x, u, d, T, w


@pytest.mark.parametrize("n,calls,bc,binned", [
    (20_000, (3, 2), (0, 0, 1), False),     # many tiles + ragged tail, two calls accumulate
    (8 * 24 * 20 * 12 + 77, (2, 3), (0, 0, 1), True),   # binned: long same-cell lane runs
    (257, (4,), (1, 1, 1), False),          # one full CTA + 1, all walls reflecting
    (1, (6,), (0, 0, 0), False),            # a single droplet, fully periodic
])
def test_micro_fp32_parity(n, calls, bc, binned):
    """The fp32 kernel against the fp32 oracle (same operations, both binary32; only the
    libm-vs-CUDA exp / pow / cbrt ulps differ) and against the fp64 oracle, each within
    the binary32 rounding bound of tests/micro_bounds.py.  dt = 1 ms, 10-30 um droplets:
    the explicit Eq. 7 / Eq. 12 updates are contractive (test_oracle_micro._stable_cloud)."""
    from tests.micro_bounds import check_fp32, run_with_gross
    mesh, F, x, u, d, T, w = _stable(n, bc=bc, binned=binned)
    props = M.MicroProps()
    dt, ns = 1e-3, sum(calls)
    g = _gpu_run(mesh, props, F, x, u, d, T, w, dt, calls, arithmetic="fp32")
    r32 = run_with_gross(mesh, props, x, u, d, T, w, F, dt, ns, arith=np.float32)
    r64 = run_with_gross(mesh, props, x, u, d, T, w, F, dt, ns)
    u_scale = float(np.max(np.abs(F[:3]))) + 9.81 * dt * ns
    check_fp32(g, r32[:6], r64[6], mesh, ns, u_scale, f"vs fp32 oracle n={n}")
    check_fp32(g, r64[:6], r64[6], mesh, ns, u_scale, f"vs fp64 oracle n={n}")
    assert g[5] == r32[5] == r64[5]


def test_micro_fp32_mass_floor_clamps_match():
    """C-32 in fp32 mode: the clamp decision is taken in binary32 on both sides."""
    mesh, F, x, u, d, T, w = _setup(3000, field_kw={"T0": 300.0, "rho_v0": 1e-4},
                                    drop_kw={"d_range": (0.5e-6, 3e-6)})
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 0.2, (1,), arithmetic="fp32")
    o = M.micro_advance(mesh, props, x, u, d, T, w, F, 0.2, 1, arith=np.float32)
    assert o[5] > 0 and g[5] == o[5]
    np.testing.assert_allclose(g[2], o[2], rtol=8 * 1.2e-7)


def test_micro_fp32_full_size_sampled():
    """2e7 droplets on the bench grid in fp32 mode: sampled droplet states against the
    fp32 oracle run on those droplets alone (droplets are independent given the frozen
    field); the vapour ledger of the whole field closes to the binary32 bound."""
    from tests.micro_bounds import C_ACC, EPS32, STATE_ULPS
    dims, h = (192, 192, 72), 1.0 / 32
    mesh = M.MicroMesh(dims=dims, origin=(0.0, 0.0, 0.0), cell_size=(h,) * 3, bc=(0, 0, 1))
    F = synth.micro_field(dims, mesh.origin, mesh.cell_size, seed=4)
    n = 20_000_000
    x, u, d, T, w = synth.droplets_np(n, (0.0, 0.0, 0.0), (6.0, 6.0, 2.25), seed=9, d_range=(10e-6, 30e-6))
    props = M.MicroProps()
    g = _gpu_run(mesh, props, F, x, u, d, T, w, 1e-3, (2,), arithmetic="fp32")
    idx = np.random.default_rng(0).choice(n, 2000, replace=False)
    o = M.micro_advance(mesh, props, x[:, idx], u[:, idx], d[idx], T[idx], w[idx], F, 1e-3, 2, arith=np.float32)
    tol = STATE_ULPS * 2 * EPS32
    assert np.max(np.abs(g[0][:, idx].astype(np.float64) - o[0])) <= tol * 6.0
    assert np.max(np.abs(g[2][idx] / o[2] - 1)) <= tol
    assert np.max(np.abs(g[3][idx] / o[3] - 1)) <= tol
    m0 = M.droplet_mass(d.astype(np.float64), props.rho_p)
    m1 = M.droplet_mass(g[2].astype(np.float64), props.rho_p)
    dM = np.sum(w * (m1 - m0))
    assert abs(g[4][3].sum() + dM) <= C_ACC * EPS32 * np.sum(w * (m0 + m1)) * 2
