"""GPU (CUDA, through the C-ABI) vs the fp32 oracle on the same seeded inputs.

Bars (BASELINE.json north_star):
  * integer work (cell, chunk, rebin order, migration counts) bit-exact given
    identical positions;
  * positions / velocities within 1e-5 after 100 steps (positions by the domain
    length, periodic-aware; velocities by the field's max speed);
  * per-cell source field within 1e-5 relative L2 for the same particle state.
"""
import math

import numpy as np
import pytest

import synth
from tests.conftest import gpu_available
from tests.helpers import by_id, gpu_config, oracle_sim, periodic_dist

pytestmark = pytest.mark.gpu

if not gpu_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2603_26691_b200 import ScaleTrack, StError  # noqa: E402

import oracle  # noqa: E402


def _setup(wl, rebin_interval=1, integrator=0, n=None, precision="f32"):
    n = wl.n_particles if n is None else n
    lo, hi = synth.domain_box(wl)
    x, u, d, w = synth.particles_np(n, lo, hi, wl.d_range, wl.d_dist, wl.w, wl.seed_particles)
    F = synth.make_field(wl)
    g = ScaleTrack(gpu_config(wl, capacity=n, rebin_interval=rebin_interval, integrator=integrator))
    o = oracle_sim(wl, precision, rebin_interval, integrator)
    g.inject(x, u, d, w)
    o.inject(x, u, d, w)
    g.set_fluid_field(F)
    o.set_fluid_field(F)
    return g, o, (x, u, d, w), F


# ------------------------------------------------------------------ integer contract
@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_locate_bit_exact(name):
    """C-6 / C-14: st_locate == oracle locate on identical fp32 positions, including
    faces, their fp32 neighbours and the upper boundary."""
    wl = synth.workload(name, n_particles=0)
    lo, hi = synth.domain_box(wl)
    x, _, _, _ = synth.particles_np(200_000, lo, hi, (1e-5, 2e-5), seed=5)
    faces = []
    for a in range(3):
        f = (np.float32(wl.origin[a]) + np.arange(wl.dims[a] + 1) * np.float32(wl.cell_size[a])).astype(np.float32)
        faces.append(np.concatenate([f, np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))]))
    m = max(len(f) for f in faces)
    xf = np.stack([np.resize(f, m) for f in faces]).astype(np.float32)
    xf = np.clip(xf, np.array(lo, np.float32)[:, None], np.array(hi, np.float32)[:, None])
    X = np.concatenate([x, xf], axis=1)
    g = ScaleTrack(gpu_config(wl, capacity=16))
    o = oracle_sim(wl)
    cg, kg = g.locate(X)
    co, ko = o.locate(X)
    assert np.array_equal(cg, co)
    assert np.array_equal(kg, ko)


def test_inject_order_and_rebin_bit_exact():
    """Injection keeps order; the first rebin equals the oracle's stable counting sort."""
    wl = synth.workload("C2", n_particles=300_000)
    g, o, (x, u, d, w), F = _setup(wl)
    p = g.get_particles()
    assert np.array_equal(p["x"], x) and np.array_equal(p["d"], d)
    assert np.array_equal(p["id"], np.arange(x.shape[1], dtype=np.uint64))
    g.advance(wl.dt, 1)
    o.advance(wl.dt, 1)
    pg = g.get_particles()
    # C-15 given the GPU's own positions: stable sort of the pre-rebin order (= id order here)
    gi = by_id(pg)
    perm, _ = oracle.stable_order(o.bin_key(gi["x"]), o.mesh.n_bins)
    assert np.array_equal(pg["id"], gi["id"][perm])
    assert np.all(np.diff(pg["chunk"]) >= 0)
    assert np.all(np.diff(o.bin_key(pg["x"])) >= 0)


def _check_rebin_given_gpu_positions(o, before, after):
    pos = {int(i): k for k, i in enumerate(after["id"])}
    idx = np.array([pos[int(i)] for i in before["id"]])
    X = after["x"][:, idx]        # post-step positions in pre-rebin order
    perm, _ = oracle.stable_order(o.bin_key(X), o.mesh.n_bins)
    assert np.array_equal(after["id"], before["id"][perm])
    c2, k2 = o.locate(after["x"])
    assert np.array_equal(after["cell"], c2) and np.array_equal(after["chunk"], k2)


@pytest.mark.parametrize("K", [1, 2, 3])
def test_rebin_order_given_gpu_positions(K):
    """After many steps at rebin interval K (fused neighbour scatter): feed the GPU's
    pre-rebin order and post-step positions to the oracle's bin key + stable sort;
    the GPU's own order must come out (C-15)."""
    wl = synth.workload("C2", n_particles=200_000)
    g, o, _, F = _setup(wl, rebin_interval=K)
    for _ in range(3 * K + K - 1):
        g.advance(wl.dt, 1)      # the last call leaves no rebin due
    before = g.get_particles()
    g.advance(wl.dt, 1)          # this call ends with a rebin
    after = g.get_particles()    # observing flushes it (standalone scatter)
    _check_rebin_given_gpu_positions(o, before, after)
    st = g.stats()
    assert st["rebins"] >= 4


def test_fused_rebin_then_observe():
    """K = 1: rebins fused into the next advance; observe after several calls."""
    wl = synth.workload("C3", n_particles=300_000)
    wl.dims, wl.cell_size = (64, 64, 64), (1 / 16,) * 3
    g, o, _, F = _setup(wl, rebin_interval=1)
    g.advance(wl.dt, 1)
    g.advance(wl.dt, 1)
    before = g.get_particles()
    for _ in range(5):
        g.advance(wl.dt, 1)
    mid = g.stats()
    assert mid["fused_rebins"] >= 4, mid
    before = g.get_particles()
    g.advance(wl.dt, 1)
    after = g.get_particles()
    _check_rebin_given_gpu_positions(o, before, after)


def _check_rebin_c15b(o, P0, after):
    """C-15 / C-15b, bit-exact: P0 is the layout of the previous rebin (home bin of every
    particle = the bin of its P0 position), `after` the layout of this one.  The oracle's
    rule — stable sort of P0's order by (bin key, far) — must give exactly `after`."""
    pos = {int(i): k for k, i in enumerate(P0["id"])}
    idx = np.array([pos[int(i)] for i in after["id"]])
    X = np.ascontiguousarray(after["x"][:, np.argsort(idx)])
    far = o.far_mask(o.bin_key(P0["x"]), X)
    perm, _ = oracle.stable_order(2 * o.bin_key(X) + far.astype(np.int64), 2 * o.mesh.n_bins)
    assert np.array_equal(after["id"], P0["id"][perm])
    return int(far.sum())


def test_far_movers_placed_in_bin_tails():
    """Particles moving more than one cell between rebins (K = 8, fast flow) stay on the
    fused neighbour-slot path: placed at the tail of their destination bin in prior
    store order (C-15b, bit-exact against the oracle's rule) — no general sort."""
    wl = synth.workload("C2", n_particles=100_000)
    g, o, _, F = _setup(wl, rebin_interval=8)
    F2 = (F * 20.0).astype(np.float32)        # up to 20 m/s: several cells per 8 calls
    g.set_fluid_field(F2)
    for _ in range(8):
        g.advance(wl.dt, 1)                    # call 8 leaves a rebin due
    P8 = g.get_particles()                     # flushed: every particle in its cell's bin
    gen0 = g.stats()["general_rebins"]
    for _ in range(8):
        g.advance(wl.dt, 1)                    # call 16 leaves the next one due
    after = g.get_particles()
    st = g.stats()
    nfar = _check_rebin_c15b(o, P8, after)
    assert nfar > 100 and st["last_far"] == nfar, (nfar, st["last_far"])
    assert st["general_rebins"] == gen0


def test_far_tails_long_dense_bins():
    """C-15b with long far tails (k_far_order_w / k_far_order_b): two dense cells of
    particles (3000 and 12000) move 2.5 cells between rebins in a uniform flow, so their
    destination bins collect ~1500 (CTA sort in shared memory) and ~6000 (beyond it)
    far particles, over a random background.  Order bit-exact against the oracle's rule."""
    wl = synth.workload("C2", n_particles=35_000)
    wl.dims, wl.cell_size = (16, 16, 16), (1 / 16,) * 3
    h, K = 1 / 16, 2
    V = 1.25 * h / wl.dt                      # 1.25 cells per call, 2.5 per rebin interval
    rng = np.random.default_rng(11)
    parts = []
    for n_c, cell in ((3000, (2, 5, 5)), (12000, (3, 9, 9))):
        parts.append((np.asarray(cell, np.float64)[:, None] + rng.random((3, n_c))) * h)
    parts.append(rng.random((3, 20000)) * 1.0)
    x = np.minimum(np.concatenate(parts, axis=1), np.nextafter(1.0, 0.0)).astype(np.float32)
    n = x.shape[1]
    u = np.zeros((3, n), np.float32)
    u[0] = V
    d = np.full(n, 20e-6, np.float32)
    w = np.ones(n, np.float32)
    F = np.zeros((3, 16, 16, 16), np.float32)
    F[0] = V
    g = ScaleTrack(gpu_config(wl, capacity=n, rebin_interval=K))
    o = oracle_sim(wl, "f32", K)
    g.inject(x, u, d, w)
    g.set_fluid_field(F)
    for _ in range(K):
        g.advance(wl.dt, 1)
    P0 = g.get_particles()                     # flushed: home bins of the next rebin
    for _ in range(K):
        g.advance(wl.dt, 1)
    after = g.get_particles()
    nfar = _check_rebin_c15b(o, P0, after)
    assert nfar == n and g.stats()["last_far"] == n, (nfar, g.stats()["last_far"])
    _, cnt = np.unique(o.bin_key(after["x"]), return_counts=True)
    assert cnt.max() > 4096, cnt.max()        # the longest tail is beyond the shared-memory sort
    g.close()


# ------------------------------------------------------------------ closed form through the GPU
@pytest.mark.parametrize("drag", [0, 1])
def test_c1_settling_terminal_velocity(drag):
    """C1 (BJ configs[0]): 1000 particles, uniform flow, gravity, 1000 steps; GPU fp32
    matches the closed-form terminal velocity u_f + g tau (Stokes) / the oracle (S-N)."""
    wl = synth.workload("C1")
    wl.drag_law = drag
    g, o, (x, u, d, w), F = _setup(wl)
    for _ in range(wl.steps):
        g.advance(wl.dt, 1)
    p = by_id(g.get_particles())
    if drag == 0:
        tau = synth.RHO_P * d.astype(np.float64) ** 2 / (18 * synth.RHO_F * synth.NU_F)
        uz = -9.81 * tau
        assert np.max(np.abs(p["u"][2] - uz)) / np.max(np.abs(uz)) < 1e-5
        assert np.max(np.abs(p["u"][0] - 0.05)) < 1e-6
    else:
        for _ in range(wl.steps):
            o.advance(wl.dt, 1)
        q = by_id(o.particles())
        assert np.max(np.abs(p["u"] - q["u"])) / 0.05 < 1e-5
        assert np.max(periodic_dist(p["x"], q["x"], wl.lengths)) < 1e-5


# ------------------------------------------------------------------ free-running float parity
def test_c2_taylor_green_100_steps():
    """C2 (BJ configs[1]) at full size: 1e6 particles, TG, one-way, periodic, 100 steps."""
    wl = synth.workload("C2")
    g, o, _, F = _setup(wl)
    for _ in range(wl.steps):
        g.advance(wl.dt, 1)
        o.advance(wl.dt, 1)
    pg, po = g.get_particles(), o.particles()
    a, b = by_id(pg), by_id(po)
    pos = np.max(periodic_dist(a["x"], b["x"], wl.lengths) / np.array(wl.lengths)[:, None])
    vel = np.max(np.abs(a["u"] - b["u"])) / 1.0   # U_max = U0 = 1 m/s
    assert pos <= 1e-5, pos
    assert vel <= 1e-5, vel


@pytest.mark.parametrize("integrator", [0, 1])
def test_two_way_fourier_100_steps(integrator):
    """Two-way, random-Fourier field, reflecting walls (C4 shape, reduced), 100 steps in
    10-step segments: at each segment start the oracle is restarted from the GPU state
    (reading C-24: in a 256-mode field the trajectories are chaotic — nearby fp32
    trajectories separate by ~e^{lambda t}, so any two correct fp32 programs differ by
    more than 1e-5 after 0.5 s; the segment form checks the step, not the chaos)."""
    wl = synth.workload("C4", n_particles=100_000)
    wl.dims = (32, 32, 96)
    wl.cell_size = (3 / 32,) * 3
    g, _, _, F = _setup(wl, integrator=integrator)
    U = float(np.max(np.linalg.norm(F.reshape(3, -1), axis=0)))
    worst_p = worst_v = 0.0
    for seg in range(10):
        st = g.get_particles()
        o = oracle_sim(wl, integrator=integrator)
        o.inject(st["x"], st["u"], st["d"], st["w"], st["id"])
        o.set_fluid_field(F)
        for s in range(10):
            g.advance(wl.dt, 1)
            o.advance(wl.dt, 1)
        a, b = by_id(g.get_particles()), by_id(o.particles())
        worst_p = max(worst_p, np.max(np.abs(a["x"].astype(np.float64) - b["x"]) / np.array(wl.lengths)[:, None]))
        worst_v = max(worst_v, np.max(np.abs(a["u"].astype(np.float64) - b["u"])) / U)
    assert worst_p <= 1e-5, worst_p
    assert worst_v <= 1e-5, worst_v


# ------------------------------------------------------------------ sources
def _inject_state(sim_g, sim_o, p):
    sim_g.inject(p["x"], p["u"], p["d"], p["w"], p["id"])
    sim_o.inject(p["x"], p["u"], p["d"], p["w"], p["id"])


@pytest.mark.parametrize("name,n,steps", [("C3", 400_000, 3), ("C4", 300_000, 2)])
def test_sources_same_state(name, n, steps):
    """Per-cell source field (C-8..C-10, C-13) within 1e-5 relative L2 for the same
    particle state (drive both with the same field, compare the step)."""
    wl = synth.workload(name, n_particles=n)
    if name == "C3":
        wl.dims, wl.cell_size = (64, 64, 64), (1 / 16,) * 3
    g, o, _, F = _setup(wl)
    g.advance(wl.dt, steps)
    o.advance(wl.dt, steps)
    Sg, Tg = g.get_sources()
    So, To = o.get_sources()
    assert Tg == pytest.approx(To, rel=1e-15)
    err = np.linalg.norm(Sg.astype(np.float64) - So) / np.linalg.norm(So)
    assert err <= 1e-5, err


def test_sources_after_100_steps_from_gpu_state():
    """After 100 free GPU steps (two-way, C3 shape reduced), hand the GPU's particle
    state to the oracle and compare one more step's source field and momentum balance."""
    wl = synth.workload("C3", n_particles=200_000)
    wl.dims, wl.cell_size = (64, 64, 64), (1 / 16,) * 3
    g, _, _, F = _setup(wl)
    for _ in range(100):
        g.advance(wl.dt, 1)
    g.get_sources()
    state = g.get_particles()
    o = oracle_sim(wl)
    o.inject(state["x"], state["u"], state["d"], state["w"], state["id"])
    o.set_fluid_field(F)
    g.advance(wl.dt, 1)
    o.advance(wl.dt, 1)
    Sg, Tg = g.get_sources()
    So, To = o.get_sources()
    err = np.linalg.norm(Sg.astype(np.float64) - So) / np.linalg.norm(So)
    assert err <= 1e-5, err


def test_momentum_conservation_gpu():
    """P-4 on the GPU path (fp32, g = 0, periodic): sum w m du + sum S V T = 0 to fp32
    accuracy relative to sum |w m du| (fp32 bound)."""
    wl = synth.workload("C3", n_particles=100_000)
    wl.dims, wl.cell_size, wl.gravity = (32, 32, 32), (1 / 8,) * 3, (0.0, 0.0, 0.0)
    g, _, (x, u0, d, w), F = _setup(wl)
    g.advance(wl.dt, 1)
    p = by_id(g.get_particles())
    S, T = g.get_sources()
    m = math.pi / 6 * synth.RHO_P * d.astype(np.float64) ** 3
    dP = np.sum(w * m * (p["u"].astype(np.float64) - u0), axis=1)
    fluid = S.reshape(3, -1).astype(np.float64).sum(axis=1) * np.prod(wl.cell_size) * T
    scale = np.sum(np.abs(w * m * (p["u"] - u0)))
    assert np.max(np.abs(dP + fluid)) / scale < 1e-4


# ------------------------------------------------------------------ edge cases
def test_empty_store_and_errors():
    wl = synth.workload("C1", n_particles=0)
    g = ScaleTrack(gpu_config(wl, capacity=10))
    with pytest.raises(StError):
        g.advance(1e-3, 1)                      # no field yet (ST_ERR_STATE)
    g.set_fluid_field(synth.make_field(wl))
    g.advance(1e-3, 1)                          # empty store
    S, T = g.get_sources()
    assert T == pytest.approx(1e-3) and not np.any(S)
    with pytest.raises(StError) as e:           # outside the domain
        g.inject(np.full((3, 1), 2.0, np.float32), np.zeros((3, 1), np.float32), np.full(1, 1e-5, np.float32))
    assert "OUT_OF_DOMAIN" in str(e.value)
    assert g.count() == 0
    with pytest.raises(StError) as e:           # capacity
        z = np.zeros((3, 11), np.float32) + 0.5
        g.inject(z, np.zeros((3, 11), np.float32), np.full(11, 1e-5, np.float32))
    assert "CAPACITY" in str(e.value)


def test_cfl_error_is_loud():
    """S:174 never silent: a displacement one wrap cannot undo -> ST_ERR_CFL."""
    wl = synth.workload("C1", n_particles=1)
    g = ScaleTrack(gpu_config(wl, capacity=4))
    g.inject(np.full((3, 1), 0.5, np.float32), np.array([[500.0], [0], [0]], np.float32),
             np.full(1, 1e-3, np.float32))
    g.set_fluid_field(synth.uniform_field(wl.dims, (500.0, 0, 0)))
    g.advance(0.01, 1)
    with pytest.raises(StError) as e:
        g.sync()
    assert "CFL" in str(e.value)


def test_ragged_chunks_and_multi_substeps():
    """Dims not divisible by the chunk edge (ragged last chunk) and nsteps > 1 per call."""
    wl = synth.workload("C4", n_particles=50_000)
    wl.dims, wl.cell_size = (20, 13, 37), (3 / 20, 3 / 13, 9 / 37)
    g, o, _, F = _setup(wl)
    for _ in range(10):
        g.advance(wl.dt / 4, 4)
        o.advance(wl.dt / 4, 4)
    a, b = by_id(g.get_particles()), by_id(o.particles())
    U = float(np.max(np.abs(F)))
    assert np.max(np.abs(a["x"].astype(np.float64) - b["x"]) / np.array(wl.lengths)[:, None]) <= 1e-5
    assert np.max(np.abs(a["u"].astype(np.float64) - b["u"])) / U <= 1e-5
    pg = g.get_particles()
    c, k = o.locate(pg["x"])
    assert np.array_equal(pg["cell"], c) and np.array_equal(pg["chunk"], k)
    assert np.all(np.diff(pg["chunk"]) >= 0)
    assert np.all(np.diff(o.bin_key(pg["x"])) >= 0)


def test_async_split_readout_and_device_buffers():
    """Asynchronous coupling buffer: request/wait readout while the next advance is
    enqueued; device (torch) field and source buffers; intervals add up."""
    import torch
    wl = synth.workload("C3", n_particles=100_000)
    wl.dims, wl.cell_size = (32, 32, 32), (1 / 8,) * 3
    g, o, _, F = _setup(wl)
    Fd = torch.from_numpy(F).cuda()
    Sd = torch.empty((3, 32, 32, 32), dtype=torch.float32, device="cuda")
    g.advance(wl.dt, 1)
    o.advance(wl.dt, 1)
    g.request_sources()
    g.set_fluid_field(Fd)
    g.advance(wl.dt, 1)                 # deposits into the other buffer while the readout runs
    S1, T1 = g.wait_sources(Sd)
    So, To = o.get_sources()
    assert T1 == pytest.approx(wl.dt)
    err = np.linalg.norm(Sd.cpu().numpy().astype(np.float64) - So) / np.linalg.norm(So)
    assert err <= 1e-5
    S2, T2 = g.get_sources()
    assert T2 == pytest.approx(wl.dt) and np.any(S2)


@pytest.mark.parametrize("K", [2, 3])
def test_counted_rebin_survives_inject_and_observation(K):
    """K >= 2: the in-place step of the call that makes a rebin due counts the slots
    itself.  An injection or an observation between that step and the rebin must
    consume or discard those counts correctly: the physics (vs the oracle, 1e-5) and
    the contract order (C-15) stay exact, and no general sort is taken beyond the
    ones injections force."""
    wl = synth.workload("C2", n_particles=60_000)
    lo, hi = synth.domain_box(wl)
    x, u, d, w = synth.particles_np(wl.n_particles, lo, hi, wl.d_range, wl.d_dist, wl.w, wl.seed_particles)
    F = synth.make_field(wl)
    g = ScaleTrack(gpu_config(wl, capacity=wl.n_particles + 5_000, rebin_interval=K))
    o = oracle_sim(wl, "f32", K, 0)
    for s in (g, o):
        s.inject(x, u, d, w)
        s.set_fluid_field(F)
    x2, u2, d2, w2 = synth.particles_np(5_000, lo, hi, wl.d_range, wl.d_dist, wl.w, 77)
    for c in range(1, 4 * K + 1):
        g.advance(wl.dt, 1)
        o.advance(wl.dt, 1)
        if c == K:                                  # counts ready, rebin due: inject in between
            ids = np.arange(10**6, 10**6 + 5_000, dtype=np.uint64)
            g.inject(x2, u2, d2, w2, ids)
            o.inject(x2, u2, d2, w2, ids)
        if c == 2 * K + K:                          # counts ready, rebin due: observe in between
            before = g.get_particles()
    after = g.get_particles()
    a, b = by_id(after), by_id(o.particles())
    assert np.array_equal(a["id"], b["id"])
    assert np.max(periodic_dist(a["x"], b["x"], wl.lengths)) < 1e-5
    assert np.max(np.abs(a["u"].astype(np.float64) - b["u"])) < 1e-5
    assert np.all(np.diff(o.bin_key(after["x"])) >= 0)
    c2, k2 = o.locate(after["x"])
    assert np.array_equal(after["cell"], c2)


@pytest.mark.parametrize("integrator", [0, 1])
def test_two_way_walls_100_steps_free_running_smooth_field(integrator):
    """The literal north-star bar without restarts: two-way, reflecting walls on every
    axis, 100 free-running steps, x within 1e-5 of L and u within 1e-5 of U_max, in a
    SMOOTH random-Fourier field (|m| <= 2: trajectories do not separate exponentially
    as in the 256-mode field of reading C-24).  A wall makes u discontinuous in x
    (C-11): exact sign flips of one axis are allowed for particles near that wall, for
    at most 1e-4 of the particles; the positions, continuous there, are not exempted."""
    wl = synth.workload("C4", n_particles=100_000)
    wl.dims, wl.cell_size = (32, 32, 96), (3 / 32,) * 3
    wl.field_args = {"u_rms": 0.3, "modes": 32, "kmax": 2}
    g, o, _, F = _setup(wl, integrator=integrator)
    for _ in range(100):
        g.advance(wl.dt, 1)
        o.advance(wl.dt, 1)
    a, b = by_id(g.get_particles()), by_id(o.particles())
    assert np.array_equal(a["id"], b["id"])
    L = np.array(wl.lengths)[:, None]
    U = float(np.max(np.linalg.norm(F.reshape(3, -1), axis=0)))
    pos = float(np.max(np.abs(a["x"].astype(np.float64) - b["x"]) / L))
    ua, ub = a["u"].astype(np.float64), b["u"].astype(np.float64)
    du = np.abs(ua - ub) / U
    near = np.minimum(b["x"], L - b["x"]) < 100 * 1.5 * U * wl.dt
    flip = (du > 1e-5) & near & (np.abs(ua + ub) / U <= 1e-5)
    assert int(flip.sum()) <= max(1, int(1e-4 * ua.shape[1])), int(flip.sum())
    vel = float(np.max(np.where(flip, 0.0, du)))
    assert pos <= 1e-5, pos
    assert vel <= 1e-5, vel
