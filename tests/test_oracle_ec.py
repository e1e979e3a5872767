"""Pins of the extrapolator-corrector oracle (oracle/extrapolator.py) against what the
paper and the algebra of its equations fix (§2.4, Eq. 14-16; SPEC.md
extrapolator-corrector examples).  CPU only."""
import numpy as np
import pytest

from oracle.extrapolator import Estimator


def test_eq15_constant_example():
    """SPEC example: constant mode, previous estimate 4, arriving true 5 -> 5 - 4 + 5 = 6."""
    e = Estimator("constant", (1,))
    e.pending.append(np.array([4.0]))
    assert e.step([np.array([5.0])])[0] == 6.0


def test_eq16_extrapolators():
    """Eq. 16a-c: zero -> 0; constant -> S^{n-1}; linear 2*5 - 3 = 7; linear falls back to
    constant with one known step and to zero with none."""
    for mode, want in (("zero", 0.0), ("constant", 5.0), ("linear", 7.0)):
        e = Estimator(mode, (2,))
        e.last_true, e.prev_true = np.full(2, 5.0), np.full(2, 3.0)
        assert np.all(e.extrapolate() == want)
    e = Estimator("linear", (2,))
    assert np.all(e.extrapolate() == 0.0)
    e.last_true = np.full(2, 5.0)
    assert np.all(e.extrapolate() == 5.0)


def test_zero_mode_three_step_delay():
    """SPEC example: zero mode, 3-step delay at constant s: 0, 0, 0, then 3s on catch-up
    (the multi-step corrector rule)."""
    s = 2.5
    e = Estimator("zero", (3,))
    out = [e.step()[0] for _ in range(3)]
    out.append(e.step([np.full(3, s)] * 3)[0])
    assert out == [0.0, 0.0, 0.0, 3 * s]


def test_dt_ratio_scales_extrapolation_only():
    """Variable step: S_est = corr + (dt^n/dt^src) S_ext."""
    e = Estimator("constant", (1,))
    e.pending.append(np.array([1.0]))
    got = e.step([np.array([3.0])], dt_ratio=0.5)[0]
    assert got == (3.0 - 1.0) + 0.5 * 3.0


@pytest.mark.parametrize("mode", ["zero", "constant", "linear"])
def test_conservativity_random_delays(mode):
    """PAPER.md:228 'conservative over time': for any arrival pattern, after every step
    the emitted estimates minus the received truths equal the estimates not yet
    corrected (1e-12 relative), i.e. nothing is lost or created."""
    rng = np.random.default_rng(7)
    shape = (3, 50)
    e = Estimator(mode, shape, emit_dtype=np.float32)
    truths, delivered = [], 0
    for n in range(300):
        k = int(rng.integers(0, 3))
        k = min(k, n - delivered)                     # truth of step m is known from step m+1 on
        if n - delivered >= 6:                        # bounded backlog
            k = n - delivered
        e.step([truths[delivered + i] for i in range(k)])
        delivered += k
        truths.append(rng.normal(1.0, 0.3, shape))    # the GPU produces step n's truth
        ct, ce, pend = e.ledger()
        assert np.abs((ce - ct) - pend).sum() <= 1e-12 * max(1.0, np.abs(ct).sum())
    assert delivered > 250


def test_zero_mode_full_catch_up_is_exact():
    e = Estimator("zero", (4,), emit_dtype=np.float32)
    rng = np.random.default_rng(3)
    ts = [rng.normal(size=4) for _ in range(6)]
    for _ in range(6):
        e.step()
    e.step(ts)                          # all six truths at once
    ct, ce, pend = e.ledger()
    # zero mode extrapolates nothing: after full catch-up the sums differ only by the
    # rounding of the last emitted (fp32) value, which stays pending for correction
    assert np.allclose(ce - ct, pend, rtol=0, atol=1e-15)
    assert np.all(np.abs(pend) <= 2.0 ** -23 * np.abs(ce))


def test_steady_state_and_ramp_exactness():
    """One-step delay (the truth of step n-1 arrives at step n): constant mode on a
    constant source is exact from step 3 on (step 2 catches up step 1), linear mode on a
    linear ramp from step 4 on (its extrapolation needs two known truths, and the step
    after the first exact extrapolation carries no correction) — SPEC's steady-state
    and ramp properties, which hold under reading C-25."""
    for mode, truth, k0 in (("constant", lambda n: 3.0, 3), ("linear", lambda n: 1.0 + 0.5 * n, 4)):
        e = Estimator(mode, (1,))
        for n in range(1, 15):
            rec = [np.array([truth(n - 1)])] if n > 1 else []
            got = e.step(rec)[0]
            if n >= k0:
                assert got == pytest.approx(truth(n), abs=1e-12), (mode, n)
    # the literal alternative (subtracting the whole emitted estimate) would oscillate:
    # constant source s, est = 0, 2s, 0, 2s, ...  -> here est = 0, 2s, s, s, ...
    e = Estimator("constant", (1,))
    seq = [e.step([np.array([3.0])] if n > 1 else [])[0] for n in range(1, 6)]
    assert seq == [0.0, 6.0, 3.0, 3.0, 3.0]


def test_protocol_violation():
    e = Estimator("constant", (1,))
    with pytest.raises(RuntimeError):
        e.step([np.array([1.0])])
