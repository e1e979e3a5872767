"""GPU extrapolator-corrector (st_ec_*, csrc/st_ec.cu) against the oracle
(oracle/extrapolator.py): bit-exact emitted fp32 estimates and fp64 ledgers on random
arrival schedules (§2.4, Eq. 14-16)."""
import numpy as np
import pytest

from oracle.extrapolator import Estimator

pytestmark = pytest.mark.gpu


def _run(mode, n, steps, seed, device_io=False, dt_var=False):
    import torch
    from paper_2603_26691_b200 import Extrapolator

    rng = np.random.default_rng(seed)
    ref = Estimator(mode, (n,), emit_dtype=np.float32, max_backlog=8)
    gpu = Extrapolator(mode, n, max_backlog=8)
    truths, delivered = [], 0
    for step in range(steps):
        k = int(rng.integers(0, 3))
        k = min(k, step - delivered)
        if step - delivered >= 7:
            k = step - delivered
        rec = np.stack(truths[delivered:delivered + k]) if k else None
        r = float(rng.uniform(0.5, 2.0)) if dt_var else 1.0
        want = ref.step(list(rec) if k else [], dt_ratio=r)
        if device_io:
            out = torch.empty(n, dtype=torch.float32, device="cuda")
            got = gpu.step(torch.from_numpy(rec).cuda() if k else None, dt_ratio=r, out=out).cpu().numpy()
        else:
            got = gpu.step(rec, dt_ratio=r)
        assert np.array_equal(got, want), (mode, step, np.abs(got - want).max())
        delivered += k
        truths.append(rng.normal(1.0, 0.5, n).astype(np.float32))
        assert gpu.backlog() == len(ref.pending)
    ct, ce, pe, tot = gpu.ledger()
    rct, rce, rpe = ref.ledger()
    assert np.array_equal(ct, rct) and np.array_equal(ce, rce)
    assert np.allclose(pe, rpe, rtol=0, atol=1e-12)
    assert np.allclose(tot, [rct.sum(), rce.sum(), rpe.sum()], rtol=1e-12, atol=1e-9)
    # conservation (C-25): emitted - received = pending, per value
    assert np.abs((ce - ct) - pe).max() <= 1e-12 * max(1.0, np.abs(ct).max())


@pytest.mark.parametrize("mode", ["zero", "constant", "linear"])
def test_ec_parity_random_delays(mode):
    _run(mode, n=3 * 4096 + 17, steps=60, seed=11)


def test_ec_parity_device_pointers_variable_dt():
    _run("linear", n=3 * 32768, steps=40, seed=5, device_io=True, dt_var=True)


def test_ec_errors():
    from paper_2603_26691_b200 import Extrapolator, StError

    e = Extrapolator("constant", 10, max_backlog=2)
    with pytest.raises(StError, match="ST_ERR_STATE"):          # truth for a step never estimated
        e.step(np.ones((1, 10), np.float32))
    e.step()
    e.step()
    with pytest.raises(StError, match="ST_ERR_STATE"):          # backlog would exceed 2
        e.step()
    with pytest.raises(StError, match="ST_ERR_INVALID_ARG"):
        e.step(dt_ratio=0.0)
    got = e.step(np.full((2, 10), 3.0, np.float32))              # catch up both
    assert np.all(got == 2 * 3.0 + 3.0)                          # corrections 3 + 3, ext 3
