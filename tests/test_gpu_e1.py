"""E1 (§3.1): the two-way coupled particle/box0d-fluid loop
through the GPU library and the GPU extrapolator-corrector, against the same loop on
the oracle, the momentum ledger, and the paper's qualitative claim."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import e1_study as E  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_e1_gpu_matches_oracle(scheme):
    g = E.run(scheme, 30, "gpu")
    o = E.run(scheme, 30, "oracle")
    # fp32 particle states, fp64 fluid: the two loops agree to fp32 rounding
    assert np.abs(g["e_f"] - o["e_f"]).max() < 1e-5
    assert np.abs(g["e_p"] - o["e_p"]).max() < 1e-5


@pytest.mark.parametrize("scheme", E.SCHEMES)
def test_e1_momentum_ledger(scheme):
    """What the particles lost is what the fluid received plus what is still in
    flight (sources not yet handed over, or estimated ahead of their truth)."""
    r = E.run(scheme, 30, "gpu")
    P0 = E.M_P * 1.0
    lost = P0 - r["Pp"]
    assert np.abs(lost - r["P_lagr_out"]).max() < 2e-5 * P0          # sources = particle momentum change
    assert np.abs(r["Pf"] - r["P_fluid_in"]).max() < 1e-12 * P0       # the fluid integrates what it is given


def test_e1_constant_extrapolator_beats_zero_early():
    """the constant extrapolator reduces the early error of the zero
    extrapolator (first step excluded: no source exists yet in any scheme)."""
    z = E.run("zero", 12, "gpu")
    c = E.run("constant", 12, "gpu")
    assert np.abs(c["e_f"][1:10]).max() < 0.5 * np.abs(z["e_f"][1:10]).max()


def test_e1_magnitudes_match_the_paper():
    """PAPER.md:270-276 at dt/tau = 0.01 (reading C-20): the conventional scheme's error is
    a few 1e-4 (paper: 0.04 %); the zero extrapolator's reaches ~1 % (paper: "up to the
    order of 1 %"); the constant extrapolator brings it back to the conventional level
    (paper: "the same level as the conventional method") — first step excluded, where
    no source exists yet in any asynchronous scheme."""
    n = 200
    conv = E.run("conventional", n, "gpu")
    zero = E.run("zero", n, "gpu")
    const = E.run("constant", n, "gpu")
    c = np.abs(conv["e_f"]).max()
    assert 1e-4 < c < 1.5e-3, c
    assert np.abs(zero["e_f"][1:]).max() > 5e-3
    assert np.abs(const["e_f"][1:]).max() < 1.5 * c
    assert np.abs(const["e_p"]).max() < 1.5 * np.abs(conv["e_p"]).max()
