"""Oracle of the extrapolator-corrector — TEST INFRASTRUCTURE ONLY.

Plain fp64 numpy, written from PAPER.md §2.4 "Extrapolator-corrector method"
(PAPER.md:216-242), step by step in the paper's notation.  Only tests/, smoke() and
bench.py's cpu_baseline may import it; the product path is the CUDA estimator
(`st_ec_*`, paper_2603_26691_b200/csrc/st_ec.cu), which shares no code with this file.

Per Eulerian step n (Eq. 14-15):

    ΔS^n_corr = S^{n-1} - S^{n-1}_est
    S^n_est   = ΔS^n_corr + S^n_ext

with a delay of more than one step: "the corrector is the sum of all
unincorporated sources from previous time steps minus the sum of the estimated sources
from these time steps".  Extrapolators (Eq. 16a-c):

    zero:     S^n_ext = 0
    constant: S^n_ext = S^{n-1}
    linear:   S^n_ext = 2 S^{n-1} - S^{n-2}

where S^{n-1}, S^{n-2} are the true sources of the last two *known* steps
(PAPER.md:238).  Readings (C-25..C-27):
  C-25  S^{n-1}_est in Eq. 14 is the estimate *of step n-1's source*, i.e. what step
        n-1 emitted beyond its own correction (its extrapolated part, including the
        rounding of the emitted value).  Subtracting the whole emitted value instead
        would count every correction twice; the paper's "conservative over time"
         holds only under this reading: Σ emitted − Σ received equals the
        estimates still awaiting their truth, exactly.
  C-26  history falls back linear → constant → zero while fewer truths are known;
  C-27  a variable step scales the extrapolated term by dt_ratio = dt^n / dt^{source}
        ("scaling the source terms with the time-step ratio").
"""
from __future__ import annotations

import collections

import numpy as np

MODES = ("zero", "constant", "linear")


class Estimator:
    """One estimator over a whole source-field array (any shape), fp64 state."""

    def __init__(self, mode: str, shape, emit_dtype=np.float64, max_backlog: int = 8):
        if mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}")
        self.mode = mode
        self.shape = tuple(shape)
        self.emit_dtype = emit_dtype
        self.max_backlog = max_backlog
        self.last_true = None            # S^{n-1}: latest known true source
        self.prev_true = None            # S^{n-2}
        self.pending = collections.deque()   # emitted estimates of steps whose truth is not known yet
        self.cum_true = np.zeros(self.shape)
        self.cum_est = np.zeros(self.shape)

    def extrapolate(self) -> np.ndarray:
        """S^n_ext from the known true sources (Eq. 16a-c)."""
        z = np.zeros(self.shape)
        if self.mode == "zero" or self.last_true is None:
            return z
        if self.mode == "constant" or self.prev_true is None:
            return self.last_true.copy()
        return 2.0 * self.last_true - self.prev_true

    def step(self, received=(), dt_ratio: float = 1.0) -> np.ndarray:
        """One Eulerian step: `received` = true sources newly available, oldest first
        (their steps are the oldest pending ones).  Returns S^n_est (emit precision)."""
        if not dt_ratio > 0:
            raise ValueError("dt_ratio must be > 0")
        if len(received) > len(self.pending):
            raise RuntimeError("protocol violation: true source for a step that was never estimated")
        corr = np.zeros(self.shape)
        for s in received:                                   # the multi-step corrector
            s = np.asarray(s, dtype=np.float64).reshape(self.shape)
            corr += s - self.pending.popleft()
            self.cum_true += s
            self.prev_true, self.last_true = self.last_true, s.copy()
        est = corr + dt_ratio * self.extrapolate()            # Eq. 15
        emitted = est.astype(self.emit_dtype)
        if len(self.pending) >= self.max_backlog:
            raise RuntimeError("backlog exceeds max_backlog")
        # C-25: the estimate of step n's own source = emitted minus the correction part
        self.pending.append(emitted.astype(np.float64) - corr)
        self.cum_est += emitted
        return emitted

    def ledger(self):
        """(Σ true received, Σ estimates emitted, Σ estimates still uncorrected)."""
        pend = np.zeros(self.shape)
        for p in self.pending:
            pend += p
        return self.cum_true.copy(), self.cum_est.copy(), pend
