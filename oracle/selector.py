"""CPU oracle for the token Selector s_{psi,tau} of arXiv 2302.06218 (NEXT-4).

TEST INFRASTRUCTURE ONLY.  Only ``tests/`` and ``bench.py``'s cpu_baseline /
reference legs may import this module.  It shares no code with
``paper_2302_06218_b200`` and never imports it.

What it computes (§10.2):
  P:617      the Selector filters tokens *before* attention is computed;
  P:630-634  Eq. ``selector``  s_{psi,tau}: X_{L x D} -> X'_{L' x D}, tau the
             pruning threshold, L >> L';
  P:622      processed tokens are "reordered and aggregated" afterwards, so the
             selector also returns the kept indices (the re-aggregation map).
The paper never defines the scoring function (reading R18); as in
SPEC S:515-530 the untrained scorers are
  l2:   score_t = ||x_t||_2
  proj: score_t = |x_t . psi|
keep every token with score_t >= tau, in original order; if none passes, keep
the single highest-scoring token (ties: the smallest index) so L' >= 1
(reading R19).  Scores are fp64 on the exact input values (reading R20).
"""
from __future__ import annotations

import numpy as np


def scores(x, scorer: str = "l2", psi=None) -> np.ndarray:
    """fp64 score of every row of x [L, width]: ||x_t||_2 or |x_t . psi|."""
    x = np.asarray(x, dtype=np.float64)
    if scorer == "l2":
        return np.sqrt(np.einsum("ij,ij->i", x, x))
    if scorer == "proj":
        return np.abs(x @ np.asarray(psi, dtype=np.float64).reshape(-1))
    raise ValueError(f"unknown scorer {scorer!r}")


def select(x, tau: float, scorer: str = "l2", psi=None):
    """s_{psi,tau}(X): returns (X' [L', width] (same dtype as x), kept indices
    [L'] int64 increasing, scores [L] fp64)."""
    x = np.asarray(x)
    s = scores(x, scorer, psi)
    kept = np.flatnonzero(s >= tau)
    if kept.size == 0 and s.size:
        kept = np.array([int(np.argmax(s))], dtype=np.int64)  # first maximum
    return x[kept], kept.astype(np.int64), s


def scatter_rows(y_sel, kept, y_full):
    """Re-aggregation: the processed kept rows go back to their
    original positions; the other rows of y_full are left as they are."""
    y = np.array(y_full, copy=True)
    y[np.asarray(kept, dtype=np.int64)] = y_sel
    return y
