"""Pins of the Selector oracle (oracle/selector.py) against what the paper and
SPEC fix, independent of the oracle's own formulas (NEXT-4; R18-R21).

* SPEC S:527-530 worked examples: tau = -inf keeps everything; tau = +inf
  keeps exactly the argmax; row norms [3, 1, 2] with tau = 1.5 keep {0, 2}.
* Pythagorean rows with integer norms (3-4-5, 5-12-13, ...) give exact scores.
* Invariants S:533-536: monotone in tau, order preserving, idempotent.
* Projection scorer against a hand-computed dot product; scatter round trip.
"""
import math

import numpy as np
import pytest

from oracle import selector as sel
from synth import inputs


def test_spec_examples():
    x = np.array([[3.0, 0.0], [0.0, 1.0], [0.0, 2.0]])  # row norms 3, 1, 2
    xs, kept, _ = sel.select(x, 1.5)
    assert kept.tolist() == [0, 2]
    np.testing.assert_array_equal(xs, x[[0, 2]])
    xs, kept, _ = sel.select(x, -math.inf)
    assert kept.tolist() == [0, 1, 2]
    np.testing.assert_array_equal(xs, x)
    xs, kept, _ = sel.select(x, math.inf)  # S:529 never-empty rule: argmax only
    assert kept.tolist() == [0]


def test_pythagorean_rows_exact_scores():
    # rows with integer norms: (3,4)->5, (5,12)->13, (8,15)->17, (7,24)->25, (20,21)->29
    pairs = [(3, 4, 5), (5, 12, 13), (8, 15, 17), (7, 24, 25), (20, 21, 29)]
    x = np.zeros((5, 8))
    for i, (a, b, _) in enumerate(pairs):
        x[i, 2 * i % 8], x[i, (2 * i + 3) % 8] = a, -b
    s = sel.scores(x)
    assert s.tolist() == [float(c) for _, _, c in pairs]
    # threshold exactly at a score keeps that row (>=)
    assert sel.select(x, 17.0)[1].tolist() == [2, 3, 4]
    assert sel.select(x, 17.0 + 1e-12)[1].tolist() == [3, 4]


def test_ties_keep_first_maximum():
    x = np.array([[1.0, 0.0], [0.0, 2.0], [2.0, 0.0], [0.0, -2.0]])
    assert sel.select(x, 100.0)[1].tolist() == [1]


def test_projection_scorer_hand_example():
    x = np.array([[1.0, 2.0, 3.0], [-4.0, 0.5, 0.0], [0.0, 0.0, 0.0]])
    psi = np.array([0.5, -1.0, 2.0])
    # x.psi = 0.5-2+6 = 4.5 ; -2-0.5+0 = -2.5 ; 0
    assert sel.scores(x, "proj", psi).tolist() == [4.5, 2.5, 0.0]
    assert sel.select(x, 2.5, "proj", psi)[1].tolist() == [0, 1]


def test_invariants_on_random_rows():
    x = inputs.normal((1000, 64), seed=11, tensor_id=30)
    s = sel.scores(x)
    prev = None
    for tau in np.quantile(s, [0.0, 0.1, 0.5, 0.9, 0.999]):
        _, kept, _ = sel.select(x, tau)
        assert np.all(np.diff(kept) > 0)  # order preserved
        if prev is not None:
            assert kept.size <= prev  # monotone in tau
        prev = kept.size
        xs, kept2, _ = sel.select(sel.select(x, tau)[0], tau)  # idempotent
        assert kept2.size == kept.size
    # brute force: the kept set is exactly {t : ||x_t|| >= tau}
    tau = float(np.median(s))
    brute = [t for t in range(x.shape[0]) if math.sqrt(sum(float(v) ** 2 for v in x[t])) >= tau]
    assert sel.select(x, tau)[1].tolist() == brute


def test_scatter_round_trip():
    x = inputs.normal((50, 16), seed=3, tensor_id=31)
    xs, kept, _ = sel.select(x, 4.0)
    y = sel.scatter_rows(xs * 2, kept, np.zeros_like(x))
    np.testing.assert_array_equal(y[kept], 2 * x[kept])
    mask = np.ones(50, bool)
    mask[kept] = False
    assert np.all(y[mask] == 0)
