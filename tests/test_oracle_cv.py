"""Est.CV oracle pins (§IV-C Exp. B, lines 121-141), CPU only:
the full sample gives CV = 0 (every probe exact); a constant-free two-point closed
form; the binomial law -- CV of a Bernoulli-sampled selectivity ~ sqrt((1 - q)/(q N S)) for
rate q, N rows, true selectivity S -- and its 1/sqrt(budget) scaling, CV(4n)/CV(n) in
0.5 +- 0.2; mean 0 -> NaN."""
import math

import numpy as np
import pytest


def test_full_sample_is_exact(oracle):
    col = np.arange(10_000, dtype=np.int32)
    P = np.array([(0, oracle.LT, 0, 5000, 0), (0, oracle.GE, 0, 2000, 0)], dtype=oracle.PRED_DTYPE)
    Q = np.array([(0, 1)], dtype=oracle.PAIR_DTYPE)
    cs, cj, cp = oracle.estimate_cv([col], P, Q, 1.0, [1, 2, 3])
    # identical estimates: only the rounding of the running mean remains
    assert max(cs + cj + cp) <= 1e-14


def test_two_point_closed_form(oracle):
    # xs = (a, b): mean (a+b)/2, sample sd |a-b|/sqrt(2)  ->  CV = sqrt(2)|a-b|/(a+b)
    assert oracle.cv([0.2, 0.4]) == pytest.approx(math.sqrt(2) * 0.2 / 0.6, rel=1e-15)
    assert math.isnan(oracle.cv([0.0, 0.0]))


def test_binomial_law_and_budget_scaling(oracle):
    N = 200_000
    col = np.arange(N, dtype=np.int32)
    P = np.array([(0, oracle.LT, 0, N // 2, 0)], dtype=oracle.PRED_DTYPE)     # S = 0.5
    seeds = list(range(1, 41))
    cvs = {}
    for q in (0.01, 0.04):
        cs, _, _ = oracle.estimate_cv([col], P, None, q, seeds)
        cvs[q] = cs[0]
        # S_hat = K/n with n ~ Bin(N, q): CV ~ sqrt((1 - S) / (S q N)) (ratio estimator)
        law = math.sqrt((1 - 0.5) / (0.5 * q * N))
        assert 0.6 * law < cs[0] < 1.5 * law
    assert 0.3 <= cvs[0.04] / cvs[0.01] <= 0.7
