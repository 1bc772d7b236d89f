"""Pins of the candidate-set oracle (oracle_probe_sets / brute_probe_sets), CPU only.

What they compute: PAPER.md §IV-H Experiment D (lines 250-270): M candidate predicate
sets, K predicates each, the conjunction of each set counted over the (sampled) rows;
SPEC.md evaluate_bitmasks: per-set count = popcount of the AND-ed predicate bitmaps.

Pinned against things other than the oracle's own formula:
* the pure-Python brute force (written separately) on random tiny tables;
* the already-pinned probe oracle: a one-member set is that predicate's count, a
  two-member set is the pair's joint count, the empty set is n_sampled;
* closed forms on arange columns (a window's size), contradictions ({p, NOT p} = 0),
  tautologies, and order / duplicate invariance and monotonicity under adding members.
"""
import numpy as np
import pytest


def _rand_batch(oracle, rng, ncols, npreds, nsets, kmax, lo, hi):
    P = np.zeros(npreds, dtype=oracle.PRED_DTYPE)
    P["col"] = rng.integers(0, ncols, npreds)
    P["op"] = rng.integers(0, 6, npreds)
    P["flags"] = rng.integers(0, 2, npreds)
    P["a"] = rng.integers(lo, hi, npreds)
    P["b"] = rng.integers(lo, hi, npreds)
    sets = [list(rng.integers(0, npreds, rng.integers(0, kmax + 1))) for _ in range(nsets)]
    return P, sets


@pytest.mark.parametrize("seed", range(6))
def test_c_matches_brute_force(oracle, seed):
    rng = np.random.default_rng(1000 + seed)
    ncols, nrows = 3, int(rng.integers(0, 60))
    dts = [np.int32, np.int64, np.int32]
    cols = [rng.integers(-8, 9, nrows).astype(d) for d in dts]
    P, sets = _rand_batch(oracle, rng, ncols, 12, 9, 5, -10, 11)
    for rate, s in ((1.0, 0), (0.5, 3), (0.0, 1)):
        n, c = oracle.probe_sets(cols, P, sets, rate=rate, seed=s, row_offset=7)
        bn, bc = oracle.brute_probe_sets([list(map(int, x)) for x in cols], P, sets, rate=rate, seed=s,
                                         row_offset=7)
        assert n == bn
        assert [int(x) for x in c] == bc


def test_relations_to_the_probe(oracle):
    rng = np.random.default_rng(7)
    nrows = 3000
    cols = [rng.integers(0, 50, nrows).astype(np.int32), rng.integers(-(2 ** 40), 2 ** 40, nrows)]
    P, _ = _rand_batch(oracle, rng, 2, 20, 0, 0, 0, 50)
    pairs = np.array([(i, (i * 7 + 3) % 20) for i in range(20)], dtype=oracle.PAIR_DTYPE)
    for rate in (1.0, 0.3):
        n, counts, joints, _ = oracle.probe(cols, P, pairs, rate=rate, seed=5)
        sets = [[p] for p in range(20)] + [[int(q["i"]), int(q["j"])] for q in pairs] + [[]]
        sn, sc = oracle.probe_sets(cols, P, sets, rate=rate, seed=5)
        assert sn == n
        assert list(sc[:20]) == list(counts)
        assert list(sc[20:40]) == list(joints)
        assert int(sc[40]) == n


def test_closed_forms(oracle):
    N = 1000
    col = np.arange(N, dtype=np.int32)
    GE, LT, EQ, BETWEEN = oracle.GE, oracle.LT, oracle.EQ, oracle.BETWEEN
    P = np.array([(0, GE, 0, 100, 0), (0, LT, 0, 350, 0), (0, BETWEEN, 0, 200, 5000), (0, EQ, 0, 300, 0),
                  (0, EQ, oracle.NEGATE, 300, 0), (0, GE, 0, -(2 ** 63), 0)], dtype=oracle.PRED_DTYPE)
    sets = [[0, 1], [0, 1, 2], [3, 4], [5], [5, 5, 0], [2, 1, 0], [0, 1, 0, 1]]
    n, c = oracle.probe_sets([col], P, sets)
    assert n == N
    assert int(c[0]) == 250            # [100, 350)
    assert int(c[1]) == 150            # [200, 350)
    assert int(c[2]) == 0              # EQ 300 and NOT EQ 300
    assert int(c[3]) == N              # v >= INT64_MIN: tautology
    assert int(c[4]) == N - 100
    assert int(c[5]) == int(c[1])      # member order
    assert int(c[6]) == int(c[0])      # duplicate members


def test_monotone_in_members(oracle):
    rng = np.random.default_rng(11)
    cols = [rng.integers(0, 20, 5000).astype(np.int32) for _ in range(3)]
    P, _ = _rand_batch(oracle, rng, 3, 16, 0, 0, 0, 20)
    chain = [list(range(k)) for k in range(17)]
    _, c = oracle.probe_sets(cols, P, chain, rate=0.7, seed=9)
    assert all(int(c[k + 1]) <= int(c[k]) for k in range(16))


def test_rejects_bad_arguments(oracle):
    col = [np.arange(10, dtype=np.int32)]
    P = np.array([(0, oracle.EQ, 0, 1, 0)], dtype=oracle.PRED_DTYPE)
    with pytest.raises(oracle.OracleError):
        oracle.probe_sets(col, P, [[1]])
    with pytest.raises(oracle.OracleError):
        oracle.probe_sets(col, P, [[0]], rate=1.5)
