"""GPU parity of gace_probe_sets (candidate-set conjunction counts, §IV-H Exp. D,
SURVEY.md §8(f) NEXT-1) against the oracle (oracle_probe_sets), bit-exact.

Covers the Exp. D workload shape, random batches over int32 / int64 columns with every
operator, negation, bounds outside the column domain and empty BETWEENs, 1..256 sets
(one to eight 32-set words), empty and duplicated members, ragged row counts, sampling
with a shard row offset, dense EQ sweeps (many breakpoints per cell), full 64-bit domains,
argument errors, and at full Exp. D size the identities with the (oracle-checked) probe:
one-member sets = counts, two-member sets = joint counts, the empty set = n_sampled.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

I64MIN, I64MAX = -(2 ** 63), 2 ** 63 - 1


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    gace.lib()
    assert torch.cuda.is_available()
    return gace


def _gpu_sets(G, cols_np, preds, sets, rate=1.0, seed=0, row_offset=0):
    cols = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols_np]
    dist = G.DistInfo(0, 1, row_offset, row_offset + len(cols_np[0])) if row_offset else None
    t = G.Table(cols, dist=dist, device=0)
    try:
        return t.probe_sets(preds, sets, rate, seed)
    finally:
        t.detach()


def _check(G, oracle, cols, preds, sets, rate=1.0, seed=0, row_offset=0):
    n, c = oracle.probe_sets(cols, preds, sets, rate=rate, seed=seed, row_offset=row_offset)
    gn, gc = _gpu_sets(G, cols, preds, sets, rate, seed, row_offset)
    assert gn == n
    np.testing.assert_array_equal(gc, c)
    return gc


@pytest.mark.parametrize("name,nrows,rate", [("D", 200_003, 1.0), ("D", 100_001, 0.3), ("D_m1_k16", 50_002, 1.0)])
def test_expd_workload(G, oracle, name, nrows, rate):
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    c = _check(G, oracle, cols, w.preds, w.sets, rate, 11)
    assert c.max() > 0


def _rand_batch(oracle, rng, cols, npreds, nsets, kmax):
    P = np.zeros(npreds, dtype=oracle.PRED_DTYPE)
    P["col"] = rng.integers(0, len(cols), npreds)
    P["op"] = rng.integers(0, 6, npreds)
    P["flags"] = rng.integers(0, 2, npreds)
    for i in range(npreds):
        col = cols[P["col"][i]]
        pick = lambda: int(col[rng.integers(0, len(col))]) if len(col) and rng.random() < 0.8 else int(  # noqa: E731
            rng.choice([I64MIN, I64MAX, -(2 ** 31) - 1, 2 ** 31, 0, -1]))
        a, b = pick(), pick()
        if P["op"][i] == 5 and rng.random() < 0.8:
            a, b = min(a, b), max(a, b)
        P["a"][i], P["b"][i] = a, b
    sets = []
    for _ in range(nsets):
        k = int(rng.integers(0, kmax + 1))
        sets.append([int(x) for x in rng.integers(0, npreds, k)])
    return P, sets


@pytest.mark.parametrize("nsets", [1, 31, 32, 33, 64, 65, 128, 200, 256])
def test_random_batches(G, oracle, nsets):
    rng = np.random.default_rng(500 + nsets)
    n = 20_011
    cols = [rng.integers(-50, 50, n).astype(np.int32), rng.integers(-(2 ** 40), 2 ** 40, n),
            rng.integers(0, 1000, n).astype(np.int32)]
    P, sets = _rand_batch(oracle, rng, cols, 40, nsets, 6)
    sets[0] = []                       # empty set: every kept row
    if nsets > 1:
        sets[1] = [3, 3, 3]            # duplicated member
    _check(G, oracle, cols, P, sets, 1.0, 0)
    _check(G, oracle, cols, P, sets, 0.42, 77, row_offset=123_457)


@pytest.mark.parametrize("nrows", [0, 1, 3, 5, 8, 4097, 77_777])
def test_ragged_rows(G, oracle, nrows):
    rng = np.random.default_rng(nrows + 3)
    cols = [rng.integers(-1000, 1000, nrows).astype(np.int32), rng.integers(-5, 5, nrows)]
    P, sets = _rand_batch(oracle, rng, [c if len(c) else np.zeros(1, c.dtype) for c in cols], 12, 20, 4)
    _check(G, oracle, cols, P, sets)
    _check(G, oracle, cols, P, sets, 0.5, 3)


def test_dense_eq_sweep(G, oracle):
    """Zipf column with EQ binds on consecutive values (C3's bind sweep): cells holding many
    breakpoints take the in-cell binary search."""
    w = synth.get("C3", 300_001)
    cols = [x.numpy() for x in w.table()]
    P = w.preds[:512]
    sets = [[v] for v in range(200)] + [[v, v + 1] for v in range(0, 40, 2)] + [[0, 512 - 1]] + \
        [[v for v in range(300, 330)]]
    _check(G, oracle, cols, P, sets[:256])


def test_full_64bit_domain(G, oracle):
    rng = np.random.default_rng(5)
    n = 30_000
    c = rng.integers(I64MIN, I64MAX, n, dtype=np.int64)
    c[:4] = [I64MIN, I64MAX, 0, -1]
    P = np.array([(0, oracle.GE, 0, 0, 0), (0, oracle.LT, 0, I64MAX, 0), (0, oracle.BETWEEN, 1, -5, 5),
                  (0, oracle.EQ, 0, I64MIN, 0), (0, oracle.EQ, 1, I64MAX, 0), (0, oracle.LE, 0, int(c[10]), 0)],
                 dtype=oracle.PRED_DTYPE)
    sets = [[0], [1], [2], [3], [4], [5], [0, 1, 2], [3, 4], [0, 5], []]
    _check(G, oracle, [c], P, sets)


def test_errors(G, oracle):
    cols = [torch.arange(100, dtype=torch.int32, device="cuda")]
    t = G.Table(cols, device=0)
    P = np.array([(0, oracle.EQ, 0, 1, 0)], dtype=oracle.PRED_DTYPE)
    try:
        with pytest.raises(G.GaceError) as e:
            t.probe_sets(P, [[1]])
        assert e.value.status == G.GACE_EINVAL
        with pytest.raises(G.GaceError) as e:
            t.probe_sets(P, [[0]] * 257)
        assert e.value.status == G.GACE_EUNSUPPORTED
        with pytest.raises(G.GaceError) as e:
            t.probe_sets(P, [[0]], sample_rate=float("nan"))
        assert e.value.status == G.GACE_EINVAL
    finally:
        t.detach()
    h = G.Table([np.arange(100, dtype=np.int32)], host=True, device=0)
    try:
        with pytest.raises(G.GaceError) as e:
            h.probe_sets(P, [[0]])
        assert e.value.status == G.GACE_EUNSUPPORTED
    finally:
        h.detach()


def test_full_size_identities(G):
    """Exp. D at BASELINE size (600M rows): sets of one / two members and the empty set
    equal the probe's counts / joints / n_sampled (both through the C-ABI).  The sets
    kernel itself is oracle-checked at this size by
    tests/test_gpu_fullsize.py::test_exp_d_full_size_vs_oracle, the probe by
    test_bench_config_full_size_vs_oracle."""
    w = synth.get("D")
    cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    t = G.Table(cols, device=0)
    try:
        pairs = np.array([(s[0], s[1]) for s in w.sets], dtype=G.PAIR_DTYPE)
        for rate, seed in ((1.0, 0), (0.01, 5)):
            r = t.probe(w.preds, pairs, rate, seed, [])
            sets = [[p] for p in range(len(w.preds))] + [list(s[:2]) for s in w.sets] + [[]]
            out = []
            for k in range(0, len(sets), 256):
                n, c = t.probe_sets(w.preds, sets[k:k + 256], rate, seed)
                assert n == r.n_sampled
                out.extend(int(x) for x in c)
            assert out[:len(w.preds)] == [int(x) for x in r.counts]
            assert out[len(w.preds):len(w.preds) + len(w.sets)] == [int(x) for x in r.joints]
            assert out[-1] == r.n_sampled
            n, c = t.probe_sets(w.preds, w.sets, rate, seed)        # the bench batch runs
            assert n == r.n_sampled and c.max() <= n
    finally:
        t.detach()


def test_estimate_cv_matches_oracle(G, oracle):
    """Est.CV (gace_estimate_cv, PAPER.md Exp. B) == the oracle's, derived doubles within
    1e-12 relative (the per-seed counts are bit-exact)."""
    w = synth.get("C1", 150_001)
    cols = [x.numpy() for x in w.table()]
    t = G.Table([torch.from_numpy(c).cuda() for c in cols], device=0)
    try:
        seeds = [11, 12, 13, 14, 15]
        for rate in (0.02, 0.3, 1.0):
            got = t.estimate_cv(w.preds, w.pairs, rate, seeds)
            want = oracle.estimate_cv(cols, w.preds, w.pairs, rate, seeds)
            for g, wv in zip(got, want):
                np.testing.assert_allclose(g, np.asarray(wv, dtype=np.float64), rtol=1e-12, atol=1e-15)
        with pytest.raises(G.GaceError):
            t.estimate_cv(w.preds, w.pairs, 0.5, [1])
    finally:
        t.detach()
