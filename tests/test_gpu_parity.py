"""GPU parity: the CUDA path through the C-ABI vs the oracle, element by element.

Counts, joint counts, HLL registers, n_sampled and the sample mask must be
bit-exact (BASELINE.json north_star).  Inputs are the seeded synthetic
workloads (synth/) at sizes the oracle finishes in seconds that still span
many CTAs, row quads and a ragged tail, plus edge cases.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu

I32MIN, I32MAX = -(2 ** 31), 2 ** 31 - 1
I64MIN, I64MAX = -(2 ** 63), 2 ** 63 - 1


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    gace.lib()
    assert torch.cuda.is_available()
    return gace


def _gpu_probe(G, cols_np, preds, pairs, rate, seed, hll_cols, row_offset=0, host=False):
    if host:
        cols = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in cols_np]
    else:
        cols = [torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols_np]
    dist = G.DistInfo(0, 1, row_offset, row_offset + len(cols_np[0])) if row_offset else None
    t = G.Table(cols, host=host, dist=dist, device=0)
    try:
        return t.probe(preds, pairs, rate, seed, hll_cols)
    finally:
        t.detach()


def _assert_same(got, want):
    n, c, j, r = want
    assert got.n_sampled == n
    np.testing.assert_array_equal(got.counts, c)
    np.testing.assert_array_equal(got.joints, j)
    assert got.regs.shape == r.shape
    np.testing.assert_array_equal(got.regs, r)


def _check(G, oracle, cols, preds, pairs=None, rate=1.0, seed=0, hll_cols=(), row_offset=0, host=False):
    want = oracle.probe(cols, preds, pairs, rate=rate, seed=seed, hll_cols=hll_cols, row_offset=row_offset)
    got = _gpu_probe(G, cols, preds, pairs, rate, seed, hll_cols, row_offset, host)
    _assert_same(got, want)
    return got


# ------------------------------------------------------------------ workload shapes

@pytest.mark.parametrize("name,nrows,rate", [
    ("C1", 100_003, 1.0), ("C1", 65_537, 0.37),
    ("C2", 200_001, 0.01), ("C2", 50_000, 0.5),
    ("C3", 300_002, 1.0), ("C3B", 100_001, 1.0),
    ("C4", 100_003, 1.0), ("C4", 40_000, 0.2),
    ("C5", 120_001, 1.0), ("C5_i64", 60_007, 1.0), ("C5", 50_000, 0.05),
])
def test_workloads(G, oracle, name, nrows, rate):
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, w.sample_seed + 17, w.hll_cols)


@pytest.mark.parametrize("name", ["C1", "C5"])
def test_host_table_path(G, oracle, name):
    w = synth.get(name, 70_001)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, 1.0, 0, w.hll_cols, host=True)
    _check(G, oracle, cols, w.preds, w.pairs, 0.3, 9, w.hll_cols, host=True)


def test_shard_offsets_and_merge(G, oracle):
    w = synth.get("C5", 90_000)
    cols = [x.numpy() for x in w.table()]
    whole = oracle.probe(cols, w.preds, w.pairs, rate=0.6, seed=5, hll_cols=w.hll_cols)
    cuts = [0, 4, 30_001, 61_113, 90_000]
    parts = []
    for s, e in zip(cuts, cuts[1:]):
        part = [c[s:e] for c in cols]
        parts.append(_check(G, oracle, part, w.preds, w.pairs, 0.6, 5, w.hll_cols, row_offset=s))
    assert sum(p.n_sampled for p in parts) == whole[0]
    np.testing.assert_array_equal(sum(p.counts for p in parts), whole[1])
    np.testing.assert_array_equal(sum(p.joints for p in parts), whole[2])
    np.testing.assert_array_equal(np.maximum.reduce([p.regs for p in parts]), whole[3])


# ------------------------------------------------------------------ edge cases

def _boundary_preds(col, vals):
    rows = []
    for op in range(5):
        for a in vals:
            for fl in (0, 1):
                rows.append((col, op, fl, a, 0))
    for a in vals[::2]:
        for b in vals[1::2]:
            rows.append((col, 5, 0, a, b))
            rows.append((col, 5, 1, a, b))
    return np.array(rows, dtype=synth.PRED_DTYPE)


@pytest.mark.parametrize("nrows", [0, 1, 3, 4, 5, 31, 32, 33, 4095, 4097, 148 * 1024 * 4 + 3])
def test_ragged_sizes(G, oracle, nrows):
    g = np.random.default_rng(nrows)
    c0 = g.integers(-5, 5, size=nrows).astype(np.int32)
    c1 = g.integers(I32MIN, I32MAX, size=nrows, endpoint=True).astype(np.int32)
    vals = [I64MIN, I32MIN - 1, I32MIN, -3, -1, 0, 2, 4, I32MAX, I32MAX + 1, I64MAX]
    P = np.concatenate([_boundary_preds(0, vals), _boundary_preds(1, [I32MIN, -7, 0, 10 ** 9, I32MAX])])
    Q = np.array([(0, 1), (5, 200), (3, 3), (100, 7)], dtype=synth.PAIR_DTYPE)
    for rate in (1.0, 0.5):
        _check(G, oracle, [c0, c1], P, Q, rate, 3, [0, 1])


def test_all_equal_column_max_contention(G, oracle):
    n = 2_000_003
    c = np.full(n, 7, dtype=np.int32)
    P = np.array([(0, 0, 0, 7, 0), (0, 1, 0, 7, 0), (0, 5, 0, 0, 10), (0, 0, 1, 7, 0)], dtype=synth.PRED_DTYPE)
    _check(G, oracle, [c, c.copy()], np.concatenate([P, P.copy().astype(synth.PRED_DTYPE)]),
           np.array([(0, 4), (1, 6)], dtype=synth.PAIR_DTYPE), 1.0, 0, [0])


@pytest.mark.parametrize("rate", [0.0, 2.0 ** -60, 0.01, 0.5, 1.0 - 2.0 ** -53, 1.0])
def test_sample_rates_and_mask(G, oracle, rate):
    w = synth.get("C1", 50_001)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, 42, w.hll_cols)
    t = G.Table([torch.from_numpy(c).cuda() for c in cols], dist=G.DistInfo(0, 1, 12345, 10 ** 9))
    try:
        np.testing.assert_array_equal(t.sample_mask(rate, 42), oracle.sample_mask(50_001, rate, 42, 12345))
    finally:
        t.detach()


def test_int64_wide_domain_search_mode(G, oracle):
    g = np.random.default_rng(1)
    n = 100_000
    c = g.integers(I64MIN, I64MAX, size=n, dtype=np.int64, endpoint=True)
    c[:10] = [I64MIN, I64MAX, 0, -1, 1, I64MIN + 1, I64MAX - 1, 5, 5, 5]
    small = g.integers(-1000, 1000, size=n).astype(np.int64) * (1 << 40)
    vals = [I64MIN, I64MIN + 1, -(1 << 62), -1, 0, 1, 5, 1 << 62, I64MAX - 1, I64MAX]
    P = np.concatenate([_boundary_preds(0, vals), _boundary_preds(1, [-(1 << 50), 0, 7 << 40, 1 << 52])])
    Q = np.array([(0, 150), (10, 11), (3, 140)], dtype=synth.PAIR_DTYPE)
    _check(G, oracle, [c, small], P, Q, 1.0, 0, [0, 1])
    _check(G, oracle, [c, small], P, Q, 0.4, 8, [0, 1], host=True)


def test_many_predicates_one_column(G, oracle):
    g = np.random.default_rng(2)
    n = 300_000
    c = g.integers(0, 1 << 20, size=n).astype(np.int32)
    lo = g.integers(0, 1 << 20, size=4096)
    w = g.integers(0, 5000, size=4096)
    ops = g.integers(0, 6, size=4096)
    P = np.zeros(4096, dtype=synth.PRED_DTYPE)
    P["col"] = 0
    P["op"] = ops
    P["flags"] = g.integers(0, 2, size=4096)
    P["a"] = lo
    P["b"] = lo + w
    Q = np.stack([g.integers(0, 4096, size=4096), g.integers(0, 4096, size=4096)], 1)
    Q = np.array([tuple(x) for x in Q], dtype=synth.PAIR_DTYPE)
    _check(G, oracle, [c], P, Q, 1.0, 0, [0])


def test_direct_pair_fallback(G, oracle):
    # many distinct predicates on both sides of one column pair: the 2-D grid does
    # not fit shared memory and the pairs are evaluated per row instead
    g = np.random.default_rng(3)
    n = 200_000
    a = g.integers(0, 100_000, size=n).astype(np.int32)
    b = g.integers(0, 100_000, size=n).astype(np.int32)
    k = 600
    P = np.zeros(2 * k, dtype=synth.PRED_DTYPE)
    P["col"][k:] = 1
    P["op"] = 5
    P["a"] = g.integers(0, 100_000, size=2 * k)
    P["b"] = P["a"] + g.integers(0, 20_000, size=2 * k)
    P["flags"] = g.integers(0, 2, size=2 * k)
    Q = np.array([(i, k + (i * 7) % k) for i in range(k)], dtype=synth.PAIR_DTYPE)
    _check(G, oracle, [a, b], P, Q, 1.0, 0, [])
    _check(G, oracle, [a, b], P, Q, 0.5, 1, [0])


def test_eight_columns_every_group(G, oracle):
    g = np.random.default_rng(4)
    n = 80_001
    cols = [g.integers(-50 * (c + 1), 50 * (c + 1), size=n).astype(np.int32 if c % 3 else np.int64)
            for c in range(9)]
    rows = []
    for c in range(8):
        for _ in range(6):
            x = int(g.integers(-60 * (c + 1), 60 * (c + 1)))
            rows.append((c, int(g.integers(0, 6)), int(g.integers(0, 2)), x, x + int(g.integers(0, 40))))
    P = np.array(rows, dtype=synth.PRED_DTYPE)
    Q = np.array([(int(i), int(j)) for i, j in zip(g.integers(0, 48, 200), g.integers(0, 48, 200))],
                 dtype=synth.PAIR_DTYPE)
    _check(G, oracle, cols, P, Q, 1.0, 0, [0, 3, 7])
    _check(G, oracle, cols, P, Q, 0.7, 2, [1, 2, 4, 5, 6])


def test_hll_only_and_nine_columns_rejected(G, oracle):
    g = np.random.default_rng(5)
    cols = [g.integers(-10 ** 6, 10 ** 6, size=10_000).astype(np.int32) for _ in range(9)]
    _check(G, oracle, cols, np.zeros(0, dtype=synth.PRED_DTYPE), None, 1.0, 0, list(range(8)))
    t = G.Table([torch.from_numpy(c).cuda() for c in cols])
    try:
        with pytest.raises(G.GaceError) as e:
            t.probe(np.zeros(0, dtype=synth.PRED_DTYPE), None, 1.0, 0, list(range(9)))
        assert e.value.status == G.GACE_EUNSUPPORTED
        with pytest.raises(G.GaceError) as e:
            t.probe(np.zeros(0, dtype=synth.PRED_DTYPE), None, float("nan"), 0, [0])
        assert e.value.status == G.GACE_EINVAL
        with pytest.raises(G.GaceError):
            t.probe(np.array([(9, 0, 0, 0, 0)], dtype=synth.PRED_DTYPE))
    finally:
        t.detach()


def test_randomised_sweep(G, oracle):
    """>= 1000 randomised small requests (SPEC.md S:543 style)."""
    g = np.random.default_rng(6)
    n = 20_011
    base = [g.integers(-30, 30, size=n).astype(np.int32), g.integers(0, 1000, size=n).astype(np.int32),
            (g.integers(-5, 5, size=n) * (1 << 33)).astype(np.int64)]
    t = G.Table([torch.from_numpy(c).cuda() for c in base])
    try:
        for trial in range(1000):
            np_ = int(g.integers(1, 12))
            rows = []
            for _ in range(np_):
                c = int(g.integers(0, 3))
                scale = [1, 30, 1 << 33][c]
                x = int(g.integers(-35, 35)) * scale
                rows.append((c, int(g.integers(0, 6)), int(g.integers(0, 2)), x, x + int(g.integers(-2, 20)) * scale))
            P = np.array(rows, dtype=synth.PRED_DTYPE)
            Q = np.array([(int(g.integers(0, np_)), int(g.integers(0, np_))) for _ in range(int(g.integers(0, 6)))],
                         dtype=synth.PAIR_DTYPE)
            rate = float(g.choice([1.0, 0.5, 0.05]))
            hll = [int(c) for c in g.choice(3, size=int(g.integers(0, 3)), replace=False)]
            got = t.probe(P, Q, rate, trial, hll)
            want = oracle.probe(base, P, Q, rate=rate, seed=trial, hll_cols=hll)
            _assert_same(got, want)
    finally:
        t.detach()


def test_derived_values_end_to_end(G, oracle):
    w = synth.get("C4", 100_000)
    cols = [x.numpy() for x in w.table()]
    got = _gpu_probe(G, cols, w.preds, w.pairs, 1.0, 0, w.hll_cols)
    sel, pcs, ndv, drift = G.derive(got.n_sampled, got.counts, w.pairs, got.joints, got.regs, w.ndv_hist)
    osel, opcs, ondv, odrift = oracle.derive(got.n_sampled, got.counts, w.pairs, got.joints, got.regs, w.ndv_hist)
    np.testing.assert_allclose(sel, osel, rtol=1e-12)
    np.testing.assert_allclose(pcs, opcs, rtol=1e-12)
    np.testing.assert_allclose(ndv, ondv, rtol=1e-12)
    np.testing.assert_allclose(drift, odrift, rtol=1e-12)


@pytest.fixture
def force_jit(monkeypatch):
    monkeypatch.setenv("GACE_JIT", "1")
    yield


@pytest.mark.parametrize("layout", ["0", "1"])
@pytest.mark.parametrize("name,nrows,rate", [
    ("C1", 100_003, 1.0), ("C1", 50_001, 0.3), ("C2", 100_001, 0.01), ("C3", 200_002, 1.0),
    ("C4", 60_003, 1.0), ("C5", 120_001, 1.0), ("C5_i64", 60_007, 1.0), ("C5", 50_000, 0.05),
])
def test_specialised_kernel_parity(G, oracle, force_jit, monkeypatch, name, nrows, rate, layout):
    """The NVRTC plan-specialised kernels (the ones large scans run) against the oracle:
    layout "0" = specialised for the plan structure (layout from the kernel parameters,
    jit == 1), "1" = structure and layout baked in (jit == 2)."""
    monkeypatch.setenv("GACE_JIT_LAYOUT", layout)
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    want = oracle.probe(cols, w.preds, w.pairs, rate=rate, seed=23, hll_cols=w.hll_cols)
    t = G.Table([torch.from_numpy(c).cuda() for c in cols])
    try:
        got = t.probe(w.preds, w.pairs, rate, 23, w.hll_cols)
        assert t.last_timing()["jit"] == 1 + int(layout), G.lib().gace_last_error()
    finally:
        t.detach()
    _assert_same(got, want)


def test_background_specialisation(G, oracle, monkeypatch):
    """Default JIT policy on a small table forced over the size threshold: the first probe
    runs the generic kernel while both specialised kernels compile in the background, the
    next ones run the structure-keyed and then the layout-keyed kernel; a second batch of
    the same structure (shifted bind values) reuses the structure-keyed kernel at once.
    Every result equals the oracle."""
    monkeypatch.delenv("GACE_JIT", raising=False)
    monkeypatch.delenv("GACE_JIT_LAYOUT", raising=False)
    monkeypatch.setenv("GACE_JIT_MIN_ROWS", "1")
    w = synth.get("C5", 90_001)
    cols = [x.numpy() for x in w.table()]
    t = G.Table([torch.from_numpy(c).cuda() for c in cols])
    try:
        want = oracle.probe(cols, w.preds, w.pairs, rate=1.0, seed=0, hll_cols=w.hll_cols)
        kinds = []
        for k in range(3):
            _assert_same(t.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols), want)
            kinds.append(t.last_timing()["jit"])
            G.jit_sync()
        assert kinds[0] in (0, 1, 2) and kinds[2] == 2, kinds
        P2 = w.preds.copy()
        P2["a"] += 3
        P2["b"] += 3
        want2 = oracle.probe(cols, P2, w.pairs, rate=1.0, seed=0, hll_cols=w.hll_cols)
        _assert_same(t.probe(P2, w.pairs, 1.0, 0, w.hll_cols), want2)
    finally:
        t.detach()


def test_specialised_kernel_edge_shapes(G, oracle, force_jit):
    test_direct_pair_fallback(G, oracle)
    test_eight_columns_every_group(G, oracle)
    test_int64_wide_domain_search_mode(G, oracle)
    for n in (1, 5, 33, 4097):
        test_ragged_sizes(G, oracle, n)


@pytest.mark.parametrize("name,rate", [("C1", 1.0), ("C5", 1.0), ("C5", 0.3), ("C5_i64", 1.0)])
def test_specialised_kernel_host_tables(G, oracle, force_jit, name, rate):
    """Host tables (clamped lookup tables, chunked launches) through the specialised kernel."""
    w = synth.get(name, 70_001)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, 3, w.hll_cols, host=True)


def test_clustered_columns(G, oracle, force_jit):
    """Sorted keys with runs (every aligned row quad equal in most places): the specialised
    kernel resolves such quads once; results must not change."""
    g = np.random.default_rng(7)
    n = 400_003
    ok = np.repeat(np.arange(n // 4 + 1, dtype=np.int32) * 3 + 5, 4)[:n]
    ok[1000:1003] = [7, 8, 9]                               # a few broken quads
    other = g.integers(0, 1000, size=n).astype(np.int32)
    P = np.array([(0, 5, 0, 100, 90_000), (0, 1, 0, 50_000, 0), (0, 0, 0, 3 * 77 + 5, 0), (1, 5, 1, 10, 500),
                  (0, 4, 1, 123_456, 0)], dtype=synth.PRED_DTYPE)
    Q = np.array([(0, 3), (1, 3), (2, 3), (4, 3)], dtype=synth.PAIR_DTYPE)
    for rate in (1.0, 0.4):
        _check(G, oracle, [ok, other], P, Q, rate, 5, [0, 1])


# ------------------------------------------------------------------ scale: many iterations per thread
# Small tables give each of the 148 x 1024 threads less than one row unit, so the HLL skip
# bound (refreshed at iterations 4, 8, 16, then every 32, from registers merged across
# CTAs) and the long-run paths never run.  These sizes give every thread 8..60 iterations.

@pytest.mark.parametrize("name,nrows,rate", [
    ("C5", 40_000_003, 1.0), ("C4", 24_000_001, 1.0), ("C3", 30_000_002, 1.0), ("C5_i64", 20_000_001, 1.0),
    ("C5", 36_000_000, 0.5),
])
def test_scale_many_iterations(G, oracle, name, nrows, rate):
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, 11, w.hll_cols)


def test_fmt1t_special_cells(G, oracle):
    """Level-1 cells holding 2, 3, 4..8 and dozens of breakpoints (direct records, lists and
    nested blocks behind the one-threshold format), on both sides of packed pair grids."""
    g = np.random.default_rng(41)
    n = 3_000_001
    a = g.integers(0, 1_000_000, size=n).astype(np.int32)
    b = g.integers(0, 1_000_000, size=n).astype(np.int32)
    # keys concentrated where the breakpoints are dense
    a[: n // 3] = g.integers(500_000, 500_400, size=n // 3)
    b[: n // 4] = g.integers(10, 90, size=n // 4)
    rows = []
    for v in range(500_000, 500_200, 3):                      # dense EQ binds: nested / list cells
        rows.append((0, 0, 0, v, 0))
    for lo in (100, 5_000, 77_777, 500_100, 900_000):        # narrow BETWEENs: 2 breakpoints per cell
        rows += [(0, 5, 0, lo, lo + 1), (0, 5, 1, lo + 2, lo + 9), (0, 5, 0, lo, lo + 30_000)]
    for v in range(10, 90, 7):                                # b: clustered EQs and ranges
        rows += [(1, 0, 0, v, 0), (1, 5, 0, v, v + 3)]
    rows += [(1, 1, 0, 500_000, 0), (1, 4, 1, 999_000, 0), (1, 5, 0, 0, 999_999)]
    P = np.array(rows, dtype=synth.PRED_DTYPE)
    na = sum(1 for r in rows if r[0] == 0)
    Q = np.array([(i, na + j) for i in range(0, na, 5) for j in range(0, len(rows) - na, 4)][:300],
                 dtype=synth.PAIR_DTYPE)
    for rate in (1.0, 0.45):
        _check(G, oracle, [a, b], P, Q, rate, 21, [0, 1])


def test_fmt1t_special_cells_specialised(G, oracle, force_jit):
    test_fmt1t_special_cells(G, oracle)


@pytest.mark.slow
def test_full_size_shard_invariance(G):
    """At BASELINE's full C5 size (the bench configuration): the whole-table probe equals the
    sum / max merge of two row shards probed with their global row offsets, and the count
    invariants hold (predicate + complement = n_sampled, joint <= both marginals)."""
    w = synth.get("C5")
    cols = [c.cuda() for c in w.table(device="cuda")]
    N = w.nrows
    t = G.Table(cols)
    try:
        for rate, seed in ((1.0, 0), (0.01, 0x5EED)):
            whole = t.probe(w.preds, w.pairs, rate, seed, w.hll_cols)
            info = (t.last_timing(), G.lib().gace_last_error())
            cut = (N // 2 + 12345) & ~3                  # 16-byte aligned shard start
            parts = []
            for s, e in ((0, cut), (cut, N)):
                tp = G.Table([c[s:e] for c in cols], dist=G.DistInfo(0, 1, s, N))
                try:
                    parts.append(tp.probe(w.preds, w.pairs, rate, seed, w.hll_cols))
                finally:
                    tp.detach()
            assert whole.n_sampled == sum(p.n_sampled for p in parts)
            bad = np.nonzero(whole.counts != parts[0].counts + parts[1].counts)[0]
            assert len(bad) == 0, (info, rate, sorted(set(int(w.preds["col"][i]) for i in bad)), bad[:8],
                                   whole.counts[bad[:4]], parts[0].counts[bad[:4]], parts[1].counts[bad[:4]])
            np.testing.assert_array_equal(whole.joints, sum(p.joints for p in parts))
            np.testing.assert_array_equal(whole.regs, np.maximum(parts[0].regs, parts[1].regs))
            P = w.preds
            assert np.all(whole.counts <= whole.n_sampled)
            for q, (i, j) in enumerate(zip(w.pairs["i"], w.pairs["j"])):
                assert whole.joints[q] <= min(whole.counts[i], whole.counts[j])
            neg = P.copy()
            neg["flags"] ^= 1
            comp = t.probe(neg, None, rate, seed, [])
            np.testing.assert_array_equal(whole.counts + comp.counts, np.full(len(P), whole.n_sampled, np.uint64))
    finally:
        t.detach()


@pytest.mark.parametrize("name,nrows,rate", [("C4", 100_003, 1.0), ("C4", 80_001, 0.3), ("C1", 100_003, 1.0),
                                             ("C1", 50_001, 0.37), ("C3", 200_002, 1.0)])
def test_presence_bitmap_hll(G, oracle, monkeypatch, name, nrows, rate):
    """HLL by presence bitmap (small int32 domains; the finalize hashes each present value)
    forced at sizes where the planner would not pick it, generic and specialised kernels."""
    monkeypatch.setenv("GACE_FORCE_BITMAP", "1")
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    for jit in ("0", "1"):
        monkeypatch.setenv("GACE_JIT", jit)
        _check(G, oracle, cols, w.preds, w.pairs, rate, 29, w.hll_cols)


def _high_rank_keys(is64: bool, n: int, seed: int):
    """Keys whose HLL rank exceeds 16 (the shared-memory registers' in-thermometer range:
    such ranks also go straight to the merged registers), found with the generator's own
    hashes restated in numpy (fmix32 / mix64(x + gamma))."""
    g = np.random.default_rng(seed)
    out = []
    M = np.uint64(0xFFFFFFFFFFFFFFFF)
    while len(out) < n:
        if is64:
            x = g.integers(-(1 << 62), 1 << 62, size=1 << 21, dtype=np.int64)
            with np.errstate(over="ignore"):
                z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
                z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
                z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
                z = z ^ (z >> np.uint64(31))
                w = (z << np.uint64(12)) & M
            ok = w < np.uint64(1 << 48)                      # rank >= 17
        else:
            x = g.integers(-(1 << 31), 1 << 31, size=1 << 22, dtype=np.int64).astype(np.int32)
            h = x.astype(np.uint32).astype(np.uint64)
            h ^= h >> np.uint64(16)
            h = (h * np.uint64(0x85EBCA6B)) & np.uint64(0xFFFFFFFF)
            h ^= h >> np.uint64(13)
            h = (h * np.uint64(0xC2B2AE35)) & np.uint64(0xFFFFFFFF)
            h ^= h >> np.uint64(16)
            w = (h << np.uint64(12)) & np.uint64(0xFFFFFFFF)
            ok = w < np.uint64(1 << 16)
        out.extend(x[ok].tolist())
    return np.array(out[:n], dtype=np.int64 if is64 else np.int32)


@pytest.mark.parametrize("jit", ["0", "1"])
def test_hll_ranks_above_16(G, oracle, monkeypatch, jit):
    """HLL ranks 17..21 (int32) and 17..53 (int64) -- beyond the 16-bit shared-memory
    thermometers -- mixed into ordinary keys, with and without predicates on the columns,
    generic and specialised kernels: registers bit-exact against the oracle."""
    monkeypatch.setenv("GACE_JIT", jit)
    g = np.random.default_rng(77)
    n = 300_007
    hi32 = _high_rank_keys(False, 64, 1)
    hi64 = _high_rank_keys(True, 64, 2)
    a = g.integers(0, 1 << 20, size=n).astype(np.int32)
    b = g.integers(-(1 << 40), 1 << 40, size=n).astype(np.int64)
    pos = g.choice(n, size=2000, replace=False)
    a[pos] = hi32[g.integers(0, len(hi32), size=2000)]
    b[pos] = hi64[g.integers(0, len(hi64), size=2000)]
    P = np.array([(0, 5, 0, 1000, 500_000), (1, 1, 0, 0, 0)], dtype=synth.PRED_DTYPE)
    Q = np.array([(0, 1)], dtype=synth.PAIR_DTYPE)
    for preds, pairs in ((P, Q), (P[:0], None)):
        for rate in (1.0, 0.6):
            _check(G, oracle, [a, b], preds, pairs, rate, 13, [0, 1])
            _check(G, oracle, [a], preds[preds["col"] == 0], None, rate, 13, [0])


@pytest.mark.parametrize("compact", ["0", "1"])
@pytest.mark.parametrize("jit", ["0", "1"])
@pytest.mark.parametrize("name,nrows,rate", [("C5", 300_001, 0.01), ("C1", 200_003, 0.3), ("C5_i64", 150_007, 0.05),
                                             ("C4", 200_001, 0.002), ("C3", 250_002, 0.1)])
def test_sample_compaction(G, oracle, monkeypatch, compact, jit, name, nrows, rate):
    """Sampled probes with the kept rows compacted per warp (GACE_COMPACT=1: rows queued in
    shared memory, worked on 32 at a time) and without (per-quad work), on generic and
    specialised kernels, at rates either side of the 1/8 default switch."""
    monkeypatch.setenv("GACE_COMPACT", compact)
    monkeypatch.setenv("GACE_JIT", jit)
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, 31, w.hll_cols)


@pytest.mark.parametrize("jit", ["0", "1"])
@pytest.mark.parametrize("name,nrows,rate", [("C5", 1_000_003, 1.0), ("C1", 700_001, 0.3), ("C5_i64", 500_009, 0.05),
                                             ("C4", 600_001, 1.0)])
def test_chunked_launches(G, oracle, monkeypatch, jit, name, nrows, rate):
    """A table scanned in several launches (GACE_MAX_LAUNCH_ROWS forces ~100K-row launches):
    each launch's own ragged tail, its row offset into the sample, HLL partials max-merged
    across launches and counters summed across them (the multi-launch path)."""
    monkeypatch.setenv("GACE_MAX_LAUNCH_ROWS", "100004")
    monkeypatch.setenv("GACE_JIT", jit)
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    _check(G, oracle, cols, w.preds, w.pairs, rate, 17, w.hll_cols)
    t = G.Table([torch.from_numpy(c).cuda() for c in cols])
    try:
        t.probe(w.preds, w.pairs, rate, 17, w.hll_cols)
        assert t.last_timing()["scan_launches"] == (nrows + 100003) // 100004
    finally:
        t.detach()


_EXIT_SCRIPT = r"""
import sys
sys.path.insert(0, ".")
import torch, synth
from paper_2512_19750_b200 import gace
w = synth.get(sys.argv[1], 300_000)
t = gace.Table([w.column(c, device="cuda") for c in range(len(w.columns))])
r = t.probe(w.preds, w.pairs, float(sys.argv[2]), 1, w.hll_cols)   # queues a background compile
print("probed", r.n_sampled, flush=True)
"""


@pytest.mark.parametrize("name,rate", [("C1", 1.0), ("C5", 1.0), ("C2", 0.01), ("C4", 1.0)])
def test_exit_with_compile_in_flight(G, name, rate):
    """A process that exits right after its first probe -- the background NVRTC compile of
    the specialised kernel still queued or running -- exits cleanly (gace_jit_shutdown from the
    binding's atexit hook; without it such exits crashed or hung)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    env.pop("GACE_JIT", None)                       # the default: background compiles
    r = subprocess.run([sys.executable, "-c", _EXIT_SCRIPT, name, str(rate)], cwd=root, env=env,
                       capture_output=True, text=True, timeout=180)
    assert r.returncode == 0, (r.returncode, r.stdout[-2000:], r.stderr[-2000:])
    assert "probed" in r.stdout


@pytest.mark.parametrize("trial", range(4))
@pytest.mark.parametrize("force_jit", [False, True])
def test_budget_bound_refined_tables(G, oracle, monkeypatch, trial, force_jit):
    """Plans at the full-scan shared-memory budget (224 KB): four wide int32 columns with up to
    160 ranges each (narrow ones put several breakpoints in a cell, others sit on power-of-two
    cell starts), 64 cross-column pairs and HLL on every column, so the planner coarsens and
    then refines the tables (test_planner.py::test_table_sizing_by_estimate).  Exact against the
    oracle through the generic and the plan-specialised kernel, full scan and sampled."""
    if force_jit:
        monkeypatch.setenv("GACE_JIT", "1")
        monkeypatch.setenv("GACE_JIT_MIN_ROWS", "0")
    g = np.random.default_rng(100 + trial)
    n = 300_007
    spans = [int(10 ** g.uniform(4, 9)) for _ in range(4)]
    cols = [g.integers(0, sp, size=n, endpoint=True).astype(np.int32) for sp in spans]
    for c, sp in enumerate(spans):          # exact domain ends, whatever the draw
        cols[c][c] = 0
        cols[c][c + 4] = sp
    rows = []
    for c, sp in enumerate(spans):
        for _ in range(int(g.integers(20, 160))):
            a = int(g.integers(0, sp))
            w = int(g.choice([0, 1, 3, 100, sp // 50 + 1]))
            rows.append((c, 5, 0, a, min(a + w, sp)))
        for k in range(8):
            rows.append((c, 2, 0, (k + 1) << int(g.integers(4, 16)), 0))
    P = np.array(rows, dtype=synth.PRED_DTYPE)
    Q = np.array([(i, j) for i in range(0, len(P), 37) for j in range(5, len(P), 53)
                  if P["col"][i] != P["col"][j]][:64], dtype=synth.PAIR_DTYPE)
    for rate in (1.0, 0.3):
        _check(G, oracle, cols, P, Q, rate=rate, seed=trial, hll_cols=[0, 1, 2, 3])
