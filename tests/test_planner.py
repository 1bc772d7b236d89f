"""The host planner on CPU (gace_debug_buckets): for every probed column the
planned lookup table must resolve each value to #{breakpoints <= v}, and every
predicate's truth (the oracle's operator evaluation) must be constant within a
bucket -- i.e. the breakpoints are exactly right and the table never reads out
of range.  Covers device-table domains (min/max) and host tables (clamp)."""
import numpy as np
import pytest

import synth

I32MIN, I32MAX = -(2 ** 31), 2 ** 31 - 1
I64MIN, I64MAX = -(2 ** 63), 2 ** 63 - 1


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    return gace


def _check_column(G, oracle, dtypes, dlo, dhi, host, preds, pairs, hll, col, values):
    b, mode, bps = G.debug_buckets(dtypes, dlo, dhi, host, preds, pairs, hll, col, values)
    np.testing.assert_array_equal(b, np.searchsorted(bps, values, side="right"))
    assert np.all(np.diff(bps) > 0)
    # predicate truth is a function of the bucket (numpy restatement of the operators)
    cnt = np.bincount(b.astype(np.int64))
    for p in preds:
        if int(p["col"]) != col:
            continue
        t = _truth(int(p["op"]), int(p["flags"]), int(p["a"]), int(p["b"]), values)
        s = np.bincount(b.astype(np.int64), weights=t.astype(np.float64), minlength=len(cnt))
        assert np.all((s == 0) | (s == cnt)), (p, bps)
    return mode


def _truth(op, fl, a, b, v):
    # exact int64 comparisons via Python-int clipping of the bounds into the int64 range
    if op == 0:
        t = v == a if I64MIN <= a <= I64MAX else np.zeros(len(v), bool)
    elif op == 1:
        t = v < a
    elif op == 2:
        t = v <= a
    elif op == 3:
        t = v > a
    elif op == 4:
        t = v >= a
    else:
        t = (v >= a) & (v <= b)
    return ~t if fl & 1 else t


def _values(g, lo, hi, bps, n=4000):
    v = list(g.integers(lo, hi, size=n, endpoint=True, dtype=np.int64)) + [lo, hi]
    for t in bps:
        for d in (-1, 0, 1):
            if lo <= t + d <= hi:
                v.append(t + d)
    return np.array(v, dtype=np.int64)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C3B", "C4", "C5", "C5_i64"])
@pytest.mark.parametrize("host", [False, True])
def test_workload_plans(G, oracle, name, host):
    w = synth.get(name, 50_000)
    t = [x.numpy() for x in w.table()]
    dtypes = [0 if x.dtype == np.int32 else 1 for x in t]
    if host:
        dlo = [I32MIN if d == 0 else I64MIN for d in dtypes]
        dhi = [I32MAX if d == 0 else I64MAX for d in dtypes]
    else:
        dlo = [int(x.min()) for x in t]
        dhi = [int(x.max()) for x in t]
    g = np.random.default_rng(0)
    for c in sorted(set(int(x) for x in w.preds["col"])):
        _, _, bps = G.debug_buckets(dtypes, dlo, dhi, host, w.preds, w.pairs, w.hll_cols, c, [])
        vals = np.concatenate([t[c].astype(np.int64), _values(g, int(t[c].min()), int(t[c].max()), bps)])
        mode = _check_column(G, oracle, dtypes, dlo, dhi, host, w.preds, w.pairs, w.hll_cols, c, vals)
        if dtypes[c] == 0:
            assert mode == 0, f"{name} column {c} fell back to binary search"


def test_equality_on_wide_columns_stays_in_lut(G, oracle):
    g = np.random.default_rng(1)
    eqs = g.integers(I32MIN, I32MAX, size=200)
    P = np.array([(0, 0, 0, int(a), 0) for a in eqs] + [(0, 5, 1, -5, 5), (0, 1, 0, 3, 0)],
                 dtype=synth.PRED_DTYPE)
    for host in (False, True):
        _, _, bps = G.debug_buckets([0], [I32MIN], [I32MAX], host, P, None, [], 0, [])
        vals = _values(g, I32MIN, I32MAX, bps)
        assert _check_column(G, oracle, [0], [I32MIN], [I32MAX], host, P, None, [], 0, vals) == 0


def test_dense_and_clustered_breakpoints(G, oracle):
    g = np.random.default_rng(2)
    rows = [(0, 0, 0, v, 0) for v in range(1024)]                       # dense bind sweep
    rows += [(0, 5, 0, 10 ** 6 + 3 * k, 10 ** 6 + 3 * k + 1) for k in range(300)]   # clustered
    rows += [(0, 2, 0, int(x), 0) for x in g.integers(0, 1 << 30, size=100)]
    P = np.array(rows, dtype=synth.PRED_DTYPE)
    for host, lo, hi in ((False, 0, 1 << 30), (True, I32MIN, I32MAX)):
        _, _, bps = G.debug_buckets([0], [lo], [hi], host, P, None, [], 0, [])
        vals = _values(g, lo, hi, bps, 20000)
        assert _check_column(G, oracle, [0], [lo], [hi], host, P, None, [], 0, vals) == 0


def test_int64_columns(G, oracle):
    g = np.random.default_rng(3)
    P = np.array([(0, op, fl, a, min(a + 10, I64MAX)) for op in range(6) for fl in (0, 1)
                  for a in (I64MIN, -(1 << 40), -1, 0, 7, 1 << 50, I64MAX)], dtype=synth.PRED_DTYPE)
    for lo, hi in ((I64MIN, I64MAX), (-(1 << 40), 1 << 40), (0, 1000)):
        _, _, bps = G.debug_buckets([1], [lo], [hi], False, P, None, [], 0, [])
        vals = _values(g, lo, hi, bps)
        _check_column(G, oracle, [1], [lo], [hi], False, P, None, [], 0, vals)


def test_random_batches(G, oracle):
    g = np.random.default_rng(4)
    for trial in range(40):
        lo = int(g.integers(-10 ** 6, 10 ** 6))
        hi = lo + int(g.integers(0, 10 ** int(g.integers(1, 9))))
        k = int(g.integers(1, 300))
        a = g.integers(lo - 5, hi + 5, size=k)
        P = np.zeros(k, dtype=synth.PRED_DTYPE)
        P["op"] = g.integers(0, 6, size=k)
        P["flags"] = g.integers(0, 2, size=k)
        P["a"] = a
        P["b"] = a + g.integers(-2, max(3, (hi - lo) // 10), size=k)
        host = bool(trial % 2)
        dlo, dhi = (I32MIN, I32MAX) if host else (lo, hi)
        _, _, bps = G.debug_buckets([0], [dlo], [dhi], host, P, None, [], 0, [])
        vals = _values(g, lo, hi, bps, 3000)
        _check_column(G, oracle, [0], [dlo], [dhi], host, P, None, [], 0, vals)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5", "C5_i64"])
def test_specialised_kernel_compiles(G, name, monkeypatch):
    """The plan-specialised probe kernel (NVRTC) compiles for every workload shape, with
    and without the clustered-column path."""
    from paper_2512_19750_b200 import gace
    w = synth.get(name, 20_000)
    t = [x.numpy() for x in w.table()]
    dt = [0 if x.dtype == np.int32 else 1 for x in t]
    for rate, clustered in ((1.0, False), (0.25, False), (1.0, True)):
        if clustered:
            monkeypatch.setenv("GACE_DEBUG_CLUSTERED", "1")
        n = gace.debug_jit_compile(dt, [int(x.min()) for x in t], [int(x.max()) for x in t], False,
                                   w.preds, w.pairs, w.hll_cols, rate)
        assert n > 1000


def test_table_sizing_by_estimate(G, oracle, monkeypatch, capfd):
    """The planner sizes candidate table resolutions by estimate and builds each table once
    (gace_host.cpp lut_estimate): the plan it picks must be the one it picks by building every
    candidate (GACE_NO_LUT_ESTIMATE=1) -- same formats, shifts, cell and record counts, shared
    memory -- on batches whose tables have to be coarsened and refined to fit (four wide
    columns, hundreds of ranges, narrow ones that put two breakpoints in a cell, breakpoints on
    cell starts, pair grids taking shared memory), and every column still resolves exactly."""
    g = np.random.default_rng(11)
    for trial in range(12):
        spans = [int(10 ** g.uniform(4, 9)) for _ in range(4)]
        rows = []
        for c, sp in enumerate(spans):
            for _ in range(int(g.integers(20, 160))):
                a = int(g.integers(0, sp))
                w = int(g.choice([0, 1, 3, 100, sp // 50 + 1]))
                rows.append((c, 5, 0, a, min(a + w, sp)))
            for k in range(8):                          # on power-of-two cell starts
                rows.append((c, 2, 0, (k + 1) << int(g.integers(4, 16)), 0))
        P = np.array(rows, dtype=synth.PRED_DTYPE)
        pairs = np.array([(i, j) for i in range(0, len(P), 37) for j in range(5, len(P), 53)
                          if P["col"][i] != P["col"][j]][:64], dtype=synth.PAIR_DTYPE)
        dt, lo, hi = [0] * 4, [0] * 4, spans
        dumps = []
        for est in (True, False):
            if est:
                monkeypatch.delenv("GACE_NO_LUT_ESTIMATE", raising=False)
            else:
                monkeypatch.setenv("GACE_NO_LUT_ESTIMATE", "1")
            monkeypatch.setenv("GACE_PLAN_DUMP", "1")
            capfd.readouterr()
            G.debug_buckets(dt, lo, hi, False, P, pairs, [0, 1, 2, 3], 0, [0])
            dumps.append([l for l in capfd.readouterr().err.splitlines() if l.startswith(("slot", "smem"))])
            monkeypatch.delenv("GACE_PLAN_DUMP")
        assert dumps[0] == dumps[1] and dumps[0], dumps
        for c in range(4):
            _, _, bps = G.debug_buckets(dt, lo, hi, False, P, pairs, [0, 1, 2, 3], c, [])
            _check_column(G, oracle, dt, lo, hi, False, P, pairs, [0, 1, 2, 3], c, _values(g, 0, spans[c], bps, 3000))
