"""Pins of the oracle against things other than itself (CPU only).

Each test names what fixes the expected value: a published known answer, the
paper's thresholds, exact rational arithmetic, a closed form, an invariant of
the definition, or a statistical bound of HyperLogLog.
"""
import json
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ---------------------------------------------------------------- hash known answers

def test_splitmix64_jdk_kat(oracle):
    kat = _gold("hash_kats.json")["splitmix64"]
    want = kat["first_nextLong_signed"] & ((1 << 64) - 1)
    assert oracle.lib().oracle_u(kat["seed"], 0) == want
    assert oracle.py_u(kat["seed"], 0) == want


def test_splitmix64_is_counter_based(oracle):
    # SplittableRandom(seed): state advances by gamma, output = mix64(state); the
    # k-th output therefore equals mix64(seed + k*gamma).  Iterate the generator.
    L = oracle.lib()
    for seed in (0, 1, 42, (1 << 64) - 1):
        state = seed
        for r in range(50):
            state = (state + oracle.GAMMA) & oracle.M64
            assert L.oracle_u(seed, r) == L.oracle_mix64(state) == oracle.py_mix64(state)


def test_murmur3_fmix32_kat(oracle):
    for v in _gold("hash_kats.json")["murmur3_x86_32_empty_key"]["vectors"]:
        assert oracle.lib().oracle_fmix32(v["seed"]) == v["hash"]
        assert oracle.py_fmix32(v["seed"]) == v["hash"]


def test_c_and_python_hashes_agree(oracle):
    L = oracle.lib()
    g = np.random.default_rng(7)
    for x in g.integers(0, 1 << 63, size=2000, dtype=np.uint64):
        x = int(x) * 2 + 1
        assert L.oracle_mix64(x & oracle.M64) == oracle.py_mix64(x)
        assert L.oracle_fmix32(x & 0xFFFFFFFF) == oracle.py_fmix32(x)


# ---------------------------------------------------------------- sample threshold / keep

def test_threshold_exact(oracle):
    L = oracle.lib()
    assert L.oracle_threshold(0.0) == 0
    assert L.oracle_threshold(0.5) == 1 << 63
    assert L.oracle_threshold(0.25) == 1 << 62
    assert L.oracle_threshold(1.0 - 2.0 ** -53) == (1 << 64) - (1 << 11)
    g = np.random.default_rng(3)
    for rate in list(g.random(2000)) + [2.0 ** -60, 1e-300, 0.01, 0.1, 0.999999]:
        # exact rational floor(rate * 2^64) from the double's integer ratio
        num, den = float(rate).as_integer_ratio()
        assert L.oracle_threshold(float(rate)) == (num << 64) // den


def test_keep_rate_extremes_and_nesting(oracle):
    n = 20000
    none = oracle.sample_mask(n, 0.0, 9)
    all_ = oracle.sample_mask(n, 1.0, 9)
    assert not none.any()
    assert int(sum(bin(int(w)).count("1") for w in all_)) == n
    prev = none
    for rate in (0.001, 0.01, 0.3, 0.5, 0.9, 1.0 - 2 ** -53, 1.0):
        cur = oracle.sample_mask(n, rate, 9)
        assert np.all((prev & ~cur) == 0), "keep must be nested in rate"
        prev = cur


def test_keep_binomial(oracle):
    for n, rate, seed in ((10 ** 6, 0.01, 0), (10 ** 5, 0.5, 7), (2 * 10 ** 5, 0.1, 123)):
        bits = oracle.sample_mask(n, rate, seed)
        k = int(sum(bin(int(w)).count("1") for w in bits))
        assert abs(k - rate * n) <= 5 * math.sqrt(n * rate * (1 - rate))


def test_keep_shard_invariant(oracle):
    n = 10000
    whole = oracle.sample_mask(n, 0.3, 5)
    bits = [(int(whole[r // 64]) >> (r % 64)) & 1 for r in range(n)]
    for off in (0, 1, 63, 64, 777):
        part = oracle.sample_mask(n - off, 0.3, 5, row_offset=off)
        got = [(int(part[r // 64]) >> (r % 64)) & 1 for r in range(n - off)]
        assert got == bits[off:]


# ---------------------------------------------------------------- HLL index / rank rule

def _hll_by_string(h, width, p):
    s = format(h, f"0{width}b")
    rest = s[p:]
    return int(s[:p], 2), (rest.find("1") + 1) if "1" in rest else (width - p + 1)


def test_hll_index_rank_rule(oracle):
    g = np.random.default_rng(11)
    L = oracle.lib()
    import ctypes
    i = ctypes.c_uint32()
    r = ctypes.c_uint32()
    for x in list(g.integers(-2 ** 31, 2 ** 31, size=3000)) + [0, -1, 2 ** 31 - 1, -2 ** 31]:
        x = int(x)
        want = _hll_by_string(oracle.py_fmix32(x & 0xFFFFFFFF), 32, 12)
        assert oracle.py_hll_i32(x) == want
        L.oracle_hll_i32(x, 12, ctypes.byref(i), ctypes.byref(r))
        assert (i.value, r.value) == want
    for x in list(g.integers(-2 ** 63, 2 ** 63, size=3000, dtype=np.int64)) + [0, -1]:
        x = int(x)
        want = _hll_by_string(oracle.py_mix64((x + oracle.GAMMA) & oracle.M64), 64, 12)
        assert oracle.py_hll_i64(x) == want
        L.oracle_hll_i64(x, 12, ctypes.byref(i), ctypes.byref(r))
        assert (i.value, r.value) == want


def test_hll_rank_distribution(oracle):
    # For a good hash, P(rank = k) = 2^-k: a dropped "+1" or a wrong shift fails this.
    vals = np.arange(200000, dtype=np.int64)
    ranks = np.array([oracle.py_hll_i32(int(v))[1] for v in vals])
    for k in range(1, 7):
        frac = float(np.mean(ranks == k))
        assert abs(frac - 2.0 ** -k) < 4 * math.sqrt(2.0 ** -k / len(vals)) + 1e-3


# ---------------------------------------------------------------- NDV estimate

def test_ndv_small_exact(oracle):
    # 8 distinct int32 values landing in 8 distinct registers: linear counting gives
    # m ln(m / (m - 8)) exactly (Whang et al. 1990 linear counting, reading L5).
    regs = np.zeros(4096, dtype=np.uint8)
    for v in range(8):
        idx, rank = oracle.py_hll_i32(v)
        regs[idx] = max(regs[idx], rank)
    assert int((regs > 0).sum()) == 8
    assert oracle.ndv_est(regs) == 4096 * math.log(4096 / 4088)
    assert abs(oracle.ndv_est(regs) - 8.0) < 0.01
    assert oracle.ndv_est(np.zeros(4096, dtype=np.uint8)) == 0.0


def test_ndv_standard_error(oracle):
    # |NDV_est/NDV - 1| <= 4 sigma per set, RMS over 20 disjoint sets <= 1.5 sigma,
    # sigma = 1.04/sqrt(m) (Flajolet et al. 2007).
    sigma = 1.04 / math.sqrt(4096)
    errs = []
    for k in range(20):
        col = np.arange(k * 100000, (k + 1) * 100000, dtype=np.int32) * 7919 + 13
        _, _, _, regs = oracle.probe([col], np.zeros(0, dtype=oracle.PRED_DTYPE), hll_cols=[0])
        e = oracle.ndv_est(regs[0]) / 100000 - 1
        assert abs(e) <= 4 * sigma
        errs.append(e)
    assert math.sqrt(np.mean(np.square(errs))) <= 1.5 * sigma
    col64 = np.arange(300000, dtype=np.int64) * (1 << 33) - 5
    _, _, _, regs = oracle.probe([col64], np.zeros(0, dtype=oracle.PRED_DTYPE), hll_cols=[0])
    assert abs(oracle.ndv_est(regs[0]) / 300000 - 1) <= 4 * sigma


def test_hll_registers_depend_on_set_only(oracle):
    g = np.random.default_rng(5)
    base = g.integers(-10 ** 6, 10 ** 6, size=5000).astype(np.int32)
    dup = np.concatenate([base, base[::-1], base[:100]])
    g.shuffle(dup)
    P = np.zeros(0, dtype=oracle.PRED_DTYPE)
    r1 = oracle.probe([base], P, hll_cols=[0])[3]
    r2 = oracle.probe([dup], P, hll_cols=[0])[3]
    assert np.array_equal(r1, r2)
    a, b = base[:3000], base[2000:]
    ra = oracle.probe([a], P, hll_cols=[0])[3]
    rb = oracle.probe([b], P, hll_cols=[0])[3]
    assert np.array_equal(np.maximum(ra, rb), r1)        # merge(H(A), H(B)) = H(A u B)


# ---------------------------------------------------------------- counts / joints

def _pred(col, op, a, b=0, flags=0):
    return (col, op, flags, a, b)


def test_closed_form_mod_column(oracle):
    # x[r] = r mod V at rate 1: count(a <= x <= b) = sum_{v=a..b} (N//V + [v < N mod V]).
    for N, V in ((1000, 7), (12345, 100), (64, 64), (65, 64)):
        col = (np.arange(N) % V).astype(np.int32)
        rows = [(a, b) for a in range(-1, V + 1, 3) for b in range(a - 1, V + 2, 4)]
        P = np.array([_pred(0, oracle.BETWEEN, a, b) for a, b in rows], dtype=oracle.PRED_DTYPE)
        n, counts, _, _ = oracle.probe([col], P)
        assert n == N
        for (a, b), c in zip(rows, counts):
            want = sum(N // V + (1 if v < N % V else 0) for v in range(max(a, 0), min(b, V - 1) + 1))
            assert int(c) == want


def test_complement_tautology_empty_partition(oracle):
    g = np.random.default_rng(2)
    col = g.integers(-50, 50, size=7777).astype(np.int32)
    col64 = g.integers(-(1 << 40), 1 << 40, size=7777).astype(np.int64)
    I64MIN, I64MAX = -(1 << 63), (1 << 63) - 1
    preds = []
    for v in (-60, -50, -1, 0, 7, 49, 50):
        for op in range(5):
            preds.append(_pred(0, op, v))
            preds.append(_pred(0, op, v, flags=oracle.NEGATE))
    preds += [_pred(0, oracle.GE, I64MIN), _pred(0, oracle.LE, I64MAX), _pred(1, oracle.GE, I64MIN),
              _pred(0, oracle.BETWEEN, 1, 0), _pred(0, oracle.LT, I64MIN), _pred(1, oracle.GT, I64MAX)]
    # partition of the int32 domain: (-inf,-10), [-10,10], (10, +inf)
    preds += [_pred(0, oracle.LT, -10), _pred(0, oracle.BETWEEN, -10, 10), _pred(0, oracle.GT, 10)]
    P = np.array(preds, dtype=oracle.PRED_DTYPE)
    for rate in (1.0, 0.37):
        n, c, _, _ = oracle.probe([col, col64], P, rate=rate, seed=4)
        for k in range(0, 70, 2):
            assert int(c[k]) + int(c[k + 1]) == n
        assert list(c[70:73]) == [n, n, n]
        assert list(c[73:76]) == [0, 0, 0]
        assert int(c[76]) + int(c[77]) + int(c[78]) == n


def test_joint_invariants(oracle):
    g = np.random.default_rng(9)
    a = g.integers(0, 100, size=5000).astype(np.int32)
    b = (a + g.integers(0, 20, size=5000)).astype(np.int32)
    preds = [_pred(0, oracle.LT, 30), _pred(0, oracle.LT, 30, flags=oracle.NEGATE),
             _pred(1, oracle.BETWEEN, 10, 60), _pred(1, oracle.BETWEEN, 10, 60, flags=oracle.NEGATE),
             _pred(0, oracle.EQ, 5)]
    P = np.array(preds, dtype=oracle.PRED_DTYPE)
    pairs = [(0, 0), (0, 1), (0, 2), (0, 3), (2, 0), (4, 2), (1, 3)]
    Q = np.array(pairs, dtype=oracle.PAIR_DTYPE)
    n, c, j, _ = oracle.probe([a, b], P, Q, rate=0.8, seed=1)
    assert j[0] == c[0]                      # joint(p, p) = count(p)
    assert j[1] == 0                         # joint(p, not p) = 0
    assert j[2] + j[3] == c[0]               # joint(p, q) + joint(p, not q) = count(p)
    assert j[4] == j[2]                      # symmetric
    for (x, y), jj in zip(pairs, j):
        assert jj <= min(c[x], c[y])


def test_shard_merge_equals_whole(oracle):
    import synth
    w = synth.get("C1", 20000)
    t = [x.numpy() for x in w.table()]
    whole = oracle.probe(t, w.preds, w.pairs, rate=0.6, seed=77, hll_cols=w.hll_cols)
    cuts = [0, 1, 5000, 13331, 20000]
    parts = [oracle.probe([x[s:e] for x in t], w.preds, w.pairs, rate=0.6, seed=77,
                          hll_cols=w.hll_cols, row_offset=s) for s, e in zip(cuts, cuts[1:])]
    assert sum(p[0] for p in parts) == whole[0]
    assert np.array_equal(sum(p[1] for p in parts), whole[1])
    assert np.array_equal(sum(p[2] for p in parts), whole[2])
    assert np.array_equal(np.maximum.reduce([p[3] for p in parts]), whole[3])


def test_threads_do_not_change_results(oracle):
    import synth
    w = synth.get("C5", 30000)
    t = [x.numpy() for x in w.table()]
    r1 = oracle.probe(t, w.preds, w.pairs, hll_cols=w.hll_cols, nthreads=1)
    r8 = oracle.probe(t, w.preds, w.pairs, hll_cols=w.hll_cols, nthreads=8)
    assert r1[0] == r8[0]
    for a, b in zip(r1[1:], r8[1:]):
        assert np.array_equal(a, b)


def test_invalid_arguments_rejected(oracle):
    col = np.zeros(4, dtype=np.int32)
    with pytest.raises(oracle.OracleError):
        oracle.probe([col], np.array([_pred(1, 0, 0)], dtype=oracle.PRED_DTYPE))
    with pytest.raises(oracle.OracleError):
        oracle.probe([col], np.array([_pred(0, 9, 0)], dtype=oracle.PRED_DTYPE))
    with pytest.raises(oracle.OracleError):
        oracle.probe([col], np.array([_pred(0, 0, 0)], dtype=oracle.PRED_DTYPE),
                     np.array([(0, 1)], dtype=oracle.PAIR_DTYPE))
    for rate in (float("nan"), -0.1, 1.5):
        with pytest.raises(oracle.OracleError):
            oracle.probe([col], np.zeros(0, dtype=oracle.PRED_DTYPE), rate=rate)


# ---------------------------------------------------------------- derive and gate

def test_gate_golden(oracle):
    ex = _gold("gate_examples.json")
    for e in ex["drift"]:
        d = oracle.drift(e["ndv_hist"], e["ndv_est"])
        assert abs(d - e["D"]) <= 1e-15
        assert oracle.gate(d=[d])[0] == (oracle.SIG_DRIFT if e["fires"] else 0)
    for e in ex["pcs"]:
        pcs = e["joint"] / (e["a"] * e["b"])
        assert pcs == e["PCS"]
        assert oracle.gate(pcs=[pcs])[0] == (oracle.SIG_CORRELATION if e["fires"] else 0)
    for e in ex["sel_error"]:
        assert oracle.gate(s_est=[e["s_est"]], s_probe=[e["s_probe"]])[0] == \
            (oracle.SIG_SEL_ERROR if e["fires"] else 0)
    # exact threshold ties: PCS exactly 1.6 / 0.7 does not fire
    assert oracle.gate(pcs=[1.6, 0.7])[0] == 0
    assert oracle.gate(pcs=[float("nan")], d=[float("nan")])[0] == 0
    mask, per = oracle.gate(d=[0.3, 0.1], s_est=[0.5], s_probe=[0.2], pcs=[1.0, 1.7])
    assert mask == 7 and per == [True, False, True, False, True]


def test_derive_from_counts(oracle):
    # PCS from counts equals Eq. 3 on the probabilities; n = 0 and zero marginals are NaN.
    sel, pcs, ndv, d = oracle.derive(100, [50, 50, 0], [(0, 1), (0, 2)], [25, 0],
                                     [np.zeros(4096, dtype=np.uint8)], [10.0])
    assert sel == [0.5, 0.5, 0.0] and pcs[0] == 1.0 and math.isnan(pcs[1])
    assert ndv == [0.0] and d == [1.0]
    sel, pcs, _, _ = oracle.derive(0, [0], [(0, 0)], [0], [], [])
    assert math.isnan(sel[0]) and math.isnan(pcs[0])
    with pytest.raises(oracle.OracleError):
        oracle.drift(0.0, 1.0)


def test_percentile_golden(oracle):
    for e in _gold("gate_examples.json")["percentile_nearest_rank"]:
        xs = list(range(1, 101)) if e["xs"] == "1..100" else e["xs"]
        assert oracle.percentile_nearest_rank(xs, e["q"]) == e["value"]
