"""Oracle for the GACE selectivity probe -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It shares no code with the CUDA
product (paper_2512_19750_b200/, include/); neither imports the other.

Three independent pieces, each following the paper's definitions
(§III-C Eq. 1-3) and the readings in SURVEY.md §8(c) / DESIGN.md:

* ``probe`` -- ctypes wrapper over oracle/gace_oracle.c, the plain per-row
  C scan (fast enough for bounded samples of the full workloads).
* ``brute_probe`` -- the same definition as pure-Python loops over Python
  ints, for tiny tables.  It is written separately from the C scan so the two
  pin each other (tests/test_oracle_bruteforce.py).
* ``probe_sets`` / ``brute_probe_sets`` -- candidate-set conjunction counts
  (§IV-H Exp. D, lines 250-270), C scan and
  pure-Python loops, pinned by tests/test_oracle_sets.py.
* ``derive`` / ``ndv_est`` / ``gate`` -- the host-side double arithmetic:
  S_probe = count / n (reading L13), PCS = P(A,B) / (P(A) P(B)) in the literal
  Eq. 3 order (L14), HLL raw + linear-counting estimate (L5), drift D (Eq. 1)
  and the three gate inequalities (Eq. 1-3 thresholds, L16).

Parity notes: ``probe`` / ``brute_probe`` are pinned (KATs, brute force,
closed forms, invariants); ``ndv_est`` is pinned by the exact small-set value
and the HLL standard-error bound; ``derive`` / ``gate`` by the paper's
thresholds and SPEC.md's worked examples (tests/golden/).
"""
from __future__ import annotations

import ctypes
import math
import os
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgace_oracle.so")

M64 = (1 << 64) - 1
GAMMA = 0x9E3779B97F4A7C15

EQ, LT, LE, GT, GE, BETWEEN = 0, 1, 2, 3, 4, 5
NEGATE = 1
I32, I64 = 0, 1

SIG_DRIFT, SIG_SEL_ERROR, SIG_CORRELATION = 1, 2, 4

PRED_DTYPE = np.dtype([("col", "<u4"), ("op", "<u2"), ("flags", "<u2"), ("a", "<i8"), ("b", "<i8")])
PAIR_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4")])


# ----------------------------------------------------------------------------- build / load

def build(force: bool = False) -> str:
    """Compile the C oracle (gcc + OpenMP).  Building the checker is not using it."""
    src = os.path.join(_HERE, "gace_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        cmd = f"gcc -O2 -fopenmp -ffp-contract=off -shared -fPIC -o {LIB_PATH} {src} -lm"
        if os.system(cmd) != 0:
            raise RuntimeError("oracle build failed: " + cmd)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_mix64.restype = ctypes.c_uint64
        L.oracle_mix64.argtypes = [ctypes.c_uint64]
        L.oracle_u.restype = ctypes.c_uint64
        L.oracle_u.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_threshold.restype = ctypes.c_uint64
        L.oracle_threshold.argtypes = [ctypes.c_double]
        L.oracle_keep.restype = ctypes.c_int
        L.oracle_keep.argtypes = [ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64]
        L.oracle_fmix32.restype = ctypes.c_uint32
        L.oracle_fmix32.argtypes = [ctypes.c_uint32]
        for f, t in ((L.oracle_hll_i32, ctypes.c_int32), (L.oracle_hll_i64, ctypes.c_int64)):
            f.restype = None
            f.argtypes = [t, ctypes.c_int, ctypes.POINTER(ctypes.c_uint32), ctypes.POINTER(ctypes.c_uint32)]
        L.oracle_probe.restype = ctypes.c_int
        L.oracle_probe.argtypes = [
            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int), ctypes.c_uint32,
            ctypes.c_uint64, ctypes.c_uint64,
            ctypes.c_void_p, ctypes.c_uint32, ctypes.c_void_p, ctypes.c_uint32,
            ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_probe_sets.restype = ctypes.c_int
        L.oracle_probe_sets.argtypes = [
            ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int), ctypes.c_uint32,
            ctypes.c_uint64, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_uint32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_uint32,
            ctypes.c_double, ctypes.c_uint64, ctypes.c_int,
            ctypes.POINTER(ctypes.c_uint64), ctypes.c_void_p]
        L.oracle_sample_mask.restype = ctypes.c_int
        L.oracle_sample_mask.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_double,
                                         ctypes.c_uint64, ctypes.c_void_p]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------- C scan wrapper

class OracleError(ValueError):
    pass


def _as_preds(preds) -> np.ndarray:
    a = np.ascontiguousarray(preds)
    if a.dtype != PRED_DTYPE:
        a = a.astype(PRED_DTYPE)
    return a


def _as_pairs(pairs) -> np.ndarray:
    if pairs is None or len(pairs) == 0:
        return np.zeros(0, dtype=PAIR_DTYPE)
    a = np.ascontiguousarray(pairs)
    if a.dtype != PAIR_DTYPE:
        a = a.astype(PAIR_DTYPE)
    return a


def probe(columns: Sequence[np.ndarray], preds, pairs=None, rate: float = 1.0, seed: int = 0,
          hll_cols: Sequence[int] = (), hll_p: int = 12, row_offset: int = 0, nthreads: int = 0):
    """C oracle scan over host numpy columns (int32 / int64).

    Returns (n_sampled, counts u64[P], joints u64[Q], regs u8[len(hll_cols), 2^p])."""
    cols = [np.ascontiguousarray(c) for c in columns]
    if not cols:
        raise OracleError("no columns")
    nrows = len(cols[0])
    dtypes = []
    for c in cols:
        if len(c) != nrows:
            raise OracleError("ragged columns")
        if c.dtype == np.int32:
            dtypes.append(I32)
        elif c.dtype == np.int64:
            dtypes.append(I64)
        else:
            raise OracleError(f"unsupported dtype {c.dtype}")
    P = _as_preds(preds)
    Q = _as_pairs(pairs)
    mask = 0
    for c in hll_cols:
        mask |= 1 << int(c)
    nh = len(set(int(c) for c in hll_cols))
    counts = np.zeros(max(len(P), 1), dtype=np.uint64)
    joints = np.zeros(max(len(Q), 1), dtype=np.uint64)
    regs = np.zeros((max(nh, 1), 1 << hll_p), dtype=np.uint8)
    ptrs = (ctypes.c_void_p * len(cols))(*[c.ctypes.data for c in cols])
    dt = (ctypes.c_int * len(cols))(*dtypes)
    n = ctypes.c_uint64(0)
    rc = lib().oracle_probe(ptrs, dt, len(cols), nrows, row_offset,
                            P.ctypes.data if len(P) else None, len(P),
                            Q.ctypes.data if len(Q) else None, len(Q),
                            float(rate), seed & M64, mask, hll_p, nthreads,
                            ctypes.byref(n), counts.ctypes.data, joints.ctypes.data, regs.ctypes.data)
    if rc != 0:
        raise OracleError("oracle_probe rejected its arguments")
    return int(n.value), counts[:len(P)], joints[:len(Q)], regs[:nh]


def sets_csr(sets) -> tuple[np.ndarray, np.ndarray]:
    """A list of member-index lists -> (offsets u32[M+1], members u32[...])."""
    offs = [0]
    mem: list[int] = []
    for s in sets:
        mem.extend(int(i) for i in s)
        offs.append(len(mem))
    return np.asarray(offs, dtype=np.uint32), np.asarray(mem, dtype=np.uint32)


def probe_sets(columns: Sequence[np.ndarray], preds, sets, rate: float = 1.0, seed: int = 0,
               row_offset: int = 0, nthreads: int = 0):
    """C oracle of the candidate-set conjunction counts (§IV-H Exp. D, lines
    250-270): set_counts[m] = #{kept r : every member predicate of set m holds on row r}.

    ``sets``: list of member-index lists.  Returns (n_sampled, set_counts u64[M])."""
    cols = [np.ascontiguousarray(c) for c in columns]
    nrows = len(cols[0])
    dtypes = [I32 if c.dtype == np.int32 else I64 for c in cols]
    for c in cols:
        if c.dtype not in (np.int32, np.int64) or len(c) != nrows:
            raise OracleError("columns must be int32 / int64 of equal length")
    P = _as_preds(preds)
    offs, mem = sets_csr(sets)
    out = np.zeros(max(len(sets), 1), dtype=np.uint64)
    ptrs = (ctypes.c_void_p * len(cols))(*[c.ctypes.data for c in cols])
    dt = (ctypes.c_int * len(cols))(*dtypes)
    n = ctypes.c_uint64(0)
    rc = lib().oracle_probe_sets(ptrs, dt, len(cols), nrows, row_offset,
                                 P.ctypes.data if len(P) else None, len(P),
                                 offs.ctypes.data, mem.ctypes.data if len(mem) else None, len(sets),
                                 float(rate), seed & M64, nthreads, ctypes.byref(n), out.ctypes.data)
    if rc != 0:
        raise OracleError("oracle_probe_sets rejected its arguments")
    return int(n.value), out[:len(sets)]


def sample_mask(nrows: int, rate: float, seed: int, row_offset: int = 0) -> np.ndarray:
    bits = np.zeros(max(1, (nrows + 63) // 64), dtype=np.uint64)
    if lib().oracle_sample_mask(nrows, row_offset, float(rate), seed & M64, bits.ctypes.data) != 0:
        raise OracleError("bad rate")
    return bits[:(nrows + 63) // 64]


# ----------------------------------------------------------------------------- pure Python definitions

def py_mix64(z: int) -> int:
    """SplitMix64 finaliser, Python ints."""
    z &= M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def py_u(seed: int, r: int) -> int:
    return py_mix64((seed + (r + 1) * GAMMA) & M64)


def py_threshold(rate: float) -> int:
    """floor(rate * 2^64) exactly, via the rational value of the double."""
    num, den = float(rate).as_integer_ratio()
    return (num << 64) // den


def py_keep(rate: float, seed: int, r: int) -> bool:
    if rate == 1.0:
        return True
    return py_u(seed, r) < py_threshold(rate)


def py_fmix32(h: int) -> int:
    h &= 0xFFFFFFFF
    h ^= h >> 16
    h = (h * 0x85EBCA6B) & 0xFFFFFFFF
    h ^= h >> 13
    h = (h * 0xC2B2AE35) & 0xFFFFFFFF
    h ^= h >> 16
    return h


def _lz(w: int, width: int) -> int:
    return width - w.bit_length()


def py_hll_i32(x: int, p: int = 12):
    h = py_fmix32(x & 0xFFFFFFFF)
    w = (h << p) & 0xFFFFFFFF
    return h >> (32 - p), (32 - p + 1) if w == 0 else _lz(w, 32) + 1


def py_hll_i64(x: int, p: int = 12):
    h = py_mix64((x + GAMMA) & M64)
    w = (h << p) & M64
    return h >> (64 - p), (64 - p + 1) if w == 0 else _lz(w, 64) + 1


def py_pred(op: int, flags: int, a: int, b: int, v: int) -> bool:
    if op == EQ:
        t = v == a
    elif op == LT:
        t = v < a
    elif op == LE:
        t = v <= a
    elif op == GT:
        t = v > a
    elif op == GE:
        t = v >= a
    elif op == BETWEEN:
        t = a <= v <= b
    else:
        raise OracleError("op")
    return (not t) if (flags & NEGATE) else t


def brute_probe(columns: Sequence[Sequence[int]], dtypes: Sequence[int], preds, pairs=(),
                rate: float = 1.0, seed: int = 0, hll_cols: Sequence[int] = (), hll_p: int = 12,
                row_offset: int = 0):
    """Pure-Python loops over the definition (tiny tables only)."""
    nrows = len(columns[0]) if columns else 0
    P = [(int(p["col"]), int(p["op"]), int(p["flags"]), int(p["a"]), int(p["b"])) for p in preds] \
        if isinstance(preds, np.ndarray) else list(preds)
    Q = [(int(q["i"]), int(q["j"])) for q in pairs] if isinstance(pairs, np.ndarray) else list(pairs)
    hcols = sorted(set(int(c) for c in hll_cols))
    m = 1 << hll_p
    n = 0
    counts = [0] * len(P)
    joints = [0] * len(Q)
    regs = [[0] * m for _ in hcols]
    for r in range(nrows):
        if not py_keep(rate, seed, row_offset + r):
            continue
        n += 1
        bits = []
        for (c, op, fl, a, b) in P:
            t = py_pred(op, fl, a, b, int(columns[c][r]))
            bits.append(t)
            counts[len(bits) - 1] += int(t)
        for k, (i, j) in enumerate(Q):
            joints[k] += int(bits[i] and bits[j])
        for k, c in enumerate(hcols):
            x = int(columns[c][r])
            idx, rank = py_hll_i32(x, hll_p) if dtypes[c] == I32 else py_hll_i64(x, hll_p)
            regs[k][idx] = max(regs[k][idx], rank)
    return n, counts, joints, regs


def brute_probe_sets(columns: Sequence[Sequence[int]], preds, sets, rate: float = 1.0, seed: int = 0,
                     row_offset: int = 0):
    """Pure-Python conjunction counts (tiny tables only): written apart from the C scan so
    the two pin each other."""
    nrows = len(columns[0]) if columns else 0
    P = [(int(p["col"]), int(p["op"]), int(p["flags"]), int(p["a"]), int(p["b"])) for p in preds] \
        if isinstance(preds, np.ndarray) else list(preds)
    n = 0
    out = [0] * len(sets)
    for r in range(nrows):
        if not py_keep(rate, seed, row_offset + r):
            continue
        n += 1
        for m, members in enumerate(sets):
            out[m] += int(all(py_pred(P[i][1], P[i][2], P[i][3], P[i][4], int(columns[P[i][0]][r]))
                              for i in members))
    return n, out


# ----------------------------------------------------------------------------- derive and gate

def hll_alpha(m: int) -> float:
    return 0.7213 / (1.0 + 1.079 / m)


def ndv_est(regs: Sequence[int]) -> float:
    """HLL estimate (reading L5): Z = sum_j 2^-R[j] in ascending j; E = alpha m^2 / Z;
    linear counting m ln(m/V) when E <= 2.5 m and V = #{R[j] = 0} > 0; no large-range term."""
    m = len(regs)
    z = 0.0
    v = 0
    for r in regs:
        z += 2.0 ** (-int(r))
        if int(r) == 0:
            v += 1
    e = hll_alpha(m) * m * m / z
    if e <= 2.5 * m and v > 0:
        return m * math.log(m / v)
    return e


def drift(ndv_hist: float, ndv_estimate: float) -> float:
    """PAPER.md Eq. 1: D = |NDV_hist - NDV_est| / NDV_hist."""
    if not ndv_hist > 0:
        raise OracleError("ndv_hist must be > 0 (SPEC.md S:209)")
    return abs(ndv_hist - ndv_estimate) / ndv_hist


def derive(n: int, counts, pairs, joints, regs_list, ndv_hist):
    """S_p, PCS_q, NDV_est_c, D_c in double."""
    nan = float("nan")
    sel = [(float(c) / float(n)) if n > 0 else nan for c in counts]
    Q = [(int(q["i"]), int(q["j"])) for q in pairs] if isinstance(pairs, np.ndarray) else list(pairs)
    pcs = []
    for (i, j), jc in zip(Q, joints):
        if n == 0 or int(counts[i]) == 0 or int(counts[j]) == 0:
            pcs.append(nan)
            continue
        fn = float(n)
        pcs.append((float(jc) / fn) / ((float(counts[i]) / fn) * (float(counts[j]) / fn)))
    ndv = [ndv_est(r) for r in regs_list]
    d = [drift(h, e) for h, e in zip(ndv_hist, ndv)]
    return sel, pcs, ndv, d


DEFAULT_THRESHOLDS = {"d": 0.25, "sel_err": 0.01, "pcs_high": 1.6, "pcs_low": 0.7}


def gate(d=(), s_est=(), s_probe=(), pcs=(), th=None):
    """Risky Gate (§III-A, Eq. 1-3 thresholds): DRIFT iff D >= 0.25, SEL_ERROR iff
    |S_est - S_probe| > 0.01, CORRELATION iff PCS > 1.6 or PCS < 0.7.  NaN never fires.
    Returns (mask, per-signal list of bools in the order d, sel, pcs)."""
    th = dict(DEFAULT_THRESHOLDS, **(th or {}))
    per = []
    mask = 0
    for x in d:
        f = bool(x >= th["d"])                       # NaN compares false
        per.append(f)
        mask |= SIG_DRIFT if f else 0
    for se, sp in zip(s_est, s_probe):
        f = bool(abs(se - sp) > th["sel_err"])
        per.append(f)
        mask |= SIG_SEL_ERROR if f else 0
    for x in pcs:
        f = bool(x > th["pcs_high"] or x < th["pcs_low"])
        per.append(f)
        mask |= SIG_CORRELATION if f else 0
    return mask, per


def percentile_nearest_rank(xs: Sequence[float], q: float) -> float:
    """value at index ceil(q n) of the ascending sort (1-based)."""
    if not xs or not (0 < q <= 1):
        raise OracleError("percentile")
    s = sorted(xs)
    return s[max(1, math.ceil(q * len(s))) - 1]


# ----------------------------------------------------------------------------- break-even cost accounting

NO_RISK, RISK_BUT_NOT_WORTH, PROBE = 0, 1, 2


def probe_cost(c0: float, ct: float, ce: float, p: float, n: float, k: float, m: float) -> float:
    """est_probe_cost_ms = c0 + c_t*N + c_e*K*M*N/p (Eq. 4 models the
    measurement cost from the measured kernel time, line 80-83)."""
    return c0 + ct * n + ce * k * m * n / p


def cost_fit(n, k, m, ms, p: float = 1.0):
    """Least-squares fit of (c0, c_t, c_e) >= 0 to measured probe times (SPEC.md S:232-235
    calibrate_cost_model; coefficients >= 0).  Every non-negativity active set of the
    3 coefficients is solved by numpy lstsq and the feasible one with the least squared
    residual wins (brute force over the 7 non-empty subsets in mask order; the all-zero model
    is the start; a later subset replaces the best only if its residual is smaller by more than
    1e-9 of sum(ms^2), so near-ties -- collinear columns -- keep the earlier subset)."""
    n, k, m, ms = (np.asarray(x, dtype=np.float64) for x in (n, k, m, ms))
    X = np.stack([np.ones_like(n), n, k * m * n / p], axis=1)
    tss = float(np.sum(ms * ms))
    best = (tss, np.zeros(3))
    for mask in range(1, 8):
        cols = [j for j in range(3) if mask >> j & 1]
        sol, *_ = np.linalg.lstsq(X[:, cols], ms, rcond=None)
        if np.any(sol < 0):
            continue
        coef = np.zeros(3)
        coef[cols] = sol
        r = float(np.sum((X @ coef - ms) ** 2))
        if r < best[0] - 1e-9 * tss:
            best = (r, coef)
    c0, ct, ce = (float(x) for x in best[1])
    return c0, ct, ce


def gate_decide(fired_mask: int, c0: float, ct: float, ce: float, p: float, benefit_weight: float,
                n: float, k: float, m: float, plan_cost_spread_ms: float):
    """GateDecision: est_benefit = weight x plan-cost spread (the
    SPEC's reading); probe iff some signal fired and est_benefit > est_cost; reason
    NO_RISK (nothing fired), RISK_BUT_NOT_WORTH (fired, not worth it), PROBE."""
    cost = probe_cost(c0, ct, ce, p, n, k, m)
    benefit = benefit_weight * plan_cost_spread_ms
    if not fired_mask:
        return cost, benefit, False, NO_RISK
    if benefit > cost:
        return cost, benefit, True, PROBE
    return cost, benefit, False, RISK_BUT_NOT_WORTH


# ----------------------------------------------------------------------------- Est.CV (Exp. B)

def cv(xs) -> float:
    """Coefficient of variation: sample standard deviation (R - 1) / mean;
    mean 0 or a NaN sample -> NaN.  Loops written out in the order sum, mean, squares."""
    R = len(xs)
    mean = 0.0
    for x in xs:
        mean += x
    mean /= float(R)
    ss = 0.0
    for x in xs:
        ss += (x - mean) * (x - mean)
    sd = math.sqrt(ss / float(R - 1))
    return float("nan") if mean == 0.0 else sd / mean


def estimate_cv(columns, preds, pairs, rate: float, seeds, row_offset: int = 0):
    """Est.CV over seeded probes (§IV-C Exp. B, lines 121-141):
    per predicate the CV of S = count/n, per pair the CV of J/n and of PCS (Eq. 3), over one
    oracle probe per seed."""
    if len(seeds) < 2:
        raise OracleError("Est.CV needs >= 2 seeds")
    P = _as_preds(preds)
    Q = _as_pairs(pairs)
    sel, js, pcs = [], [], []
    for s in seeds:
        n, c, j, _ = probe(columns, P, Q, rate=rate, seed=s, row_offset=row_offset)
        sp, pq, _, _ = derive(n, c, Q, j, [], [])
        sel.append(sp)
        js.append([(float(x) / float(n)) if n > 0 else float("nan") for x in j])
        pcs.append(pq)
    cs = [cv([sel[r][p] for r in range(len(seeds))]) for p in range(len(P))]
    cj = [cv([js[r][q] for r in range(len(seeds))]) for q in range(len(Q))]
    cp = [cv([pcs[r][q] for r in range(len(seeds))]) for q in range(len(Q))]
    return cs, cj, cp


# ----------------------------------------------------------------------------- probe cache (§V item 3)

class CacheModel:
    """Plain model of the probe cache (§V item 3, line 314):
    key = (table, sorted set of (col, op, flags, bucket(a), bucket(b) if BETWEEN else 0));
    bucket = exact bind, or the equal-width range bucket of [lo, hi] split in `buckets`
    (-1 below, `buckets` above); FIFO eviction of the least recently inserted key."""

    def __init__(self, capacity: int = 4096, buckets: int = 0):
        self.capacity = capacity or 4096
        self.buckets = buckets
        self.entries = {}           # key -> [s, count, n, hits]
        self.order = []             # keys, oldest insertion first
        self.hits = self.misses = self.evictions = 0

    def _bucket(self, x, dom):
        if not self.buckets or dom is None:
            return x
        lo, hi = dom
        if x < lo:
            return -1
        if x > hi:
            return self.buckets
        from fractions import Fraction
        b = int(Fraction(x - lo) * self.buckets / Fraction(hi - lo + 1))
        return min(max(b, 0), self.buckets - 1)

    def key(self, table, conj, domains=None):
        items = set()
        for i, p in enumerate(conj):
            col, op, fl, a, b = (int(p[f]) for f in ("col", "op", "flags", "a", "b"))
            dom = None if domains is None else (int(domains[i][0]), int(domains[i][1]))
            items.add((col, op, fl, self._bucket(a, dom), self._bucket(b, dom) if op == BETWEEN else 0))
        return (int(table), tuple(sorted(items)))

    def put(self, table, conj, s, count=0, n=0, domains=None):
        k = self.key(table, conj, domains)
        if k in self.entries:
            self.order.remove(k)
        self.entries[k] = [float(s), int(count), int(n), 0]
        self.order.append(k)
        while len(self.entries) > self.capacity:
            old = self.order.pop(0)
            del self.entries[old]
            self.evictions += 1

    def lookup(self, table, conj, domains=None):
        k = self.key(table, conj, domains)
        if k not in self.entries:
            self.misses += 1
            return None
        self.hits += 1
        e = self.entries[k]
        e[3] += 1
        return tuple(e)

    def invalidate(self, table):
        for k in [k for k in self.entries if k[0] == int(table)]:
            del self.entries[k]
            self.order.remove(k)
