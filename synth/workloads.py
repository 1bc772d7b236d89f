"""Synthetic probe workloads C1..C5 (BASELINE.json configs[0..4]).

Inputs only: table columns (seeded, counter-based via ``synth.rng``) and
predicate / pair batches (seeded numpy).  No probe arithmetic lives here.

The predicate record layout is the C-ABI's ``gace_pred`` (include/gace.h):
``{u32 col; u16 op; u16 flags; i64 a; i64 b}`` = 24 bytes, and a pair is
``{u32 i; u32 j}``.  The op codes are the interface's, restated here so that
this module imports neither the product nor the oracle.

Shapes:
  C1  1M rows; status Zipf(1.2, 8) (§IV-A "orders" table, s=1.2),
      day correlated with status (rho=0.8), u1 U[0,1e6), u2 U[int32];
      16 predicates (4 per column), 4 pairs, HLL on all 4, rate 1.
  C2  TPC-H SF10 lineitem-shaped keys (59,986,052 rows), 256 BETWEEN
      predicates (64 per column), no pairs, no HLL, Bernoulli rate 0.01.
  C3  100M rows, one Zipf(1.2, 2^20) column, 1024 EQ bind sweep v=0..1023
      (variant "C3B": strided binds v=1024*j), HLL on, rate 1.
  C4  200M rows, 4 correlated pairs (a_k, b_k), rho=(0, .5, .9, .99) over
      U[0,2^16); 128 BETWEEN windows, 64 aligned pairs, HLL on all 8.
  C5  TPC-H SF100 lineitem-shaped keys (600,037,902 rows), 256 BETWEEN
      predicates, 64 pairs over 4 column pairs, HLL on all 4, rate 1.
      ("C5_i64": orderkey and partkey stored as int64.)
  D   Exp. D (§IV-H): C5's table, a 64-predicate pool, M=16 candidate
      sets of K=16 members (conjunction counts; "D_m1_k16": M=1).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable

import numpy as np
import torch

from . import rng

PRED_DTYPE = np.dtype([("col", "<u4"), ("op", "<u2"), ("flags", "<u2"), ("a", "<i8"), ("b", "<i8")])
PAIR_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4")])
assert PRED_DTYPE.itemsize == 24 and PAIR_DTYPE.itemsize == 8

EQ, LT, LE, GT, GE, BETWEEN = 0, 1, 2, 3, 4, 5
NEGATE = 1

INT32_MIN, INT32_MAX = -(2 ** 31), 2 ** 31 - 1

SF10_ROWS = 59_986_052
SF100_ROWS = 600_037_902


@dataclass
class Column:
    name: str
    dtype: str                      # "i32" | "i64"
    gen: Callable[[torch.Tensor], torch.Tensor]   # global row ids (int64) -> int64 values
    lo: int                         # value domain, for drawing predicate widths
    hi: int

    @property
    def torch_dtype(self):
        return torch.int32 if self.dtype == "i32" else torch.int64

    @property
    def width(self) -> int:
        return 4 if self.dtype == "i32" else 8


@dataclass
class Workload:
    name: str
    nrows: int
    columns: list[Column]
    preds: np.ndarray
    pairs: np.ndarray
    hll_cols: list[int]
    rate: float = 1.0
    sample_seed: int = 0
    ndv_hist: list[float] = field(default_factory=list)   # one per hll column
    s_est: list[float] = field(default_factory=list)      # optimizer S_est per predicate
    sets: list[list[int]] = field(default_factory=list)   # candidate sets (member predicate indices)

    @property
    def hll_mask(self) -> int:
        m = 0
        for c in self.hll_cols:
            m |= 1 << c
        return m

    @property
    def probed_cols(self) -> list[int]:
        cols = set(int(c) for c in self.preds["col"]) | set(self.hll_cols)
        return sorted(cols)

    @property
    def bytes_per_row(self) -> int:
        """Algorithmic bytes per table row: each probed key read once."""
        return sum(self.columns[c].width for c in self.probed_cols)

    def column(self, c: int, r0: int = 0, r1: int | None = None, device="cpu",
               chunk: int = 1 << 25, out: torch.Tensor | None = None) -> torch.Tensor:
        """Rows [r0, r1) of column c (global row ids), generated on ``device``."""
        r1 = self.nrows if r1 is None else r1
        col = self.columns[c]
        n = r1 - r0
        if out is None:
            out = torch.empty(n, dtype=col.torch_dtype, device=device)
        for s in range(0, n, chunk):
            e = min(n, s + chunk)
            idx = torch.arange(r0 + s, r0 + e, dtype=torch.int64, device=device)
            out[s:e] = col.gen(idx).to(col.torch_dtype)
        return out

    def table(self, r0: int = 0, r1: int | None = None, device="cpu") -> list[torch.Tensor]:
        return [self.column(c, r0, r1, device) for c in range(len(self.columns))]

    def values_at(self, c: int, rows: np.ndarray) -> np.ndarray:
        idx = torch.as_tensor(np.asarray(rows, dtype=np.int64))
        return self.columns[c].gen(idx).numpy()


# --------------------------------------------------------------------------- columns

_zipf_cdf_cache: dict = {}


def _zipf_cdf(n: int, s: float) -> np.ndarray:
    key = (n, s)
    if key not in _zipf_cdf_cache:
        w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
        cdf = np.cumsum(w) / w.sum()
        cdf[-1] = 2.0                     # u < 1 always lands on a rank <= n
        _zipf_cdf_cache[key] = cdf
    return _zipf_cdf_cache[key]


def zipf_share(n: int, s: float, rank: int = 1) -> float:
    """Theoretical frequency of the rank-`rank` value of Zipf(s, n)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    return float(w[rank - 1] / w.sum())


def zipf_col(seed: int, stream: str, n: int, s: float) -> Callable:
    """v = rank - 1 of Zipf(s, n) by inverse CDF (SPEC.md gen_zipf_column)."""
    def gen(idx: torch.Tensor) -> torch.Tensor:
        cdf = torch.as_tensor(_zipf_cdf(n, s), device=idx.device)
        u = rng.uniform_f64(seed, stream, idx)
        return torch.searchsorted(cdf, u, right=True).to(torch.int64)
    return gen


def uniform_col(seed: int, stream: str, lo: int, hi: int) -> Callable:
    def gen(idx):
        return rng.uniform_int(seed, stream, idx, lo, hi)
    return gen


def correlated_col(seed: int, stream: str, base: Callable, rho: float, fn: Callable,
                   lo: int, hi: int) -> Callable:
    """out = fn(base) w.p. rho else U[lo, hi] (SPEC.md gen_correlated_column)."""
    def gen(idx):
        b = base(idx)
        coin = rng.uniform_f64(seed, stream + ".coin", idx) < rho
        other = rng.uniform_int(seed, stream + ".other", idx, lo, hi)
        return torch.where(coin, fn(b), other)
    return gen


def lineitem_cols(seed: int, sf: int, nrows: int, i64: bool = False) -> list[Column]:
    """TPC-H-lineitem-shaped key columns, counter-based.

    order index o = r // 4 (4 lines per order on average, clustered);
    l_orderkey = sparse TPC-H keys, 8 used of every 32: (o//8)*32 + o%8 + 1;
    l_partkey  = U[1, 200000*SF];
    l_suppkey  = TPC-H's supplier of the part: (p + i*(S/4 + (p-1)/S)) % S + 1, i in 0..3;
    l_shipdate = orderdate(o) + U[1, 121], orderdate = 8035 + U[0, 2405] (days).
    """
    P = 200_000 * sf
    S = 10_000 * sf

    def orderkey(idx):
        o = idx // 4
        return (o // 8) * 32 + (o % 8) + 1

    def partkey(idx):
        return rng.uniform_int(seed, "partkey", idx, 1, P)

    def suppkey(idx):
        p = partkey(idx)
        i = rng.uniform_int(seed, "supp_i", idx, 0, 3)
        return (p + i * (S // 4 + (p - 1) // S)) % S + 1

    def shipdate(idx):
        o = idx // 4
        od = 8035 + rng.uniform_int(seed, "orderdate", o, 0, 2405)
        return od + rng.uniform_int(seed, "shipdelay", idx, 1, 121)

    max_ok = int(orderkey(torch.tensor([max(nrows - 1, 0)]))[0])
    t = "i64" if i64 else "i32"
    return [
        Column("l_orderkey", t, orderkey, 1, max(max_ok, 2)),
        Column("l_partkey", t, partkey, 1, P),
        Column("l_suppkey", "i32", suppkey, 1, S),
        Column("l_shipdate", "i32", shipdate, 8036, 8035 + 2405 + 121),
    ]


# --------------------------------------------------------------------------- predicates

def _preds(rows) -> np.ndarray:
    a = np.zeros(len(rows), dtype=PRED_DTYPE)
    for k, (c, op, fl, x, y) in enumerate(rows):
        a[k] = (c, op, fl, x, y)
    return a


def _pairs(rows) -> np.ndarray:
    a = np.zeros(len(rows), dtype=PAIR_DTYPE)
    for k, (i, j) in enumerate(rows):
        a[k] = (i, j)
    return a


def _log_uniform_width(g: np.random.Generator, wmax: int) -> int:
    wmax = max(1, wmax)
    return int(min(wmax, max(1, math.floor(math.exp(g.uniform(0.0, math.log(wmax + 1)))))))


def _between_batch(w: Workload, g: np.random.Generator, cols: list[int], per_col: int):
    """`per_col` BETWEEN predicates per column: lo drawn from the data (a random
    row's value), width log-uniform in [1, domain/2]."""
    rows = []
    for c in cols:
        col = w.columns[c]
        los = w.values_at(c, g.integers(0, w.nrows, size=per_col))
        dom = col.hi - col.lo + 1
        for lo in los:
            wd = _log_uniform_width(g, dom // 2)
            rows.append((c, BETWEEN, 0, int(lo), int(lo) + wd - 1))
    return rows


def make_c1(nrows: int = 1_000_000, data_seed: int = 1, pred_seed: int = 101) -> Workload:
    status = zipf_col(data_seed, "status", 8, 1.2)
    day = correlated_col(data_seed, "day", status, 0.8, lambda b: 45 * b, 0, 364)
    cols = [
        Column("status", "i32", status, 0, 7),
        Column("day", "i32", day, 0, 364),
        Column("u1", "i32", uniform_col(data_seed, "u1", 0, 999_999), 0, 999_999),
        Column("u2", "i32", uniform_col(data_seed, "u2", INT32_MIN, INT32_MAX), INT32_MIN, INT32_MAX),
    ]
    w = Workload("C1", nrows, cols, _preds([]), _pairs([]), [0, 1, 2, 3])
    g = np.random.default_rng(pred_seed)
    rows = []
    for c in range(4):
        col = cols[c]
        v = w.values_at(c, g.integers(0, nrows, size=4))
        dom = col.hi - col.lo + 1
        wd = _log_uniform_width(g, dom // 2)
        rows += [(c, EQ, 0, int(v[0]), 0), (c, LT, 0, int(v[1]), 0),
                 (c, GE, 0, int(v[2]), 0), (c, BETWEEN, 0, int(v[3]), int(v[3]) + wd - 1)]
    w.preds = _preds(rows)
    # 2x (status, day) Q_SC-style (§IV-A), (u1, u2), (status, u1)
    w.pairs = _pairs([(0, 7), (1, 6), (11, 15), (3, 8)])
    w.ndv_hist = [8.0, 365.0, 632_000.0, 1_000_000.0]
    w.s_est = [1.0 / 8] * 16
    return w


def make_c2(nrows: int = SF10_ROWS, data_seed: int = 2, pred_seed: int = 202) -> Workload:
    cols = lineitem_cols(data_seed, 10, nrows)
    w = Workload("C2", nrows, cols, _preds([]), _pairs([]), [], rate=0.01, sample_seed=0x5EED)
    g = np.random.default_rng(pred_seed)
    w.preds = _preds(_between_batch(w, g, [0, 1, 2, 3], 64))
    return w


def make_c3(nrows: int = 100_000_000, data_seed: int = 3, variant: str = "A") -> Workload:
    cols = [Column("k", "i32", zipf_col(data_seed, "zipf", 1 << 20, 1.2), 0, (1 << 20) - 1)]
    binds = range(1024) if variant == "A" else range(0, 1024 * 1024, 1024)
    w = Workload("C3" if variant == "A" else "C3B", nrows, cols,
                 _preds([(0, EQ, 0, v, 0) for v in binds]), _pairs([]), [0])
    w.ndv_hist = [float(1 << 20)]
    return w


C4_RHO = (0.0, 0.5, 0.9, 0.99)


def make_c4(nrows: int = 200_000_000, data_seed: int = 4, pred_seed: int = 404) -> Workload:
    cols = []
    for k, rho in enumerate(C4_RHO):
        a = uniform_col(data_seed, f"a{k}", 0, 65535)
        b = correlated_col(data_seed, f"b{k}", a, rho, lambda x: x, 0, 65535)
        cols += [Column(f"a{k}", "i32", a, 0, 65535), Column(f"b{k}", "i32", b, 0, 65535)]
    w = Workload("C4", nrows, cols, _preds([]), _pairs([]), list(range(8)))
    g = np.random.default_rng(pred_seed)
    rows, pairs = [], []
    for k in range(4):
        wins = []
        for e in range(1, 9):                       # width fraction 2^-e
            wd = 65536 >> e
            for _ in range(2):                      # two offsets
                lo = int(g.integers(0, 65536 - wd + 1))
                wins.append((lo, lo + wd - 1))
        base_a = len(rows)
        rows += [(2 * k, BETWEEN, 0, lo, hi) for lo, hi in wins]
        base_b = len(rows)
        rows += [(2 * k + 1, BETWEEN, 0, lo, hi) for lo, hi in wins]
        pairs += [(base_a + i, base_b + i) for i in range(16)]
    w.preds, w.pairs = _preds(rows), _pairs(pairs)
    w.ndv_hist = [65536.0, 49152.0, 32768.0, 131072.0] * 2
    w.s_est = [float(p["b"] - p["a"] + 1) / 65536.0 for p in w.preds]
    return w


C5_GROUPS = ((1, 2), (0, 3), (0, 1), (2, 3))   # (partkey,suppkey) (orderkey,shipdate) (orderkey,partkey) (suppkey,shipdate)


def make_c5(nrows: int = SF100_ROWS, data_seed: int = 5, pred_seed: int = 505,
            i64: bool = False) -> Workload:
    cols = lineitem_cols(data_seed, 100, nrows, i64=i64)
    w = Workload("C5_i64" if i64 else "C5", nrows, cols, _preds([]), _pairs([]), [0, 1, 2, 3])
    g = np.random.default_rng(pred_seed)
    w.preds = _preds(_between_batch(w, g, [0, 1, 2, 3], 64))
    pairs = []
    for (ca, cb) in C5_GROUPS:
        ia = g.choice(64, size=16, replace=False) + 64 * ca
        ib = g.choice(64, size=16, replace=False) + 64 * cb
        pairs += [(int(x), int(y)) for x, y in zip(ia, ib)]
    w.pairs = _pairs(pairs)
    w.ndv_hist = [nrows / 4.0, 2.0e7, 1.0e6, 2000.0]
    return w


def make_d(nrows: int = SF100_ROWS, data_seed: int = 5, pred_seed: int = 606, m: int = 16,
           k: int = 16) -> Workload:
    """Exp. D shape (§IV-H: M candidate sets of K predicates; the
    paper's largest point M=16, K=16) on the C5 lineitem table: a pool of 64 predicates (16
    per column: GE at a low / LT at a high quantile, a wide BETWEEN, 13 NOT-BETWEEN narrow windows
    at values drawn from the data, so a conjunction of 16 keeps a fair share of the rows) and
    M sets of K members drawn from the pool, so sets share predicates."""
    cols = lineitem_cols(data_seed, 100, nrows)
    w = Workload("D" if (m, k) == (16, 16) else f"D_m{m}_k{k}", nrows, cols, _preds([]), _pairs([]), [])
    g = np.random.default_rng(pred_seed)
    rows = []
    for c in range(4):
        col = cols[c]
        v = w.values_at(c, g.integers(0, nrows, size=16))
        dom = col.hi - col.lo + 1
        for j in range(16):
            x = int(v[j])
            if j == 0:
                rows.append((c, GE, 0, col.lo + int(g.uniform(0.0, 0.15) * dom), 0))
            elif j == 1:
                rows.append((c, LT, 0, col.hi - int(g.uniform(0.0, 0.15) * dom), 0))
            elif j == 2:
                rows.append((c, BETWEEN, 0, col.lo + int(g.uniform(0.0, 0.1) * dom), col.hi - int(g.uniform(0.0, 0.1) * dom)))
            else:
                wd = _log_uniform_width(g, max(1, dom // 32))
                rows.append((c, BETWEEN, NEGATE, x, x + wd - 1))
    w.preds = _preds(rows)
    w.sets = [sorted(int(i) for i in g.choice(len(rows), size=k, replace=False)) for _ in range(m)]
    return w


CONFIGS = {
    "C1": make_c1, "C2": make_c2, "C3": make_c3, "C4": make_c4, "C5": make_c5,
    "C3B": lambda nrows=100_000_000: make_c3(nrows, variant="B"),
    "C5_i64": lambda nrows=SF100_ROWS: make_c5(nrows, i64=True),
    "D": make_d,
    "D_m1_k16": lambda nrows=SF100_ROWS: make_d(nrows, m=1, k=16),
}

FULL_ROWS = {"C1": 1_000_000, "C2": SF10_ROWS, "C3": 100_000_000, "C3B": 100_000_000,
             "C4": 200_000_000, "C5": SF100_ROWS, "C5_i64": SF100_ROWS, "D": SF100_ROWS,
             "D_m1_k16": SF100_ROWS}


def get(name: str, nrows: int | None = None) -> Workload:
    """Workload `name` at its BASELINE size, or scaled to `nrows` rows."""
    return CONFIGS[name](FULL_ROWS[name] if nrows is None else nrows)
