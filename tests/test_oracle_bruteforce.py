"""C oracle scan == pure-Python brute force, on exhaustive and random tiny tables (CPU).

The two are written separately (oracle/gace_oracle.c vs oracle/reference.py
brute_probe) from SURVEY.md §8(c); agreement over every tiny table catches a
slip in either (a wrong operator, a dropped negation, a transposed pair index,
an HLL shift)."""
import itertools

import numpy as np

I32MIN, I32MAX = -(2 ** 31), 2 ** 31 - 1
I64MIN, I64MAX = -(2 ** 63), 2 ** 63 - 1
BOUNDARY = [I64MIN, I32MIN - 1, I32MIN, I32MIN + 1, -3, -2, -1, 0, 1, 2, 3,
            I32MAX - 1, I32MAX, I32MAX + 1, I64MAX]
VALUES = [-2, -1, 0, 1, 2, I32MIN, I32MAX]


def _all_preds(oracle, col=0):
    rows = []
    for op in range(5):
        for a in BOUNDARY:
            for fl in (0, 1):
                rows.append((col, op, fl, a, 0))
    for a in (I32MIN, -2, 0, 1, I32MAX, I64MIN):
        for b in (I32MIN, -1, 0, 2, I32MAX, I64MAX):
            for fl in (0, 1):
                rows.append((col, oracle.BETWEEN, fl, a, b))
    return np.array(rows, dtype=oracle.PRED_DTYPE)


def _check(oracle, cols, dtypes, P, Q, rate, seed, hll_cols, row_offset=0):
    npcols = [np.array(c, dtype=np.int32 if d == oracle.I32 else np.int64) for c, d in zip(cols, dtypes)]
    n, c, j, r = oracle.probe(npcols, P, Q, rate=rate, seed=seed, hll_cols=hll_cols, row_offset=row_offset)
    bn, bc, bj, br = oracle.brute_probe(cols, dtypes, P, Q, rate=rate, seed=seed, hll_cols=hll_cols,
                                        row_offset=row_offset)
    assert n == bn
    assert [int(x) for x in c] == bc
    assert [int(x) for x in j] == bj
    for k in range(len(br)):
        assert list(r[k]) == br[k]


def test_exhaustive_single_column(oracle):
    P = _all_preds(oracle)
    Q = np.array([(0, 1), (3, 40), (100, 7), (5, 5)], dtype=oracle.PAIR_DTYPE)
    for nrows in range(0, 4):
        for tab in itertools.product(VALUES, repeat=nrows):
            _check(oracle, [list(tab)], [oracle.I32], P, Q, 1.0, 0, [0] if nrows else [])


def test_random_two_column_tables(oracle):
    g = np.random.default_rng(1234)
    P = np.concatenate([_all_preds(oracle, 0), _all_preds(oracle, 1)])
    for trial in range(60):
        nrows = int(g.integers(1, 9))
        d1 = oracle.I32 if trial % 2 else oracle.I64
        c0 = [int(x) for x in g.choice(VALUES, size=nrows)]
        pool = BOUNDARY if d1 == oracle.I64 else VALUES
        c1 = [int(x) for x in g.choice(pool, size=nrows)]
        Q = np.array([(int(g.integers(0, len(P))), int(g.integers(0, len(P)))) for _ in range(40)],
                     dtype=oracle.PAIR_DTYPE)
        rate = [1.0, 0.5, 0.1, 0.0][trial % 4]
        _check(oracle, [c0, c1], [oracle.I32, d1], P, Q, rate, trial, [0, 1],
               row_offset=int(g.integers(0, 1 << 40)))


def test_random_medium_tables(oracle):
    g = np.random.default_rng(99)
    for trial in range(6):
        nrows = 300
        c0 = [int(x) for x in g.integers(-20, 20, size=nrows)]
        c1 = [int(x) for x in g.integers(-(1 << 35), 1 << 35, size=nrows)]
        rows = []
        for _ in range(40):
            c = int(g.integers(0, 2))
            op = int(g.integers(0, 6))
            a = int(g.integers(-25, 25)) if c == 0 else int(g.integers(-(1 << 35), 1 << 35))
            b = a + int(g.integers(-3, 30)) * (1 if c == 0 else (1 << 30))
            rows.append((c, op, int(g.integers(0, 2)), a, b))
        P = np.array(rows, dtype=oracle.PRED_DTYPE)
        Q = np.array([(int(g.integers(0, 40)), int(g.integers(0, 40))) for _ in range(30)],
                     dtype=oracle.PAIR_DTYPE)
        _check(oracle, [c0, c1], [oracle.I32, oracle.I64], P, Q, [1.0, 0.3][trial % 2], trial, [0, 1])
