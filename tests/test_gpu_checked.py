"""Specialised kernels built with device-side bounds checks (GACE_JIT_DEFS=GACE_CHECK=1:
every shared-memory access through the probe's helpers is checked against the launch's
dynamic shared memory and traps outside it; gace_probe.cuh smem_check) run over the
workload shapes and edge cases, results compared with the oracle.  compute-sanitizer is
closed on the B200 pool; these checks are the probe's own memcheck for shared memory (global
reads are bounded by the loop structure and covered by the ragged-size cases)."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    gace.lib()
    assert torch.cuda.is_available()
    return gace


@pytest.fixture
def checked(monkeypatch):
    monkeypatch.setenv("GACE_JIT", "1")
    monkeypatch.setenv("GACE_JIT_DEFS", "GACE_CHECK=1")
    yield


def _check(G, oracle, cols, preds, pairs, rate, seed, hll):
    want = oracle.probe(cols, preds, pairs, rate=rate, seed=seed, hll_cols=hll)
    t = G.Table([torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols], device=0)
    try:
        got = t.probe(preds, pairs, rate, seed, hll)
        assert t.last_timing()["jit"] >= 1
    finally:
        t.detach()
    n, c, j, r = want
    assert got.n_sampled == n
    np.testing.assert_array_equal(got.counts, c)
    np.testing.assert_array_equal(got.joints, j)
    np.testing.assert_array_equal(got.regs, r)


@pytest.mark.parametrize("layout", ["0", "1"])
@pytest.mark.parametrize("name,nrows,rate", [
    ("C1", 100_003, 1.0), ("C2", 150_001, 0.01), ("C3", 200_002, 1.0), ("C3B", 100_001, 1.0),
    ("C4", 80_003, 1.0), ("C5", 120_001, 1.0), ("C5", 90_001, 0.05), ("C5_i64", 60_007, 1.0),
])
def test_checked_workloads(G, oracle, checked, monkeypatch, layout, name, nrows, rate):
    monkeypatch.setenv("GACE_JIT_LAYOUT", layout)
    w = synth.get(name, nrows)
    _check(G, oracle, [x.numpy() for x in w.table()], w.preds, w.pairs, rate, 7, w.hll_cols)


@pytest.mark.parametrize("n", [1, 5, 33, 4097, 606_211])
def test_checked_ragged(G, oracle, checked, n):
    w = synth.get("C5", n)
    _check(G, oracle, [x.numpy() for x in w.table()], w.preds, w.pairs, 1.0, 3, w.hll_cols)


def test_checked_special_cells(G, oracle, checked):
    """Dense breakpoints: nested blocks, lists and records behind the one-threshold cells."""
    g = np.random.default_rng(41)
    n = 400_001
    a = g.integers(0, 1_000_000, size=n).astype(np.int32)
    a[: n // 3] = g.integers(500_000, 500_400, size=n // 3)
    b = g.integers(0, 100, size=n).astype(np.int32)
    rows = [(0, 0, 0, v, 0) for v in range(500_000, 500_200, 3)]
    rows += [(0, 5, 0, lo, lo + 1) for lo in (100, 5_000, 77_777, 500_100, 900_000)]
    rows += [(1, 0, 0, v, 0) for v in range(10, 90, 7)]
    P = np.array(rows, dtype=synth.PRED_DTYPE)
    na = sum(1 for r in rows if r[0] == 0)
    Q = np.array([(i, na + j) for i in range(0, na, 5) for j in range(0, len(rows) - na, 3)],
                 dtype=synth.PAIR_DTYPE)
    for rate in (1.0, 0.3):
        _check(G, oracle, [a, b], P, Q, rate, 21, [0, 1])
