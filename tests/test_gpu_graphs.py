"""CUDA-graph replay of repeated probes (gace_table_set_graphs).

A replayed graph runs the same kernels on the same inputs, so every result must be
bit-identical to the oracle; the tests also check when a graph is captured, replayed
and re-captured (plan, seed or sample-rate change).
"""
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


def _same(got, want):
    n, c, j, r = want
    assert got.n_sampled == n
    np.testing.assert_array_equal(got.counts, c)
    np.testing.assert_array_equal(got.joints, j)
    np.testing.assert_array_equal(got.regs, r)


@pytest.mark.parametrize("jit", ["0", "1"])
@pytest.mark.parametrize("name,nrows,rate", [("C1", 100_003, 1.0), ("C5", 120_001, 1.0), ("C2", 200_001, 0.01)])
def test_graph_replay_parity(G, oracle, monkeypatch, jit, name, nrows, rate):
    monkeypatch.setenv("GACE_JIT", jit)
    # one specialised kernel kind (the layout-keyed one, compiled synchronously): a kernel
    # that a background compile upgrades mid-sequence changes the graph key, so the counts
    # of captures below would depend on the compile's timing (results would not)
    monkeypatch.setenv("GACE_JIT_LAYOUT", "1")
    w = synth.get(name, nrows)
    cols_np = [x.numpy() for x in w.table()]
    want = oracle.probe(cols_np, w.preds, w.pairs, rate=rate, seed=5, hll_cols=w.hll_cols)
    t = G.Table([torch.from_numpy(np.ascontiguousarray(c)).cuda() for c in cols_np], device=0)
    try:
        t.set_graphs(True)
        for _ in range(5):          # eager, capture, 3 replays
            _same(t.probe(w.preds, w.pairs, rate, 5, w.hll_cols), want)
        assert t.graph_stats() == (1, 3)
        tm = t.last_timing()
        assert tm["scan_ms"] > 0 and tm["total_ms"] >= tm["scan_ms"]
        # another seed: eager once, then captured again
        want2 = oracle.probe(cols_np, w.preds, w.pairs, rate=rate, seed=6, hll_cols=w.hll_cols)
        for _ in range(3):
            _same(t.probe(w.preds, w.pairs, rate, 6, w.hll_cols), want2)
        assert t.graph_stats() == (2, 4)
        # another batch (new plan): its own capture; the old graph is never replayed for it
        preds = w.preds[: max(1, len(w.preds) // 2)]
        want3 = oracle.probe(cols_np, preds, None, rate=rate, seed=5, hll_cols=w.hll_cols)
        for _ in range(3):
            _same(t.probe(preds, None, rate, 5, w.hll_cols), want3)
        assert t.graph_stats() == (3, 5)
        # back to the first batch: a new plan generation, so a fresh capture, same results
        for _ in range(3):
            _same(t.probe(w.preds, w.pairs, rate, 5, w.hll_cols), want)
        assert t.graph_stats() == (4, 6)
        t.set_graphs(False)
        _same(t.probe(w.preds, w.pairs, rate, 5, w.hll_cols), want)
        assert t.graph_stats() == (4, 6)
    finally:
        t.detach()


def test_graphs_skip_host_tables(G, oracle):
    w = synth.get("C1", 50_001)
    cols_np = [x.numpy() for x in w.table()]
    want = oracle.probe(cols_np, w.preds, w.pairs, rate=1.0, seed=0, hll_cols=w.hll_cols)
    t = G.Table([torch.from_numpy(np.ascontiguousarray(c)).pin_memory() for c in cols_np], host=True, device=0)
    try:
        t.set_graphs(True)
        for _ in range(3):
            _same(t.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols), want)
        assert t.graph_stats() == (0, 0)
    finally:
        t.detach()
