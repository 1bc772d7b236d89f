"""GPU parity at BASELINE's full sizes: the bench configurations compared with the oracle
element by element (BASELINE.json north_star: "bit-exact versus the oracle ... on a
600M-row table"; §III-B, the Measurement Engine measures selectivities).

Each test builds the workload at its full size on the GPU (counter-based generators,
synth/), copies the keys to the host for the oracle's C scan (all host cores), runs the
probe through the C-ABI in the launch configuration bench.py times (device table, one
launch of the plan-specialised kernel over the whole table), and compares n_sampled,
every count, every joint count and every HLL register.  At these sizes the data-dependent
early exits of the kernel all fire (HLL register ceilings on l_partkey / l_suppkey, the
presence-bitmap completion on C4, the clustered l_orderkey path), so they are covered
here against the oracle, not only by invariants.
"""
import gc

import numpy as np
import pytest
import torch

import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    gace.lib()
    assert torch.cuda.is_available()
    return gace


def _full(G, oracle, name, rate=None, seed=None, monkeypatch=None):
    """Probe the full-size workload with every scan kernel a caller can get -- the generic
    kernel (first call: nothing compiled yet), the layout-specialised kernel bench.py times
    (after the background compiles), and the structure-specialised kernel of a new batch
    of the same structure (fresh table, GACE_JIT_LAYOUT=0) -- and compare each with the
    oracle."""
    w = synth.get(name)
    rate = w.rate if rate is None else rate
    seed = w.sample_seed if seed is None else seed
    dcols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    got, kinds = [], []
    t = G.Table(dcols, device=0)
    try:
        for k in range(3):
            got.append(t.probe(w.preds, w.pairs, rate, seed, w.hll_cols))
            kinds.append(t.last_timing()["jit"])
            G.jit_sync()
    finally:
        t.detach()
    if monkeypatch is not None:
        monkeypatch.setenv("GACE_JIT_LAYOUT", "0")
        t = G.Table(dcols, device=0)
        try:
            got.append(t.probe(w.preds, w.pairs, rate, seed, w.hll_cols))
            kinds.append(t.last_timing()["jit"])
        finally:
            t.detach()
        monkeypatch.delenv("GACE_JIT_LAYOUT")
    hcols = [c.cpu().numpy() for c in dcols]
    del dcols
    torch.cuda.empty_cache()
    want = oracle.probe(hcols, w.preds, w.pairs, rate=rate, seed=seed, hll_cols=w.hll_cols)
    del hcols
    gc.collect()
    n, c, j, r = want
    for g, kind in zip(got, kinds):
        assert g.n_sampled == n, kind
        bad = np.nonzero(g.counts != c)[0]
        assert len(bad) == 0, (name, kind, bad[:8], g.counts[bad[:4]], c[bad[:4]])
        np.testing.assert_array_equal(g.joints, j)
        np.testing.assert_array_equal(g.regs, r)
    return kinds


@pytest.mark.parametrize("name", ["C5", "C5_i64", "C4", "C3", "C2"])
def test_bench_config_full_size_vs_oracle(G, oracle, monkeypatch, name):
    monkeypatch.delenv("GACE_JIT", raising=False)
    kinds = _full(G, oracle, name, monkeypatch=monkeypatch if name in ("C5", "C3") else None)
    assert kinds[2] == 2, kinds                 # the layout-specialised kernel bench.py times
    if len(kinds) > 3:
        assert kinds[3] == 1, kinds             # structure-specialised (a new batch's kernel)


def test_c5_full_size_sampled_vs_oracle(G, oracle):
    """C5 at 1 % (the sampled, quad-skipping path at the north star's table size)."""
    _full(G, oracle, "C5", rate=0.01, seed=0x5EED)


def test_exp_d_full_size_vs_oracle(G, oracle):
    """Exp. D (candidate sets, §IV-H) at 600M rows against the oracle's set scan."""
    w = synth.get("D")
    dcols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    t = G.Table(dcols, device=0)
    try:
        n, c = t.probe_sets(w.preds, w.sets, w.rate, w.sample_seed)
    finally:
        t.detach()
    hcols = [x.cpu().numpy() for x in dcols]
    del dcols
    torch.cuda.empty_cache()
    wn, wc = oracle.probe_sets(hcols, w.preds, w.sets, rate=w.rate, seed=w.sample_seed)
    assert n == wn
    np.testing.assert_array_equal(c, wc)
