"""The cross-GPU merge (§IV-B P:100 "Reduction") through the
product's own NCCL path, on one GPU.

A table attached with an NCCL unique id uses the NCCL merge at any rank count, so a
one-rank communicator drives exactly the code a multi-GPU job runs: ncclCommInitRank at
attach, the attach-time all-reduce(min / max) that makes every rank plan over the same
global domains, the plan-agreement all-reduce on every new batch, the grouped
all-reduce(sum u64) + all-reduce(max u8) of the packed result, the device-to-host copy
after the merge (no zero-copy write), and the polled wait with ncclCommGetAsyncError.
Results must equal the oracle bit for bit.
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


def _nccl_table(G, cols, row_offset=0, total=None):
    n = len(cols[0])
    total = row_offset + n if total is None else total
    return G.Table(cols, dist=G.DistInfo(0, 1, row_offset, total, G.nccl_unique_id()), device=0)


@pytest.mark.parametrize("name,nrows,rate,force_jit", [
    ("C1", 100_003, 1.0, False), ("C1", 90_001, 0.3, False), ("C5", 300_001, 1.0, True),
    ("C4", 120_001, 1.0, True), ("C5_i64", 80_003, 0.7, True),
])
def test_nccl_merge_matches_oracle(G, oracle, monkeypatch, name, nrows, rate, force_jit):
    if force_jit:
        monkeypatch.setenv("GACE_JIT", "1")
    w = synth.get(name, nrows)
    cols = [x.numpy() for x in w.table()]
    t = _nccl_table(G, [torch.from_numpy(c).cuda() for c in cols])
    try:
        for seed in (3, 4):                     # a repeated batch reuses the agreed plan
            got = t.probe(w.preds, w.pairs, rate, seed, w.hll_cols)
            n, c, j, r = oracle.probe(cols, w.preds, w.pairs, rate=rate, seed=seed, hll_cols=w.hll_cols)
            assert got.n_sampled == n
            np.testing.assert_array_equal(got.counts, c)
            np.testing.assert_array_equal(got.joints, j)
            np.testing.assert_array_equal(got.regs, r)
        tm = t.last_timing()
        assert tm["merge_ms"] > 0 and tm["d2h_ms"] > 0      # the merge and the copy after it ran
        assert tm["merge"] in (1, 2), tm                    # all-reduce, or the fused window kernel
    finally:
        t.detach()


def test_nccl_merge_shard_with_offset(G, oracle):
    """A shard [r0, r1) of a larger table, global row ids for the sample, NCCL merge."""
    w = synth.get("C1", 200_000)
    cols = [x.numpy() for x in w.table()]
    r0, r1 = 70_004, 161_337
    t = _nccl_table(G, [torch.from_numpy(c[r0:r1].copy()).cuda() for c in cols], r0, 200_000)
    try:
        got = t.probe(w.preds, w.pairs, 0.45, 9, w.hll_cols)
    finally:
        t.detach()
    n, c, j, r = oracle.probe([c[r0:r1] for c in cols], w.preds, w.pairs, rate=0.45, seed=9,
                              hll_cols=w.hll_cols, row_offset=r0)
    assert got.n_sampled == n
    np.testing.assert_array_equal(got.counts, c)
    np.testing.assert_array_equal(got.joints, j)
    np.testing.assert_array_equal(got.regs, r)


def test_nccl_candidate_sets(G, oracle):
    w = synth.get("D", 150_001)
    cols = [x.numpy() for x in w.table()]
    t = _nccl_table(G, [torch.from_numpy(c).cuda() for c in cols])
    try:
        n, c = t.probe_sets(w.preds, w.sets, 1.0, 0)
    finally:
        t.detach()
    wn, wc = oracle.probe_sets(cols, w.preds, w.sets, rate=1.0, seed=0)
    assert n == wn
    np.testing.assert_array_equal(c, wc)


def test_nccl_plan_failure_is_agreed(G):
    """A batch no rank can plan (9 probed columns) fails through the plan agreement, and the
    communicator stays usable for the next batch."""
    g = np.random.default_rng(1)
    cols = [torch.from_numpy(g.integers(0, 100, 4096).astype(np.int32)).cuda() for _ in range(9)]
    t = _nccl_table(G, cols)
    try:
        P = np.array([(c, 0, 0, 5, 0) for c in range(9)], dtype=G.PRED_DTYPE)
        with pytest.raises(G.GaceError) as e:
            t.probe(P)
        assert e.value.status == G.GACE_EUNSUPPORTED
        ok = t.probe(P[:3])
        host = [c.cpu().numpy() for c in cols]
        assert [int(x) for x in ok.counts] == [int((host[c] == 5).sum()) for c in range(3)]
    finally:
        t.detach()


def test_nccl_domain_agreement_empty_shard(G, oracle):
    """An empty shard contributes nothing to the agreed domains; probing it gives zeros."""
    w = synth.get("C1", 1000)
    t = _nccl_table(G, [torch.zeros(0, dtype=c.dtype).cuda() for c in w.table()], 1000, 1000)
    try:
        got = t.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols)
        assert got.n_sampled == 0 and not got.counts.any() and not got.joints.any() and not got.regs.any()
    finally:
        t.detach()


@pytest.mark.parametrize("fused", ["0", "1"])
def test_nccl_merge_kinds(G, oracle, monkeypatch, fused):
    """Both merge implementations on one rank: the grouped ncclAllReduce (GACE_NCCL_FUSED=0)
    and the fused kernel over the NCCL symmetric window (LSA barrier, peer loads: SURVEY.md
    §8(f) NEXT-2b) -- the latter whenever the loaded libnccl has the device API (2.28+)."""
    monkeypatch.setenv("GACE_NCCL_FUSED", fused)
    w = synth.get("C5", 100_003)
    cols = [x.numpy() for x in w.table()]
    t = _nccl_table(G, [torch.from_numpy(c).cuda() for c in cols])
    try:
        for rate in (1.0, 0.3):
            got = t.probe(w.preds, w.pairs, rate, 8, w.hll_cols)
            n, c, j, r = oracle.probe(cols, w.preds, w.pairs, rate=rate, seed=8, hll_cols=w.hll_cols)
            assert got.n_sampled == n
            np.testing.assert_array_equal(got.counts, c)
            np.testing.assert_array_equal(got.joints, j)
            np.testing.assert_array_equal(got.regs, r)
            kind = t.last_timing()["merge"]
            if fused == "0":
                assert kind == 1
            else:
                assert kind in (1, 2)
    finally:
        t.detach()
    if fused == "1":
        import ctypes
        h = ctypes.CDLL("libnccl.so.2", mode=ctypes.RTLD_GLOBAL)
        if hasattr(h, "ncclDevCommCreate"):             # device API present: the fused kernel ran
            assert kind == 2
