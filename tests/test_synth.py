"""Input generators: determinism, shard locality, and the distributions the
configs promise (SPEC.md gen_zipf_column / gen_correlated_column)."""
import math

import numpy as np
import torch

import synth
from synth import workloads as W


def test_deterministic_and_shard_local():
    w = synth.get("C5", 5000)
    whole = w.table()
    again = synth.get("C5", 5000).table()
    for a, b in zip(whole, again):
        assert torch.equal(a, b)
    for c in range(4):
        part = w.column(c, 1234, 4321)
        assert torch.equal(part, whole[c][1234:4321])
        chunked = w.column(c, 0, 5000, chunk=777)
        assert torch.equal(chunked, whole[c])


def test_zipf_share():
    # Zipf(1.2, 8) rank-1 share = 1/sum_j j^-1.2 (= 0.4286; SPEC.md S:57's 0.447 is a slip)
    share = W.zipf_share(8, 1.2)
    assert abs(share - 1.0 / sum(j ** -1.2 for j in range(1, 9))) < 1e-15
    w = synth.get("C1", 200000)
    st = w.column(0).numpy()
    freq = np.bincount(st, minlength=8) / len(st)
    theo = np.array([W.zipf_share(8, 1.2, k) for k in range(1, 9)])
    assert np.abs(freq - theo).sum() < 0.02


def test_correlated_pair_pcs():
    # b = a w.p. rho: aligned windows of width fraction f give E[PCS] = rho/f + 1 - rho
    w = synth.get("C4", 200000)
    t = [x.numpy() for x in w.table()]
    for k, rho in enumerate(W.C4_RHO):
        a, b = t[2 * k], t[2 * k + 1]
        lo, hi = 0, 65535 // 4               # f = 1/4
        pa = np.mean((a >= lo) & (a <= hi))
        pb = np.mean((b >= lo) & (b <= hi))
        pab = np.mean((a >= lo) & (a <= hi) & (b >= lo) & (b <= hi))
        assert abs(pab / (pa * pb) - (rho * 4 + 1 - rho)) < 0.1


def test_config_shapes():
    for name, P, Q, H in (("C1", 16, 4, 4), ("C2", 256, 0, 0), ("C3", 1024, 0, 1),
                          ("C4", 128, 64, 8), ("C5", 256, 64, 4)):
        w = synth.get(name, 1000)
        assert len(w.preds) == P and len(w.pairs) == Q and len(w.hll_cols) == H
        assert int(w.preds["col"].max()) < len(w.columns)
        if Q:
            assert int(w.pairs["i"].max()) < P and int(w.pairs["j"].max()) < P
    assert synth.get("C2", 1000).rate == 0.01
    lineitem = synth.get("C5", 10 ** 6).table()
    ok = lineitem[0].numpy()
    assert np.all(np.diff(ok) >= 0)                 # clustered orderkey
    assert ok.max() <= 4 * 10 ** 6
    assert W.FULL_ROWS["C5"] == 600_037_902 and math.isclose(W.FULL_ROWS["C2"] / 59_986_052, 1.0)
