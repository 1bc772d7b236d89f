"""Full-size C5 consistency check (design debugging): whole-table vs two-shard probes, with
and without the FMT1T format and the specialised kernel.  GPU only."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
w = synth.get(name)
cols = [c for c in w.table(device="cuda")]
N = w.nrows
cut = (N // 2 + 12345) & ~3


def run(env, rate=1.0, seed=0):
    for k, v in env.items():
        os.environ[k] = v
    t = gace.Table(cols)
    whole = t.probe(w.preds, w.pairs, rate, seed, w.hll_cols)
    t.detach()
    parts = []
    for s, e in ((0, cut), (cut, N)):
        tp = gace.Table([c[s:e] for c in cols], dist=gace.DistInfo(0, 1, s, N))
        parts.append(tp.probe(w.preds, w.pairs, rate, seed, w.hll_cols))
        tp.detach()
    for k in env:
        del os.environ[k]
    return whole, parts


for env, rate in (({}, 0.01), ({"GACE_NO_T1": "1"}, 0.01), ({"GACE_JIT": "0"}, 0.01), ({}, 1.0)):
    whole, parts = run(env, rate, 0x5EED if rate < 1 else 0)
    merged = parts[0].counts + parts[1].counts
    bad = np.nonzero(whole.counts != merged)[0]
    cols_bad = sorted(set(int(w.preds["col"][i]) for i in bad))
    print(env, "n", whole.n_sampled, parts[0].n_sampled + parts[1].n_sampled, "bad preds", len(bad), "cols", cols_bad,
          "joints bad", int((whole.joints != parts[0].joints + parts[1].joints).sum()),
          "regs bad", int((whole.regs != np.maximum(parts[0].regs, parts[1].regs)).sum()), flush=True)
    if len(bad):
        i = bad[0]
        print("  pred", w.preds[i], "whole", whole.counts[i], "parts", parts[0].counts[i], parts[1].counts[i])
    if env == {}:
        ref_whole = whole
# cross-check formats on the whole table
