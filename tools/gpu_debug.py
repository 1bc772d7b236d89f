"""Tiny single-probe driver for compute-sanitizer / ncu runs (not a test, not a bench)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
rows = (int(sys.argv[2]) or None) if len(sys.argv) > 2 else 10_000   # 0: full size
rate = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
w = synth.get(name, rows)
cols = [x.cuda() for x in w.table()]
t = gace.Table(cols)
r = t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
torch.cuda.synchronize()
print(name, rows, "n_sampled", r.n_sampled, "counts[:8]", r.counts[:8], "joints[:4]", r.joints[:4],
      "regs nz", int((r.regs > 0).sum()), t.last_timing())
t.detach()
