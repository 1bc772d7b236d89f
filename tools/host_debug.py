"""Host-table vs device-table probe at moderate size (chunked H2D launches), JIT on/off."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 40_000_000
w = synth.get(name, rows)
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
dev = gace.Table(cols)
ref = dev.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols)
print("device", ref.n_sampled, dev.last_timing()["jit"], flush=True)
hcols = [c.cpu().pin_memory() for c in cols]
for jit in ("0", "1"):
    os.environ["GACE_JIT"] = jit
    h = gace.Table(hcols, host=True, device=0)
    r = h.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols)
    torch.cuda.synchronize()
    print("host jit", jit, r.n_sampled, np.array_equal(r.counts, ref.counts), np.array_equal(r.joints, ref.joints),
          np.array_equal(r.regs, ref.regs), h.last_timing(), flush=True)
    h.detach()
