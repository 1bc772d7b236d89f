"""Reproduce the order-dependent full-size mismatch (design debugging)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

pre = sys.argv[1] if len(sys.argv) > 1 else "C5:40000003"
for spec in pre.split(","):
    nm, n = spec.split(":")
    w0 = synth.get(nm, int(n))
    c0 = [x.cuda() for x in w0.table()]
    t0 = gace.Table(c0)
    r0 = t0.probe(w0.preds, w0.pairs, 1.0, 11, w0.hll_cols)
    print("pre", spec, t0.last_timing()["jit"], flush=True)
    t0.detach()
    del c0
w = synth.get("C5")
cols = [c for c in w.table(device="cuda")]
torch.cuda.synchronize()
res = {}
for jit in ("1", "0"):
    os.environ["GACE_JIT"] = jit
    os.environ["GACE_PLAN_DUMP"] = "1" if jit == "1" else ""
    t = gace.Table(cols)
    r = t.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols)
    print("jit", jit, t.last_timing()["jit"], "col3 counts[:4]", r.counts[192:196], "n", r.n_sampled, flush=True)
    res[jit] = r
    t.detach()
print("equal counts", np.array_equal(res["1"].counts, res["0"].counts), "joints", np.array_equal(res["1"].joints, res["0"].joints),
      "regs", np.array_equal(res["1"].regs, res["0"].regs))
