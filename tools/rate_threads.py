"""C5 sampled probes (rates 0.5 / 0.2 / 0.1) with 1024- vs 768-thread specialised kernels
(GACE_JIT_THREADS), scan medians -- the sampled 4-column kernel spills at 64 registers."""
import os
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

w = synth.get("C5")
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
for thr in ("1024", "768"):
    os.environ["GACE_JIT_THREADS"] = thr
    for rate in (0.5, 0.2, 0.1, 1.0):
        t = gace.Table(cols)
        for _ in range(3):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        for _ in range(2):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        s = []
        for _ in range(15):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
            s.append(t.last_timing()["scan_ms"])
        t.detach()
        print(f"threads {thr} rate {rate}: scan {statistics.median(s):.4f} ms", flush=True)
