"""C5 scan at sample rates 0.5 .. 0.05 with the per-warp compaction queue forced on / off
(GACE_COMPACT=1 / 0; the default switches at rate 1/8)."""
import os
import statistics
import sys

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

w = synth.get("C5")
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
for comp in ("0", "1"):
    os.environ["GACE_COMPACT"] = comp
    for rate in (0.5, 0.3, 0.2, 0.15, 0.1, 0.05):
        t = gace.Table(cols)
        for _ in range(3):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        for _ in range(2):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        s = []
        for _ in range(10):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
            s.append(t.last_timing()["scan_ms"])
        t.detach()
        print(f"compact {comp} rate {rate}: scan {statistics.median(s):.4f} ms", flush=True)
