"""C5 scan time at sample rates 1 / 0.5 / 0.2 / 0.1 / 0.01 (medians of 15 after warm-up)."""
import statistics
import sys

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

w = synth.get("C5")
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
for rate in (1.0, 0.5, 0.2, 0.1, 0.01):
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
    print(f"rate {rate}: scan {statistics.median(s):.4f} ms", flush=True)
