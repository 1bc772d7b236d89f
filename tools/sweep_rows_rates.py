"""Probe time over table size and sample rate (GPU box): C5's batch on row prefixes of the C5
table (the paper's sampling budget: a larger N at the same latency), and on
the full table at sample rates 1 .. 0.001.  Median of 20 probes after warm-up and jit_sync;
scan = the dominant kernel (CUDA events), total = the call's device span.
    python tools/sweep_rows_rates.py [out.jsonl]"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

w = synth.get("C5")
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
torch.cuda.synchronize()
out = []


def run(n, rate, reps=20):
    t = gace.Table([c[:n] for c in cols])
    try:
        for _ in range(3):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        for _ in range(2):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
        gace.jit_sync()
        scan, tot = [], []
        for _ in range(reps):
            t.probe(w.preds, w.pairs, rate, 1, w.hll_cols)
            tm = t.last_timing()
            scan.append(tm["scan_ms"])
            tot.append(tm["total_ms"])
    finally:
        t.detach()
    r = {"rows": n, "rate": rate, "scan_ms": statistics.median(scan), "total_ms": statistics.median(tot),
         "rows_per_s": n / (statistics.median(tot) * 1e-3),
         "key_gbs": 16 * n / (statistics.median(scan) * 1e-3) / 1e9}
    print(json.dumps(r), flush=True)
    out.append(r)


for n in (1_000_000, 10_000_000, 75_004_736, 150_009_472, 300_018_944, w.nrows):
    run(n, 1.0)
for rate in (0.5, 0.1, 0.01, 0.001):
    run(w.nrows, rate)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        for r in out:
            f.write(json.dumps(r) + "\n")
