"""Scan time of probe-batch variants on a full-size workload (design exploration, not a bench)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
rows = int(sys.argv[2]) if len(sys.argv) > 2 else None
w = synth.get(name, rows)
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
t = gace.Table(cols)
E = w.preds[:0]
variants = {
    "nothing (n_sampled only)": (E, None, [], 1.0),
    "hll only": (E, None, w.hll_cols, 1.0),
    "1 pred per column": (w.preds[::max(1, len(w.preds) // len(w.probed_cols))], None, [], 1.0),
    "preds only": (w.preds, None, [], 1.0),
    "preds + pairs": (w.preds, w.pairs, [], 1.0),
    "all": (w.preds, w.pairs, w.hll_cols, 1.0),
    "all, rate 0.01": (w.preds, w.pairs, w.hll_cols, 0.01),
}
for k, (P, Q, H, rate) in variants.items():
    for _ in range(2):
        t.probe(P, Q, rate, 1, H)
    gace.jit_sync()
    ms, read = [], 0
    for _ in range(5):
        t.probe(P, Q, rate, 1, H)
        tm = t.last_timing()
        ms.append(tm["scan_ms"])
        read = tm["bytes_scanned"]          # the bytes THIS variant's probe reads (its probed columns)
    if not read:
        # a batch that probes no column reads nothing: no bandwidth to report (round 1 divided
        # the full table's bytes by this empty scan and reported an impossible 16 TB/s)
        print(f"{name} {k:28s} scan {np.median(ms):8.3f} ms  (reads no column)", flush=True)
        continue
    gb = read / (np.median(ms) * 1e-3) / 1e9
    print(f"{name} {k:28s} scan {np.median(ms):8.3f} ms  ({gb:7.1f} GB/s of the bytes it reads)", flush=True)
t.detach()
