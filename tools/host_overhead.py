"""Host-side overhead of one probe call (GPU box): wall time of Table.probe vs the library's
own first-to-last event span, and the same call through ctypes with preallocated outputs."""
import ctypes
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
w = synth.get(name)
cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
torch.cuda.synchronize()
t = gace.Table(cols)
for _ in range(5):
    t.probe(w.preds, w.pairs, w.rate, w.sample_seed, w.hll_cols)
wall, tot = [], []
for _ in range(50):
    t0 = time.perf_counter()
    t.probe(w.preds, w.pairs, w.rate, w.sample_seed, w.hll_cols)
    wall.append(1e3 * (time.perf_counter() - t0))
    tot.append(t.last_timing()["total_ms"])
P = gace.as_preds(w.preds)
Q = gace.as_pairs(w.pairs)
mask = sum(1 << c for c in w.hll_cols)
counts = np.zeros(max(len(P), 1), np.uint64)
joints = np.zeros(max(len(Q), 1), np.uint64)
regs = np.zeros((max(len(w.hll_cols), 1), 4096), np.uint8)
n = ctypes.c_uint64()
L = gace.lib()
raw = []
for _ in range(50):
    t0 = time.perf_counter()
    L.gace_probe(t._h, P.ctypes.data, len(P), Q.ctypes.data if len(Q) else None, len(Q), float(w.rate),
                 w.sample_seed, mask, 12, ctypes.byref(n), counts.ctypes.data, joints.ctypes.data, regs.ctypes.data)
    raw.append(1e3 * (time.perf_counter() - t0))
print(f"{name}: Table.probe wall p50 {statistics.median(wall):.4f} ms, raw ctypes p50 {statistics.median(raw):.4f} ms, "
      f"event span p50 {statistics.median(tot):.4f} ms")
t.detach()
