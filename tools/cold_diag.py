"""Where a new batch's extra latency goes (GPU box): for each config, the warm probe and a run
of new bind-sweep batches (bench.fresh_batch), each split into wall, the library's device span
(total_ms), its scan and plan-upload parts and the kernel kind used.
python tools/cold_diag.py C5 C2 C3B ..."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

for name in sys.argv[1:] or ["C5"]:
    w = synth.get(name)
    cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    t = gace.Table(cols)
    for _ in range(3):
        t.probe(w.preds, w.pairs, w.rate, w.sample_seed, w.hll_cols)
    gace.jit_sync()

    def one(P):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        t.probe(P, w.pairs, w.rate, w.sample_seed, w.hll_cols)
        wall = 1e3 * (time.perf_counter() - t0)
        tm = t.last_timing()
        return wall, tm["total_ms"], tm["scan_ms"], tm["plan_upload_ms"], tm["jit"]

    warm = [one(w.preds) for _ in range(20)]
    cold = [one(bench.fresh_batch(w, b)) for b in range(1, 25)]
    for label, xs in (("warm", warm), ("cold", cold)):
        med = [statistics.median(x[i] for x in xs) for i in range(4)]
        kinds = sorted(set(x[4] for x in xs))
        print(f"{name} {label}: wall {med[0]:.4f}  device {med[1]:.4f}  scan {med[2]:.4f}  upload {med[3]:.4f}  "
              f"host {med[0] - med[1]:.4f} ms  kernels {kinds}", flush=True)
    t.detach()
    del cols
    torch.cuda.empty_cache()
