"""Which cross-GPU merge a one-rank NCCL table runs (gace_timing.merge: 1 grouped all-reduce,
2 fused peer-memory kernel) and the merge stage time of each, on C1 and C5 (100 probes each).
    python tools/merge_check.py"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

for name, rows in (("C1", 1_000_000), ("C5", 20_000_003)):
    w = synth.get(name, rows)
    cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    for fused in ("0", "1"):
        os.environ["GACE_NCCL_FUSED"] = fused
        t = gace.Table(cols, dist=gace.DistInfo(0, 1, 0, rows, gace.nccl_unique_id()))
        ms, kinds = [], set()
        for k in range(100):
            t.probe(w.preds, w.pairs, 1.0, 0, w.hll_cols)
            tm = t.last_timing()
            kinds.add(tm["merge"])
            if k >= 10:
                ms.append(tm["merge_ms"])
        t.detach()
        print(f"{name} GACE_NCCL_FUSED={fused}: merge kind {sorted(kinds)}, merge stage median "
              f"{1e3 * statistics.median(ms):.1f} us", flush=True)
