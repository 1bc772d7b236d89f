"""Print the planner's layout for a workload (env GACE_PLAN_DUMP; host only, no GPU)."""
import os
import sys

sys.path.insert(0, ".")
os.environ["GACE_PLAN_DUMP"] = "1"
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
w = synth.get(name, int(sys.argv[2]) if len(sys.argv) > 2 else None)
dt = [0 if c.dtype == "i32" else 1 for c in w.columns]
gace.debug_buckets(dt, [c.lo for c in w.columns], [c.hi for c in w.columns], False, w.preds, w.pairs,
                   w.hll_cols, int(w.preds["col"][0]) if len(w.preds) else 0, [w.columns[0].lo])
