"""Calibrate the break-even cost model (Eq. 4; SPEC.md S:232-235 calibrate_cost_model)
on this GPU: wall time of gace_probe_sets over a grid of (N rows, K members, M sets) on
prefixes of the Exp. D table, fitted with gace_cost_fit.

    python tools/calibrate_cost.py [out.json] [--cold]      (needs a GPU)

--cold: every timed call gets a NEW predicate pool (the bind-sweep shift of bench.fresh_batch),
so each call pays planning and plan upload -- the cost a new batch sees.

Every set also holds a tautology on each of the 4 columns (v >= INT64_MIN), so every grid
point scans the same key bytes per row and only K and M vary the evaluation work (the
SPEC's model charges per row, not per byte).  Prints / writes the grid, the fitted
(c0, c_t, c_e, p) and the model's relative error per point.  p = 148 (SMs)."""
import json
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402


def measure(grid_n=(100_000, 1_000_000, 10_000_000, 100_000_000, 600_037_902), grid_k=(1, 4, 16),
            grid_m=(1, 4, 16), reps=7, p=148.0, cold=False):
    w = synth.get("D", max(grid_n))
    cols = [w.column(c, device="cuda") for c in range(len(w.columns))]
    torch.cuda.synchronize()
    g = np.random.default_rng(7)
    npool = len(w.preds)
    taut = np.zeros(4, dtype=w.preds.dtype)
    for c in range(4):
        taut[c] = (c, 4, 0, -(2 ** 63), 0)             # GE INT64_MIN: every row
    preds = np.concatenate([w.preds, taut])
    pts = []
    batch = [0]

    def pool():                  # cold: a new bind-sweep batch of the pool per call
        if not cold:
            return preds
        batch[0] += 1
        return np.concatenate([bench.fresh_batch(w, batch[0]), taut])
    for n in grid_n:
        t = gace.Table([c[:n] for c in cols], device=0)
        for k in grid_k:
            for m in grid_m:
                sets = [sorted(int(i) for i in g.choice(npool, size=k, replace=False)) + list(range(npool, npool + 4))
                        for _ in range(m)]
                t.probe_sets(pool(), sets)                  # plan + warm-up
                ts = []
                for _ in range(reps):
                    P = pool()
                    t0 = time.perf_counter()
                    t.probe_sets(P, sets)
                    ts.append(1e3 * (time.perf_counter() - t0))
                pts.append({"n": n, "k": k, "m": m, "ms": statistics.median(ts)})
        t.detach()
    arr = {key: np.array([q[key] for q in pts], dtype=np.float64) for key in ("n", "k", "m", "ms")}
    c0, ct, ce, pp, wgt = gace.cost_fit(arr["n"], arr["k"], arr["m"], arr["ms"], p)
    for q in pts:
        pred = c0 + ct * q["n"] + ce * q["k"] * q["m"] * q["n"] / pp
        q["model_ms"] = pred
        q["rel_err"] = (pred - q["ms"]) / q["ms"]
    return {"model": {"c0_ms": c0, "ct_ms_per_row": ct, "ce_ms_per_eval": ce, "p": pp, "benefit_weight": wgt},
            "points": pts, "gpu": torch.cuda.get_device_name(0),
            "note": "wall time per gace_probe_sets call (%s), median of %d" %
                    ("a new predicate batch per call: planning + upload included" if cold else "plan cached", reps)}


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    r = measure(cold="--cold" in sys.argv)
    s = json.dumps(r, indent=1)
    print(s)
    if args:
        open(args[0], "w").write(s)
