"""Probe one workload a few times through the C-ABI (for ncu / compute-sanitizer runs).

    python tools/profile_probe.py [--config C5] [--rows N] [--probes 3] [--rate R]

The first probe runs whatever kernel is compiled (the generic one on a fresh process), the
second the structure-specialised one, and from the third on the layout-specialised kernel
(`gace_jit_probe`), which is what bench.py times: profile it with
`ncu -k regex:gace_jit_probe -c 1 ...`.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C5")
ap.add_argument("--rows", type=int, default=None)
ap.add_argument("--probes", type=int, default=3)
ap.add_argument("--rate", type=float, default=None)
a = ap.parse_args()
w = synth.get(a.config, a.rows)
rate = w.rate if a.rate is None else a.rate
cols = [w.column(c, device="cuda") if c in w.probed_cols else torch.zeros(w.nrows, dtype=w.columns[c].torch_dtype,
                                                                               device="cuda")
        for c in range(len(w.columns))]
torch.cuda.synchronize()
t = gace.Table(cols)
for k in range(a.probes):
    if w.sets:
        t.probe_sets(w.preds, w.sets, rate, w.sample_seed)
    else:
        r = t.probe(w.preds, w.pairs, rate, w.sample_seed, w.hll_cols)
    tm = t.last_timing()
    print(f"probe {k}: kernel {tm['jit']} scan {tm['scan_ms']:.3f} ms total {tm['total_ms']:.3f} ms", flush=True)
    if k < 2:
        gace.jit_sync()             # probe 1: structure-keyed kernel, probe 2 on: layout-keyed
t.detach()
