"""How many fresh bind-sweep batches (bench.fresh_batch) of a workload keep the structure of
the base batch (the structure-keyed JIT source, gace_debug_jit_source); no GPU needed.
    python tools/struct_stability.py C5 [nbatches]"""
import ctypes
import difflib
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import synth  # noqa: E402
from paper_2512_19750_b200 import gace  # noqa: E402

L = gace.lib()
vp, u32, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
L.gace_debug_jit_source.argtypes = [u32, vp, vp, vp, i32, vp, u32, vp, u32, u64, dbl, i32, vp, u64, ctypes.POINTER(u64)]
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 24
w = synth.get(name)


def src(P):
    dt = np.array([0 if c.dtype == "i32" else 1 for c in w.columns], dtype=np.int32)
    lo = np.array([c.lo for c in w.columns], dtype=np.int64)
    hi = np.array([c.hi for c in w.columns], dtype=np.int64)
    Q = gace.as_pairs(w.pairs)
    P = gace.as_preds(P)
    buf = ctypes.create_string_buffer(1 << 17)
    n = ctypes.c_uint64()
    rc = L.gace_debug_jit_source(len(dt), dt.ctypes.data, lo.ctypes.data, hi.ctypes.data, 0, P.ctypes.data, len(P),
                                 Q.ctypes.data if len(Q) else None, len(Q), w.hll_mask, w.rate, 0, buf, 1 << 17,
                                 ctypes.byref(n))
    assert rc == 0, L.gace_last_error()
    return buf.value.decode()


base = src(w.preds)
same = 0
for b in range(1, nb + 1):
    d = [x for x in difflib.unified_diff(base.splitlines(), src(bench.fresh_batch(w, b)).splitlines(), lineterm="")
         if x[:1] in "+-" and x[:3] not in ("+++", "---")]
    same += not d
    if d:
        print(f"batch {b}: " + "; ".join(x[:120] for x in d[:2]))
print(f"{name}: {same}/{nb} fresh batches keep the base structure")
