"""Write the plan-specialised kernel source of a workload's batch (as the library would
compile it with NVRTC) and report ptxas registers / spills / opcode counts for sm_100a.
No GPU needed.   python tools/jit_src.py C5 [out.cu]"""
import os
import subprocess
import sys

sys.path.insert(0, ".")
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
out = sys.argv[2] if len(sys.argv) > 2 else f"build/jit_{name}.cu"
rows = int(sys.argv[3]) if len(sys.argv) > 3 else None     # default: the workload's full size
# GACE_DEBUG_CLUSTERED=<column mask> plans and compiles those columns as clustered (C5: l_orderkey = 1)
os.makedirs("build", exist_ok=True)
os.environ["GACE_JIT_SRC"] = out
from paper_2512_19750_b200 import gace  # noqa: E402

w = synth.get(name, rows)
os.environ.setdefault("GACE_DEBUG_ROWS", str(w.nrows))
dt = [0 if c.dtype == "i32" else 1 for c in w.columns]
gace.debug_jit_compile(dt, [c.lo for c in w.columns], [c.hi for c in w.columns], False, w.preds, w.pairs,
                       w.hll_cols, w.rate)
cub = out.replace(".cu", ".cubin")
r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-std=c++17", "-O3", "-lineinfo", "-cubin",
                    "-Xptxas", "-v", "-I", "paper_2512_19750_b200/csrc", "-I", "include", "-o", cub, out],
                   capture_output=True, text=True)
print(r.stderr.strip().splitlines()[-3:] if r.returncode == 0 else r.stderr)
sass = subprocess.run(["cuobjdump", "-sass", cub], capture_output=True, text=True).stdout
print("SASS instructions:", sum(1 for l in sass.splitlines() if l.strip().startswith("/*") and ";" in l))
