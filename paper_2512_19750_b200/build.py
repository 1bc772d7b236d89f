"""Build libgace.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_2512_19750_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(ROOT, "build")
LIB = os.path.join(PKG, "libgace.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC,-ffp-contract=off",
          "-I", os.path.join(ROOT, "include"), "-I", CSRC]
SOURCES = ["gace_kernels.cu", "gace_sets.cu", "gace_merge.cu", "gace_host.cpp", "gace_jit.cpp"]
HEADERS = ["gace_plan.h", "gace_kernels.h", "gace_probe.cuh", "gace_jit.h", "gace_sets.h", "gace_merge.h"]


def _nccl_include() -> str | None:
    """NCCL >= 2.28 headers with the device API (nccl_device.h), for the fused merge kernel
    (gace_merge.cu).  The library itself is loaded at run time (dlopen), never linked."""
    try:
        import nvidia.nccl
        for d in list(getattr(nvidia.nccl, "__path__", [])):
            inc = os.path.join(d, "include")
            if os.path.exists(os.path.join(inc, "nccl_device.h")):
                return inc
    except ImportError:
        pass
    return None


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _embed_sources() -> str:
    """build/gace_jit_sources.inc: the probe's device sources as C++ raw strings for NVRTC."""
    inc = os.path.join(OBJ, "gace_jit_sources.inc")
    parts = []
    for var, name in (("kSrcPlanH", "gace_plan.h"), ("kSrcProbeCuh", "gace_probe.cuh")):
        text = open(os.path.join(CSRC, name)).read()
        assert ')GACESRC"' not in text
        parts.append(f'static const char {var}[] = R"GACESRC({text})GACESRC";\n')
    body = "".join(parts)
    if not os.path.exists(inc) or open(inc).read() != body:
        with open(inc, "w") as f:
            f.write(body)
    return inc


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    inc = _embed_sources()
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "gace.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(OBJ, src + ".o")
        objs.append(o)
        if force or _stale(o, [s] + hdrs + [inc]):
            cmd = [NVCC] + ARCH + COMMON + (["-Xptxas", "-v"] if verbose else []) + ["-c", s, "-o", o]
            if src == "gace_merge.cu":
                ninc = _nccl_include()
                cmd[-4:-4] = ["-I", ninc, "-DGACE_NCCL_DEVICE=1"] if ninc else ["-DGACE_NCCL_DEVICE=0"]
            if src.endswith(".cpp"):
                cmd = [NVCC] + COMMON + ["-I", OBJ, "-x", "c++", "-c", s, "-o", o]
            r = subprocess.run(cmd, capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
            if verbose:
                print(r.stderr)
    if force or _stale(LIB, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
