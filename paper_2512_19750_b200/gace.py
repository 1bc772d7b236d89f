"""Thin ctypes binding over libgace.so (include/gace.h) -- argument marshalling only.

Every step of the probe runs in the library's sm_100a kernels; this module
only converts torch / numpy buffers into pointers and copies results into
numpy arrays.  If libgace.so is missing it raises; there is no CPU fallback.

Names follow the C-ABI: ``table_attach`` / ``table_attach_host`` ->
``Table``; ``Table.probe`` (gace_probe); ``Table.sample_mask``;
``derive`` (gace_derive); ``gate`` (gace_gate).
"""
from __future__ import annotations

import atexit
import ctypes
import os
from dataclasses import dataclass
from typing import Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libgace.so")

GACE_OK, GACE_EINVAL, GACE_ENOMEM, GACE_ECUDA, GACE_ENCCL, GACE_EHANDLE, GACE_EUNSUPPORTED = range(7)
STATUS_NAMES = ["OK", "EINVAL", "ENOMEM", "ECUDA", "ENCCL", "EHANDLE", "EUNSUPPORTED"]
I32, I64 = 0, 1
EQ, LT, LE, GT, GE, BETWEEN = range(6)
NEGATE = 1
SIG_DRIFT, SIG_SEL_ERROR, SIG_CORRELATION = 1, 2, 4
HLL_P = 12
HLL_M = 1 << HLL_P

PRED_DTYPE = np.dtype([("col", "<u4"), ("op", "<u2"), ("flags", "<u2"), ("a", "<i8"), ("b", "<i8")])
PAIR_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4")])

EXPORTS = ["gace_table_attach", "gace_table_attach_host", "gace_table_detach", "gace_table_set_graphs",
           "gace_table_graph_stats", "gace_probe", "gace_probe_sets", "gace_cost_fit", "gace_gate_decide", "gace_estimate_cv", "gace_cache_create", "gace_cache_destroy", "gace_cache_put",
           "gace_cache_lookup", "gace_cache_invalidate", "gace_cache_stats",
           "gace_sample_mask", "gace_derive", "gace_gate", "gace_last_timing", "gace_nccl_unique_id",
           "gace_jit_sync", "gace_jit_shutdown", "gace_debug_buckets", "gace_debug_jit_compile", "gace_kernel_launches", "gace_last_error"]


class GaceError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < 7 else status}: {msg}")
        self.status = status


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("row_offset", ctypes.c_uint64),
                ("nrows_total", ctypes.c_uint64), ("nccl_unique_id", ctypes.c_void_p),
                ("nccl_comm", ctypes.c_void_p)]


class _Thresholds(ctypes.Structure):
    _fields_ = [("d_threshold", ctypes.c_double), ("sel_err_threshold", ctypes.c_double),
                ("pcs_high", ctypes.c_double), ("pcs_low", ctypes.c_double)]


class _CostModel(ctypes.Structure):
    _fields_ = [("c0_ms", ctypes.c_double), ("ct_ms_per_row", ctypes.c_double), ("ce_ms_per_eval", ctypes.c_double),
                ("p", ctypes.c_double), ("benefit_weight", ctypes.c_double)]


class _CacheEntry(ctypes.Structure):
    _fields_ = [("s_probe", ctypes.c_double), ("count", ctypes.c_uint64), ("n_sampled", ctypes.c_uint64),
                ("hits", ctypes.c_uint64)]


class _Timing(ctypes.Structure):
    _fields_ = [("plan_upload_ms", ctypes.c_double), ("h2d_ms", ctypes.c_double), ("scan_ms", ctypes.c_double),
                ("finalize_ms", ctypes.c_double), ("merge_ms", ctypes.c_double), ("d2h_ms", ctypes.c_double),
                ("total_ms", ctypes.c_double), ("scan_launches", ctypes.c_uint64),
                ("bytes_scanned", ctypes.c_uint64), ("jit", ctypes.c_int32), ("merge", ctypes.c_int32),
                ("jit_compile_ms", ctypes.c_double)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libgace.so (built in-tree by paper_2512_19750_b200.build); raise if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2512_19750_b200.build` "
                          "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, u32, u64, i32, dbl = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_double
    L.gace_table_attach.argtypes = [vp, vp, u32, u64, vp, i32, vp, ctypes.POINTER(vp)]
    L.gace_table_attach_host.argtypes = [vp, vp, u32, u64, vp, i32, vp, ctypes.POINTER(vp)]
    L.gace_table_detach.argtypes = [vp]
    L.gace_table_set_graphs.argtypes = [vp, i32]
    L.gace_table_graph_stats.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.gace_probe.argtypes = [vp, vp, u32, vp, u32, dbl, u64, u64, u32, ctypes.POINTER(u64), vp, vp, vp]
    L.gace_sample_mask.argtypes = [vp, dbl, u64, vp]
    L.gace_cache_create.argtypes = [u32, u32, ctypes.POINTER(vp)]
    L.gace_cache_destroy.argtypes = [vp]
    L.gace_cache_put.argtypes = [vp, u64, vp, u32, vp, ctypes.POINTER(_CacheEntry)]
    L.gace_cache_lookup.argtypes = [vp, u64, vp, u32, vp, ctypes.POINTER(_CacheEntry), ctypes.POINTER(u32)]
    L.gace_cache_invalidate.argtypes = [vp, u64]
    L.gace_cache_stats.argtypes = [vp] + [ctypes.POINTER(u64)] * 4
    L.gace_estimate_cv.argtypes = [vp, vp, u32, vp, u32, dbl, vp, u32, vp, vp, vp]
    L.gace_cost_fit.argtypes = [vp, vp, vp, vp, u32, dbl, ctypes.POINTER(_CostModel)]
    L.gace_gate_decide.argtypes = [u32, ctypes.POINTER(_CostModel), dbl, dbl, dbl, dbl, ctypes.POINTER(dbl),
                                   ctypes.POINTER(dbl), ctypes.POINTER(u32), ctypes.POINTER(u32)]
    L.gace_probe_sets.argtypes = [vp, vp, u32, vp, vp, u32, dbl, u64, ctypes.POINTER(u64), vp]
    L.gace_derive.argtypes = [u64, vp, u32, vp, vp, u32, vp, u32, u32, vp, vp, vp, vp, vp]
    L.gace_gate.argtypes = [vp, u32, vp, vp, u32, vp, u32, vp, ctypes.POINTER(u32), vp]
    L.gace_last_timing.argtypes = [vp, ctypes.POINTER(_Timing)]
    L.gace_nccl_unique_id.argtypes = [vp]
    L.gace_jit_sync.argtypes = [dbl, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.gace_jit_shutdown.argtypes = []
    L.gace_debug_jit_compile.argtypes = [u32, vp, vp, vp, i32, vp, u32, vp, u32, u64, dbl, ctypes.POINTER(u64)]
    L.gace_debug_buckets.argtypes = [u32, vp, vp, vp, i32, vp, u32, vp, u32, u64, u32, vp, u64, vp,
                                     ctypes.POINTER(u32), vp, u32, ctypes.POINTER(u32)]
    for f in EXPORTS:
        if f not in ("gace_kernel_launches", "gace_last_error"):
            getattr(L, f).restype = ctypes.c_int
    L.gace_kernel_launches.restype = u64
    L.gace_kernel_launches.argtypes = []
    L.gace_last_error.restype = ctypes.c_char_p
    L.gace_last_error.argtypes = []
    _lib = L
    # stop the background compile worker before the interpreter tears down torch / CUDA
    atexit.register(L.gace_jit_shutdown)
    return L


def _check(status: int):
    if status != GACE_OK:
        raise GaceError(status, lib().gace_last_error().decode())


def _ptr(a: np.ndarray | None):
    return None if a is None or a.size == 0 else a.ctypes.data


def as_preds(preds) -> np.ndarray:
    a = np.ascontiguousarray(preds)
    return a if a.dtype == PRED_DTYPE else a.astype(PRED_DTYPE)


def as_pairs(pairs) -> np.ndarray:
    if pairs is None or len(pairs) == 0:
        return np.zeros(0, dtype=PAIR_DTYPE)
    a = np.ascontiguousarray(pairs)
    return a if a.dtype == PAIR_DTYPE else a.astype(PAIR_DTYPE)


def debug_buckets(dtypes, dlo, dhi, host: bool, preds, pairs, hll_cols, col: int, values):
    """Planner test hook (host only): bucket of each value of `col` through the planned
    lookup table, using the kernel's lookup code.  Returns (buckets u32, mode, breakpoints)."""
    P = as_preds(preds)
    Q = as_pairs(pairs)
    mask = 0
    for c in hll_cols:
        mask |= 1 << int(c)
    n = len(dtypes)
    dt = np.ascontiguousarray(dtypes, dtype=np.int32)
    lo = np.ascontiguousarray(dlo, dtype=np.int64)
    hi = np.ascontiguousarray(dhi, dtype=np.int64)
    v = np.ascontiguousarray(values, dtype=np.int64)
    out = np.zeros(max(len(v), 1), dtype=np.uint32)
    bps = np.zeros(2 * len(P) + 2, dtype=np.int64)
    mode = ctypes.c_uint32()
    nbp = ctypes.c_uint32()
    _check(lib().gace_debug_buckets(n, dt.ctypes.data, lo.ctypes.data, hi.ctypes.data, int(host), _ptr(P), len(P),
                                    _ptr(Q), len(Q), mask, col, _ptr(v), len(v), out.ctypes.data,
                                    ctypes.byref(mode), bps.ctypes.data, len(bps), ctypes.byref(nbp)))
    return out[:len(v)], int(mode.value), bps[:nbp.value]


def debug_jit_compile(dtypes, dlo, dhi, host: bool, preds, pairs, hll_cols, sample_rate=1.0) -> int:
    """Test hook: NVRTC-compile the plan-specialised probe kernel of this batch (no device);
    returns the cubin size."""
    P = as_preds(preds)
    Q = as_pairs(pairs)
    mask = 0
    for c in hll_cols:
        mask |= 1 << int(c)
    dt = np.ascontiguousarray(dtypes, dtype=np.int32)
    lo = np.ascontiguousarray(dlo, dtype=np.int64)
    hi = np.ascontiguousarray(dhi, dtype=np.int64)
    n = ctypes.c_uint64()
    _check(lib().gace_debug_jit_compile(len(dt), dt.ctypes.data, lo.ctypes.data, hi.ctypes.data, int(host),
                                        _ptr(P), len(P), _ptr(Q), len(Q), mask, float(sample_rate),
                                        ctypes.byref(n)))
    return int(n.value)


def jit_sync(timeout_ms: float = 120_000.0) -> dict:
    """Wait for the background compiles of specialised scan kernels (gace_jit_sync)."""
    c, f, p = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    _check(lib().gace_jit_sync(float(timeout_ms), ctypes.byref(c), ctypes.byref(f), ctypes.byref(p)))
    return {"compiled": c.value, "failed": f.value, "pending": p.value}


def kernel_launches() -> int:
    return int(lib().gace_kernel_launches())


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().gace_nccl_unique_id(buf))
    return buf.raw


@dataclass
class ProbeResult:
    n_sampled: int
    counts: np.ndarray        # u64[P]
    joints: np.ndarray        # u64[Q]
    regs: np.ndarray          # u8[H, 4096], ascending column order


@dataclass
class DistInfo:
    rank: int
    nranks: int
    row_offset: int
    nrows_total: int
    unique_id: bytes | None = None
    comm: int | None = None


def _dtype_code(dt) -> int:
    s = str(dt)
    if s.endswith("int32"):
        return I32
    if s.endswith("int64"):
        return I64
    raise GaceError(GACE_EINVAL, f"unsupported column dtype {dt}")


class Table:
    """A table attached to the library.  ``columns``: CUDA torch tensors (device
    table, zero-copy) or, with ``host=True``, CPU tensors / numpy arrays (host table:
    every probe streams the probed keys over PCIe)."""

    def __init__(self, columns: Sequence, host: bool = False, dist: DistInfo | None = None,
                 device: int | None = None, stream=None):
        L = lib()
        self._cols = list(columns)
        if not self._cols:
            raise GaceError(GACE_EINVAL, "no columns")
        nrows = len(self._cols[0])
        ptrs, codes = [], []
        for c in self._cols:
            if len(c) != nrows:
                raise GaceError(GACE_EINVAL, "columns differ in length")
            codes.append(_dtype_code(c.dtype))
            if isinstance(c, np.ndarray):
                if not host:
                    raise GaceError(GACE_EINVAL, "numpy columns need host=True")
                ptrs.append(c.ctypes.data)
            else:
                if not c.is_contiguous():
                    raise GaceError(GACE_EINVAL, "columns must be contiguous")
                if host != (not c.is_cuda):
                    raise GaceError(GACE_EINVAL, "device tables take CUDA tensors, host tables CPU tensors")
                ptrs.append(c.data_ptr())
                if device is None and c.is_cuda:
                    device = c.device.index
        self.nrows = nrows
        self.ncols = len(self._cols)
        self.host = host
        arr_p = (ctypes.c_void_p * self.ncols)(*ptrs)
        arr_t = (ctypes.c_int * self.ncols)(*codes)
        d = None
        self._uid = None
        if dist is not None:
            self._uid = ctypes.create_string_buffer(dist.unique_id, 128) if dist.unique_id else None
            d = _Dist(dist.rank, dist.nranks, dist.row_offset, dist.nrows_total,
                      ctypes.cast(self._uid, ctypes.c_void_p) if self._uid else None, dist.comm)
        self.row_offset = dist.row_offset if dist else 0
        s = None
        if stream is None and not host:
            # the attach-time domain scan (and every probe) must see the finished columns:
            # work on the caller's current torch stream, or -- for the legacy default stream,
            # handle 0, which the C-ABI reads as "library stream" -- wait for it here
            import torch
            stream = torch.cuda.current_stream(device)
        if stream is not None:
            s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
            if not s:
                if hasattr(stream, "synchronize"):
                    stream.synchronize()
                s = None
        h = ctypes.c_void_p()
        fn = L.gace_table_attach_host if host else L.gace_table_attach
        _check(fn(arr_p, arr_t, self.ncols, nrows, ctypes.byref(d) if d is not None else None,
                  0 if device is None else device, s, ctypes.byref(h)))
        self._h = h

    def probe(self, preds, pairs=None, sample_rate: float = 1.0, seed: int = 0,
              hll_cols: Sequence[int] = (), hll_p: int = HLL_P) -> ProbeResult:
        P = as_preds(preds)
        Q = as_pairs(pairs)
        mask = 0
        for c in hll_cols:
            mask |= 1 << int(c)
        nh = bin(mask).count("1")
        counts = np.zeros(max(len(P), 1), dtype=np.uint64)
        joints = np.zeros(max(len(Q), 1), dtype=np.uint64)
        regs = np.zeros((max(nh, 1), HLL_M), dtype=np.uint8)
        n = ctypes.c_uint64()
        _check(lib().gace_probe(self._h, _ptr(P), len(P), _ptr(Q), len(Q), float(sample_rate),
                                int(seed) & ((1 << 64) - 1), mask, hll_p, ctypes.byref(n),
                                counts.ctypes.data, joints.ctypes.data, regs.ctypes.data))
        return ProbeResult(int(n.value), counts[:len(P)], joints[:len(Q)], regs[:nh])

    def probe_sets(self, preds, sets, sample_rate: float = 1.0, seed: int = 0):
        """Candidate-set conjunction counts (gace_probe_sets; §IV-H Exp. D).
        ``sets``: list of member-index lists.  Returns (n_sampled, u64[len(sets)])."""
        P = as_preds(preds)
        offs = [0]
        mem: list[int] = []
        for st in sets:
            mem.extend(int(i) for i in st)
            offs.append(len(mem))
        O = np.asarray(offs, dtype=np.uint32)
        M = np.asarray(mem if mem else [0], dtype=np.uint32)
        out = np.zeros(max(len(sets), 1), dtype=np.uint64)
        n = ctypes.c_uint64()
        _check(lib().gace_probe_sets(self._h, _ptr(P), len(P), O.ctypes.data, M.ctypes.data, len(sets),
                                     float(sample_rate), int(seed) & ((1 << 64) - 1), ctypes.byref(n),
                                     out.ctypes.data))
        return int(n.value), out[:len(sets)]

    def estimate_cv(self, preds, pairs, sample_rate: float, seeds):
        """Est.CV over seeded probes (gace_estimate_cv; PAPER.md Exp. B).
        Returns (cv_sel[P], cv_joint[Q], cv_pcs[Q])."""
        P = as_preds(preds)
        Q = as_pairs(pairs)
        S = np.ascontiguousarray([int(x) & ((1 << 64) - 1) for x in seeds], dtype=np.uint64)
        cs = np.zeros(max(len(P), 1))
        cj = np.zeros(max(len(Q), 1))
        cp = np.zeros(max(len(Q), 1))
        _check(lib().gace_estimate_cv(self._h, _ptr(P), len(P), _ptr(Q), len(Q), float(sample_rate),
                                      S.ctypes.data, len(S), cs.ctypes.data, cj.ctypes.data, cp.ctypes.data))
        return cs[:len(P)], cj[:len(Q)], cp[:len(Q)]

    def sample_mask(self, sample_rate: float, seed: int) -> np.ndarray:
        bits = np.zeros(max(1, (self.nrows + 63) // 64), dtype=np.uint64)
        _check(lib().gace_sample_mask(self._h, float(sample_rate), int(seed) & ((1 << 64) - 1),
                                      bits.ctypes.data))
        return bits[:(self.nrows + 63) // 64]

    def set_graphs(self, enable: bool = True):
        """gace_table_set_graphs: CUDA-graph replay of repeated identical probes."""
        _check(lib().gace_table_set_graphs(self._h, 1 if enable else 0))

    def graph_stats(self) -> tuple[int, int]:
        """gace_table_graph_stats: (captures, replays)."""
        c, r = ctypes.c_uint64(0), ctypes.c_uint64(0)
        _check(lib().gace_table_graph_stats(self._h, ctypes.byref(c), ctypes.byref(r)))
        return c.value, r.value

    def last_timing(self) -> dict:
        t = _Timing()
        _check(lib().gace_last_timing(self._h, ctypes.byref(t)))
        return {f: getattr(t, f) for f, _ in _Timing._fields_}

    def detach(self):
        if self._h is not None and self._h.value:
            _check(lib().gace_table_detach(self._h))
        self._h = None

    def __del__(self):
        try:
            self.detach()
        except Exception:
            pass


def table_attach(columns, dist: DistInfo | None = None, stream=None) -> Table:
    return Table(columns, host=False, dist=dist, stream=stream)


def table_attach_host(columns, dist: DistInfo | None = None, device: int = 0, stream=None) -> Table:
    return Table(columns, host=True, dist=dist, device=device, stream=stream)


def derive(n_sampled: int, counts, pairs, joints, regs, ndv_hist=None):
    """gace_derive: (sel[P], pcs[Q], ndv_est[H], drift[H]) as float64 arrays."""
    counts = np.ascontiguousarray(counts, dtype=np.uint64)
    Q = as_pairs(pairs)
    joints = np.ascontiguousarray(joints, dtype=np.uint64)
    regs = np.ascontiguousarray(regs, dtype=np.uint8).reshape(-1, HLL_M) if regs is not None and len(regs) \
        else np.zeros((0, HLL_M), np.uint8)
    H = regs.shape[0]
    sel = np.zeros(max(len(counts), 1))
    pcs = np.zeros(max(len(Q), 1))
    ndv = np.zeros(max(H, 1))
    drift = np.zeros(max(H, 1))
    hist = None if ndv_hist is None else np.ascontiguousarray(ndv_hist, dtype=np.float64)
    _check(lib().gace_derive(n_sampled, _ptr(counts), len(counts), _ptr(Q), _ptr(joints), len(Q),
                             _ptr(regs), H, HLL_P, _ptr(hist), sel.ctypes.data, pcs.ctypes.data,
                             ndv.ctypes.data, drift.ctypes.data if hist is not None else None))
    return sel[:len(counts)], pcs[:len(Q)], ndv[:H], (drift[:H] if hist is not None else None)


class ProbeCache:
    """Probe-result cache keyed by (table, normalised conjunction, bind value or range
    bucket) -- gace_cache_* (§V item 3)."""

    def __init__(self, capacity: int = 4096, range_buckets: int = 0):
        h = ctypes.c_void_p()
        _check(lib().gace_cache_create(capacity, range_buckets, ctypes.byref(h)))
        self._h = h

    @staticmethod
    def _args(conj, domains):
        P = as_preds(conj)
        D = None if domains is None else np.ascontiguousarray(domains, dtype=np.int64).reshape(-1)
        return P, D

    def put(self, table_id: int, conj, s_probe: float, count: int = 0, n_sampled: int = 0, domains=None):
        P, D = self._args(conj, domains)
        e = _CacheEntry(float(s_probe), int(count), int(n_sampled), 0)
        _check(lib().gace_cache_put(self._h, int(table_id), _ptr(P), len(P), _ptr(D), ctypes.byref(e)))

    def lookup(self, table_id: int, conj, domains=None):
        """(s_probe, count, n_sampled, hits) or None."""
        P, D = self._args(conj, domains)
        e = _CacheEntry()
        hit = ctypes.c_uint32()
        _check(lib().gace_cache_lookup(self._h, int(table_id), _ptr(P), len(P), _ptr(D), ctypes.byref(e),
                                       ctypes.byref(hit)))
        return (e.s_probe, e.count, e.n_sampled, e.hits) if hit.value else None

    def invalidate(self, table_id: int):
        _check(lib().gace_cache_invalidate(self._h, int(table_id)))

    def stats(self) -> dict:
        v = [ctypes.c_uint64() for _ in range(4)]
        _check(lib().gace_cache_stats(self._h, *[ctypes.byref(x) for x in v]))
        return dict(zip(("hits", "misses", "evictions", "size"), (x.value for x in v)))

    def close(self):
        if self._h is not None and self._h.value:
            _check(lib().gace_cache_destroy(self._h))
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def cost_fit(n, k, m, ms, p: float = 1.0, benefit_weight: float = 0.5):
    """gace_cost_fit: (c0_ms, ct_ms_per_row, ce_ms_per_eval, p, benefit_weight) fitted to
    measured probe times (Eq. 4)."""
    arrs = [np.ascontiguousarray(x, dtype=np.float64) for x in (n, k, m, ms)]
    cm = _CostModel(0.0, 0.0, 0.0, 0.0, float(benefit_weight))
    _check(lib().gace_cost_fit(*[a.ctypes.data for a in arrs], len(arrs[0]), float(p), ctypes.byref(cm)))
    return (cm.c0_ms, cm.ct_ms_per_row, cm.ce_ms_per_eval, cm.p, cm.benefit_weight)


def gate_decide(fired_mask: int, cost_model, n_sample: float, k: float, m: float, plan_cost_spread_ms: float):
    """gace_gate_decide: (est_cost_ms, est_benefit_ms, probe, reason)."""
    cm = _CostModel(*[float(x) for x in cost_model])
    c, b = ctypes.c_double(), ctypes.c_double()
    pr, rs = ctypes.c_uint32(), ctypes.c_uint32()
    _check(lib().gace_gate_decide(int(fired_mask), ctypes.byref(cm), float(n_sample), float(k), float(m),
                                  float(plan_cost_spread_ms), ctypes.byref(c), ctypes.byref(b), ctypes.byref(pr),
                                  ctypes.byref(rs)))
    return c.value, b.value, bool(pr.value), int(rs.value)


def gate(drift=(), s_est=(), s_probe=(), pcs=(), thresholds: dict | None = None):
    """gace_gate: (fired_mask, per-signal bool array in the order drift, sel, pcs)."""
    d = np.ascontiguousarray(drift, dtype=np.float64)
    se = np.ascontiguousarray(s_est, dtype=np.float64)
    sp = np.ascontiguousarray(s_probe, dtype=np.float64)
    pc = np.ascontiguousarray(pcs, dtype=np.float64)
    if len(se) != len(sp):
        raise GaceError(GACE_EINVAL, "s_est and s_probe differ in length")
    th = None
    if thresholds is not None:
        t = {"d": 0.25, "sel_err": 0.01, "pcs_high": 1.6, "pcs_low": 0.7}
        t.update(thresholds)
        th = _Thresholds(t["d"], t["sel_err"], t["pcs_high"], t["pcs_low"])
    per = np.zeros(max(len(d) + len(se) + len(pc), 1), dtype=np.uint8)
    mask = ctypes.c_uint32()
    _check(lib().gace_gate(_ptr(d), len(d), _ptr(se), _ptr(sp), len(se), _ptr(pc), len(pc),
                           ctypes.byref(th) if th is not None else None, ctypes.byref(mask),
                           per.ctypes.data))
    return int(mask.value), per[:len(d) + len(se) + len(pc)].astype(bool)
