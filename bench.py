#!/usr/bin/env python
"""GACE selectivity-probe benchmark (BASELINE.json metric: probe rows/s and HBM
GB/s (% of B200 peak) at 1/2/4/8 GPUs; probe p50 latency).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl reference]

One step = one gace_probe call = one pass of the whole hot path (sample bit,
predicate buckets, counts, joint grids, HLL, finalize, NCCL merge, D2H) over
the table.  Default workload: C5 (BASELINE configs[4], the config the north
star's target is quoted on: 600,037,902-row lineitem-shaped table, 256
predicates, 64 pairs, HLL on 4 columns; it fits one B200).  For N > 1 the
same table is sharded contiguously across ranks (strong scaling) and merged
with one NCCL all-reduce(sum) + one all-reduce(max) inside gace_probe.

`value` = table rows / device time of the K steps (CUDA events on the
table's stream, barrier + synchronize on both sides, max over ranks).
`e2e` = the same metric through the host-table C-ABI path (keys in pinned
host memory, H2D of every probed key inside every step, result D2H).
`--impl reference` times the oracle (oracle/, plain C scan) on this host's
cores, on a bounded row sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

with open(os.path.join(ROOT, "BASELINE.json")) as _f:
    BASELINE = json.load(_f)
METRIC = BASELINE["metric"]
L2_BYTES = 126 * 1024 * 1024


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


NOMINAL_HBM_GBS = 8000.0      # BASELINE.json north_star "~8 TB/s" (B200_PROFILING.md: 7.7 HGX / 8 DGX)


def read_ceiling():
    """Measured read-only streaming ceiling (tools/stream_read.cu on a B200, profiles/stream_read.json)."""
    p = os.path.join(ROOT, "profiles", "stream_read.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["read_ceiling_gbs"]), d.get("read_ceiling_variant", "")
    return None, None


def fresh_batch(w, b: int):
    """Batch b of a bind-variable sweep over w's query template (the
    bind centre moves per query): the same predicates and pairs with every bound shifted,
    so each batch is new to the library (new plan, new lookup tables), its structure is
    the template's.  EQ binds move by 37 values per batch (C3's sliding bind window);
    range bounds by 0.05 % of the column's domain per batch, wrapping inside the domain."""
    P = w.preds.copy()
    for c, col in enumerate(w.columns):
        m = P["col"] == c
        if not m.any():
            continue
        step = 37 if np.all(P["op"][m] == 0) else max(1, int((col.hi - col.lo) * 5e-4))
        # the bind stays inside the column's value domain (wrapping around it), the range keeps
        # its width: a real sweep moves the bind centre over the data, not off it
        span = col.hi - col.lo + 1
        a = P["a"][m]
        a2 = col.lo + (a - col.lo + b * step) % span
        P["b"][m] += a2 - a
        P["a"][m] = a2
    return P


def describe(w) -> dict:
    if w.sets:
        ks = sorted(set(len(x) for x in w.sets))
        return {"workload": f"{w.name}: {w.nrows:,} rows x {len(w.probed_cols)} key columns "
                            f"({'/'.join(w.columns[c].dtype for c in w.probed_cols)}), {len(w.sets)} candidate sets "
                            f"x K={'/'.join(map(str, ks))} predicates from a pool of {len(w.preds)} "
                            f"(conjunction counts, PAPER.md Exp. D), sample rate {w.rate}",
                "rows": w.nrows, "predicates": int(len(w.preds)), "sets": len(w.sets), "k": ks,
                "sample_rate": w.rate, "bytes_per_row": w.bytes_per_row}
    return {"workload": f"{w.name}: {w.nrows:,} rows x {len(w.probed_cols)} key columns "
                        f"({'/'.join(w.columns[c].dtype for c in w.probed_cols)}), {len(w.preds)} predicates, "
                        f"{len(w.pairs)} pairs, HLL p=12 on {len(w.hll_cols)} columns, sample rate {w.rate}",
            "rows": w.nrows, "predicates": int(len(w.preds)), "pairs": int(len(w.pairs)),
            "hll_cols": len(w.hll_cols), "sample_rate": w.rate,
            "bytes_per_row": w.bytes_per_row}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region (B200_PROFILING.md)."""
    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = f"/tmp/gace_clocks_{os.getpid()}.csv"

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.index), "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self) -> dict | None:
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx = max(mx, float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def nearest_rank(xs, q):
    s = sorted(xs)
    return s[max(1, math.ceil(q * len(s))) - 1]


# ------------------------------------------------------------------ oracle (CPU) leg

def oracle_rate(w, rows: int, threads: int = 0):
    """Oracle rows/s on rows [0, rows) of workload w (host cores); returns (rows/s, seconds, threads)."""
    from oracle import reference as R
    cols = [w.column(c, 0, rows).numpy() for c in range(len(w.columns))]
    t0 = time.perf_counter()
    if w.sets:
        R.probe_sets(cols, w.preds, w.sets, rate=w.rate, seed=w.sample_seed, nthreads=threads)
    else:
        R.probe(cols, w.preds, w.pairs, rate=w.rate, seed=w.sample_seed, hll_cols=w.hll_cols, nthreads=threads)
    dt = time.perf_counter() - t0
    return rows / dt, dt, (threads or os.cpu_count())


def calibrate_oracle_rows(w, budget_s: float) -> int:
    probe_rows = min(w.nrows, 200_000)
    r, dt, _ = oracle_rate(w, probe_rows)
    return int(min(w.nrows, max(probe_rows, r * budget_s)))


def run_reference(args, w, rank, world):
    if rank != 0:
        return
    rows = calibrate_oracle_rows(w, budget_s=max(2.0, 60.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_rate(w, min(rows, 100_000))
    times = []
    for _ in range(args.steps):
        _, dt, cores = oracle_rate(w, rows)
        times.append(dt)
    value = rows * len(times) / sum(times)
    cfg = run_config(w, world, args)
    sample = (f"rows [0, {rows:,}) of {w.name} per step ({rows / w.nrows:.2%} of the table; every predicate, "
              f"pair and HLL column), oracle C scan on {cores} host threads ({cpu_model()})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": dtype_of(w), "data": "synthetic",
        "config": cfg,
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": cores, "kind": "oracle", "sample": sample,
                         "cpu_model": cpu_model(), "rows_per_step": rows},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def dtype_of(w) -> str:
    return "int32" if all(w.columns[c].dtype == "i32" for c in w.probed_cols) else "int32/int64"


def run_config(w, world, args) -> dict:
    """The `config` object both arms print (identical for the same workload and N)."""
    return dict(describe(w), parallelism=f"dp{world}: contiguous row shards, NCCL sum/max merge",
                cuda_graphs=bool(args.graphs),
                l2=("flushed between steps (2x L2 buffer write)"
                    if (w.nrows // max(world, 1)) * w.bytes_per_row < 2 * L2_BYTES
                    else f"inputs larger than L2 ({w.nrows // max(world, 1) * w.bytes_per_row / 1e9:.2f} GB per GPU)"))


# ------------------------------------------------------------------ GPU leg

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--rows", type=int, default=None, help="override table rows (not a bench number)")
    ap.add_argument("--impl", default="gace", choices=["gace", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--graphs", action="store_true",
                    help="replay each repeated probe as a CUDA graph (gace_table_set_graphs; side stream)")
    ap.add_argument("--cold-batches", type=int, default=24,
                    help="after the timed region: wall latency of this many NEW batches of the same query "
                         "template (bind-variable sweep; planning, upload and kernel choice inside)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = synth.get(args.config, args.rows)

    if args.impl == "reference":
        return run_reference(args, w, rank, world)

    import torch.distributed as dist
    from paper_2512_19750_b200 import gace
    from paper_2512_19750_b200 import dist as gdist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    r0, r1 = gdist.shard_range(rank, world, w.nrows)
    nloc = r1 - r0
    probed = w.probed_cols
    cols = []
    for c in range(len(w.columns)):
        if c in probed:
            cols.append(w.column(c, r0, r1, device="cuda"))
        else:                                      # never read by this probe batch
            cols.append(torch.zeros(4, dtype=w.columns[c].torch_dtype, device="cuda"))
    if any(len(c) != nloc for c in cols):
        cols = [c if len(c) == nloc else torch.zeros(nloc, dtype=c.dtype, device="cuda") for c in cols]
    torch.cuda.synchronize()
    dinfo = gdist.dist_info(w.nrows) if world > 1 else None
    if args.graphs:                    # graphs need a capturable (non-legacy) stream
        stream = torch.cuda.Stream()
        torch.cuda.set_stream(stream)
    stream = torch.cuda.current_stream()
    table = gace.Table(cols, dist=dinfo, stream=stream)
    if args.graphs:
        table.set_graphs(True)

    flush = None
    if nloc * w.bytes_per_row < 2 * L2_BYTES:
        flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device="cuda")

    def step():
        if w.sets:
            return table.probe_sets(w.preds, w.sets, w.rate, w.sample_seed)
        return table.probe(w.preds, w.pairs, w.rate, w.sample_seed, w.hll_cols)

    for k in range(2 * args.warmup + 1):
        if flush is not None:
            flush.fill_(1)
        step()
        if k in (args.warmup - 1, args.warmup):
            gace.jit_sync()         # the background compiles of the batch's specialised kernels
    jit_kind = table.last_timing()["jit"] if not w.sets else None

    clocks = ClockSampler(local)
    L0 = gace.kernel_launches()
    scan_ms, stage = [], {}
    lat = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    ev_s = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev_e = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        if flush is not None:
            flush.fill_(k)          # evict the table from L2 between steps (outside the step's events)
        ev_s[k].record(stream)
        t0 = time.perf_counter()
        res = step()
        lat.append(1e3 * (time.perf_counter() - t0))
        ev_e[k].record(stream)
        tm = table.last_timing()
        scan_ms.append(tm["scan_ms"])
        for key in ("plan_upload_ms", "scan_ms", "finalize_ms", "merge_ms", "d2h_ms", "total_ms"):
            stage.setdefault(key, []).append(tm[key])
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = gace.kernel_launches() - L0
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(ev_s, ev_e))
    t = torch.tensor([dev_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    value = w.nrows / (ms_per_step * 1e-3)

    # roofline of the dominant kernel: algorithmic bytes / CUDA-event scan time
    hbm_peak, peak_src = peaks()
    bytes_scanned = tm["bytes_scanned"]
    scan_avg = statistics.mean(scan_ms)
    achieved = bytes_scanned / (scan_avg * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", f"traffic_{w.name}.json")
    if os.path.exists(tp) and args.rows is None:
        with open(tp) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")

    rc, rc_src = read_ceiling()
    out = {
        "metric": METRIC, "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": dtype_of(w),
        "data": "synthetic",
        "config": run_config(w, world, args),
        "hbm_gbs": w.nrows * w.bytes_per_row / (ms_per_step * 1e-3) / 1e9,
        "latency_ms": {"p50": nearest_rank(lat, 0.5), "p99": nearest_rank(lat, 0.99), "kind": "wall, per gace_probe"},
        "stages_ms": {k: statistics.mean(v) for k, v in stage.items()},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": ("sets_kernel (candidate-set conjunction kernel)" if w.sets
                                else {0: "probe_kernel (generic)", 1: "gace_jit_probe (structure-specialised)",
                                      2: "gace_jit_probe (layout-specialised)"}.get(jit_kind, str(jit_kind))),
                     "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": bytes_scanned,
                     "frac_of_nominal": achieved / NOMINAL_HBM_GBS, "nominal_gbs": NOMINAL_HBM_GBS,
                     "frac_of_read_ceiling": (achieved / rc) if rc else None, "read_ceiling_gbs": rc,
                     "read_ceiling_source": (f"tools/stream_read.cu {rc_src} (profiles/stream_read.json)"
                                             if rc else None)},
        "gpu_launches": launches,
        "clocks": clk,
    }

    # e2e: host-resident keys, H2D inside every step (pinned host memory)
    if w.sets:
        out["e2e"] = None     # gace_probe_sets takes device tables only (include/gace.h)
    elif not args.no_e2e:
        hcols = [c.cpu().pin_memory() if len(c) == nloc else c.cpu() for c in cols]
        htable = gace.Table(hcols, host=True, dist=dinfo, device=local, stream=stream)
        hstep = lambda: htable.probe(w.preds, w.pairs, w.rate, w.sample_seed, w.hll_cols)  # noqa: E731
        for _ in range(2):
            hstep()
            gace.jit_sync()         # the host table's plan has its own specialised kernels
        hstep()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            hres = hstep()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        ht = htable.last_timing()
        assert hres.n_sampled == res.n_sampled and np.array_equal(hres.counts, res.counts)
        out["e2e"] = {"value": w.nrows / (float(te.item()) / args.e2e_steps * 1e-3), "unit": "rows/s",
                      "h2d_bytes_per_step": int(nloc * w.bytes_per_row),
                      "d2h_bytes_per_step": int(8 * (1 + len(w.preds) + len(w.pairs)) + 4096 * len(w.hll_cols)),
                      "steps": args.e2e_steps, "h2d_ms": ht["h2d_ms"],
                      "path": "gace_table_attach_host + gace_probe (pinned host keys, chunked H2D overlapped with scan)"}
        htable.detach()
        del hcols

    # cold batches: new predicate batches of the same template, one probe each (wall latency
    # through the C-ABI: planning, plan upload, kernel choice -- no call waits for a compile)
    if args.cold_batches and not w.sets:
        cl, ck = [], []
        for b in range(1, args.cold_batches + 1):
            Pb = fresh_batch(w, b)
            if flush is not None:
                flush.fill_(b)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            table.probe(Pb, w.pairs, w.rate, w.sample_seed, w.hll_cols)
            cl.append(1e3 * (time.perf_counter() - t0))
            ck.append(table.last_timing()["jit"])
        warm = nearest_rank(lat, 0.5)
        out["cold_batches"] = {"n": len(cl), "p50_ms": nearest_rank(cl, 0.5), "p99_ms": nearest_rank(cl, 0.99),
                               "warm_p50_ms": warm, "ratio_p50": nearest_rank(cl, 0.5) / warm,
                               "kernels": {str(k): ck.count(k) for k in sorted(set(ck))},
                               "kind": "wall per gace_probe, a new bind-sweep batch each call (bench.fresh_batch)"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rows = calibrate_oracle_rows(w, budget_s=15.0)
        r, dt, cores = oracle_rate(w, rows)
        out["cpu_baseline"] = {"value": r, "unit": "rows/s", "cores": cores, "kind": "oracle",
                               "cpu_model": cpu_model(),
                               "sample": f"rows [0, {rows:,}) of {w.name} ({dt:.1f} s, "
                                         f"{'all sets' if w.sets else 'all predicates/pairs/HLL'})"}
        if w.name == "C1" or args.config == "C1":
            r1, dt1, _ = oracle_rate(w, min(w.nrows, rows), threads=1)
            out["cpu_baseline"]["single_thread"] = {"value": r1, "unit": "rows/s", "cores": 1,
                                                    "seconds": dt1}
    table.detach()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
