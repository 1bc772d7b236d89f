"""Summarise an ncu --set full capture of the probe kernel: key metrics, stalls, opcode mix
per warp row-quad, hot SASS.  python tools/ncu_summary.py <rep> <rows> [hot-out]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, rows = sys.argv[1], int(sys.argv[2])
quads = rows / 4 / 32


def page(*a):
    out = subprocess.run(["ncu", "-i", rep, *a, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("--page", "raw")
hdr, units, vals = raw[0], raw[1], raw[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__cycles_elapsed.avg",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum"]
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:70s} {units[i]:10s} {vals[i]}")
print("-- stalls per issue")
for i, h in enumerate(hdr):
    if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
        try:
            if float(vals[i]) > 0.05:
                print(f"  {h[34:-23]:30s} {float(vals[i]):.3f}")
        except ValueError:
            pass
src = page("--page", "source", "--print-source", "sass")
sh, data = src[1], src[2:]
iS, iE, iW = sh.index("Source"), sh.index("Instructions Executed"), sh.index("Warp Stall Sampling (All Samples)")
c, st = collections.Counter(), collections.Counter()
tot = 0
hot = []
for k, r in enumerate(data):
    n = int(r[iE] or 0)
    w = int(r[iW] or 0)
    m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[iS].strip())
    op = m.group(2) if m else r[iS]
    c[op] += n
    st[op] += w
    tot += n
    if n / quads > 0.02:
        hot.append(f"{k:4d} {n / quads:5.2f} {w:6d}  {r[iS].strip()}")
print(f"-- warp instructions per warp row-quad: {tot / quads:.1f}")
ts = sum(st.values()) or 1
print("  " + "  ".join(f"{op} {n / quads:.1f}({100 * st[op] / ts:.0f}%)" for op, n in c.most_common(24)))
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write("\n".join(hot) + "\n")
