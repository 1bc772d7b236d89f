"""Per-instruction dynamic profile of a kernel from an ncu report's SASS source page:
    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_sass_profile.py src.csv [rows_per_unit]
Prints executed warp instructions per opcode (per 128 rows if the row count is given as
the 2nd argument), and the hottest straight-line blocks with their counts and stalls."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        n = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    ins.append((r[ix["Address"]], r[ix["Source"]].strip(), n, int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
tot = sum(n for _, _, n, _ in ins)
units = float(sys.argv[2]) / 128 if len(sys.argv) > 2 else None
print(f"total warp instructions {tot:,}" + (f" = {tot / units:.1f} per 128 rows" if units else ""))
ops = collections.Counter()
for _, s, n, _ in ins:
    t = s.split()
    op = t[1] if t and t[0].startswith("@") else (t[0] if t else "?")
    ops[op.split(".")[0]] += n
print("by opcode:", "  ".join(f"{o} {n / (units or 1):.1f}" for o, n in ops.most_common(28)))
stall_tot = sum(x for *_, x in ins)
print(f"stall samples {stall_tot:,}")
# hot instructions in address order with counts (print those executed >= 1% of the max)
mx = max(n for _, _, n, _ in ins)
if "--dump" in sys.argv:
    for a, s, n, st in ins:
        if n >= mx * 0.001:
            print(f"{a[-5:]} {n / (units or 1):8.2f} {st:6d}  {s}")
