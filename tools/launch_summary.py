"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel:
launches, total and mean ns, share of the listed time.  python tools/launch_summary.py <csv>"""
import collections
import csv
import sys

rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
acc = collections.OrderedDict()
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0] if not r[ki].startswith("void ") else r[ki].rsplit("(", 1)[0]
    n, t = acc.get(name, (0, 0))
    acc[name] = (n + 1, t + float(r[vi]))
tot = sum(t for _, t in acc.values())
print("kernel,launches,total_ns,mean_ns,share_of_listed")
for name, (n, t) in sorted(acc.items(), key=lambda kv: -kv[1][1]):
    print(f'"{name}",{n},{int(t)},{int(t / n)},{t / tot:.4f}')
