"""Markdown table (kernel, launches, total us, share) from an ncu --csv launch list
(--metrics gpu__time_duration.sum).  usage: launch_table.py LAUNCHES.csv"""
import csv, sys
from collections import defaultdict
rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
tot, cnt = defaultdict(float), defaultdict(int)
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}
for r in rows[h + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").split("::")[-1]
    tot[name] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    cnt[name] += 1
T = sum(tot.values())
print("| kernel | launches | total us | share |\n|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| {k} | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / T:.1f}% |")
print(f"\nTotal {T:.1f} us.")
