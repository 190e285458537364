"""Summarise the issue_ceiling.py ncu CSVs: per blend kernel, warp instructions, duration,
issue-active % and warp instructions per SM cycle (4.0 = every scheduler issuing every cycle).
usage: ic_summary.py CSV [CSV ...]"""
import csv
import sys
from collections import defaultdict

for path in sys.argv[1:]:
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        k = (d["ID"], d["Kernel Name"].split("(")[0].replace("void ", "").replace("unnamed>::", ""))
        per[k][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    for (i, name), m in sorted(per.items()):
        ipc = m["smsp__inst_executed.sum"] / (m["sm__cycles_elapsed.avg"] * 148)
        print(f"{path.split('/')[-1]:14s} {name:22s} {m['gpu__time_duration.sum'] / 1e3:8.1f} us  "
              f"inst {m['smsp__inst_executed.sum'] / 1e6:7.1f} M  issue-active "
              f"{m['smsp__issue_active.avg.pct_of_peak_sustained_active']:5.1f} %  warps-active "
              f"{m['sm__warps_active.avg.pct_of_peak_sustained_active']:5.1f} %  inst/SM-cycle {ipc:4.2f}")
