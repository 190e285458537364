"""Per-launch summary table of an ncu --set full report: time, DRAM bytes, throughput, occupancy, issue.
usage: ncu_summary.py REPORT"""
import csv, subprocess, sys
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out))
h = r[0]
units = dict(zip(h, r[1]))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9, "B": 1,
         "us": 1, "ns": 1e-3, "ms": 1e3, "usecond": 1, "nsecond": 1e-3, "msecond": 1e3}
print(f"{'kernel':40s} {'us':>8s} {'DRAM rd MB':>10s} {'wr MB':>8s} {'GB/s':>7s} {'sm%':>5s} {'mem%':>5s} {'occ%':>5s} {'regs':>4s} {'issue%':>6s} grid")
for row in r[2:]:
    d = dict(zip(h, row))
    f = lambda k: (float(d[k].replace(",", "")) * SCALE.get(units.get(k, ""), 1)) if d.get(k) not in (None, "", "n/a") else float("nan")
    name = d["Kernel Name"].split("(")[0].replace("unnamed>::", "").replace("void ", "")
    t = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum") / 1e6, f("dram__bytes_write.sum") / 1e6
    print(f"{name[:40]:40s} {t:8.1f} {rd:10.1f} {wr:8.1f} {(rd + wr) * 1e6 / (t * 1e-6) / 1e9:7.0f} "
          f"{f('sm__throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} {f('gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed'):5.1f} "
          f"{f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f} {d.get('launch__registers_per_thread','')[:4]:>4s} "
          f"{f('smsp__issue_active.avg.pct_of_peak_sustained_active'):6.1f} {d.get('launch__grid_size','')}")
