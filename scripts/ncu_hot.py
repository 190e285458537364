"""Top stall-sampled and most-executed SASS instructions of one kernel launch in an ncu report.
usage: ncu_hot.py REPORT KERNEL_REGEX [SKIP] [TOP]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", str(skip),
                      "--launch-count", "1"], capture_output=True, text=True).stdout.splitlines()
print(out[0][:160])
r = list(csv.reader(out[1:]))
h = r[0]
ci = {k: i for i, k in enumerate(h)}
rows = []
for idx, row in enumerate(r[1:]):
    try:
        v = float(row[ci["Warp Stall Sampling (All Samples)"]])
        n = float(row[ci["Instructions Executed"]])
    except Exception:
        continue
    rows.append((v, n, idx, row[ci["Source"]].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
totn = sum(x[1] for x in rows) or 1
print(f"total warp instructions {totn:.0f}")
print("-- stall samples --")
for v, n, i, s in sorted(rows, reverse=True)[:top]:
    print(f"{100*v/tot:5.1f}%  #{i:4d}  {s}")
print("-- executed --")
for v, n, i, s in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{100*n/totn:5.1f}%  #{i:4d}  {s}")
