"""Top stall-sampled SASS instructions of one kernel in an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout.splitlines()
r = list(csv.reader(out[1:]))
h = r[0]
ci = {k: i for i, k in enumerate(h)}
rows = []
for idx, row in enumerate(r[1:]):
    try:
        v = float(row[ci["Warp Stall Sampling (All Samples)"]])
    except Exception:
        continue
    rows.append((v, idx, row[ci["Source"]].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
for v, i, s in sorted(rows, reverse=True)[:top]:
    print(f"{100*v/tot:5.1f}%  #{i:4d}  {s}")
