"""Aggregate an ncu source page by CUDA source line (cuda,sass view): executed warp instructions and
stall samples per line, all files.  usage: ncu_lines.py REPORT KERNEL_REGEX [SKIP] [TOP]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k", f"regex:{kern}",
                      "--launch-skip", skip, "--launch-count", "1"], capture_output=True, text=True).stdout.splitlines()
rows, fname, h = [], "", None
for r in csv.reader(out):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        h = {k: i for i, k in enumerate(r)}
        continue
    if h is None or len(r) < 3 or r[2] != "-":
        continue  # keep CUDA-line rows only (SASS rows have an address)
    try:
        n = float(r[h["Instructions Executed"]] or 0); v = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, KeyError, IndexError):
        continue
    rows.append((n, v, f"{fname}:{r[0]}", r[1].strip()[:100]))
tn = sum(x[0] for x in rows) or 1
tv = sum(x[1] for x in rows) or 1
print(f"total warp instructions {tn:.4e}  stall samples {tv:.0f}")
for n, v, loc, s in sorted(rows, key=lambda x: -x[1])[:top]:
    print(f"{100*n/tn:5.1f}% inst {100*v/tv:5.1f}% stall  {loc:24s} {s}")
