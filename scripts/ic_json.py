"""profiles/issue_ceiling.json from the issue_ceiling.py ncu CSVs (dense and H runs):
warp instructions per SM cycle of blend_fwd / blend_bwd on the dense scene (the ceiling) and at H.
usage: ic_json.py DENSE.csv H.csv"""
import csv
import json
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rates(path):
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        d = dict(zip(h, r))
        per[(d["ID"], d["Kernel Name"])][d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    out = {}
    for (_, name), m in per.items():
        k = "blend_bwd" if "blend_bwd" in name else "blend" if "blend_fwd" in name else None
        if k and k not in out:  # first launch of each kernel
            out[k] = (m["smsp__inst_executed.sum"] / (m["sm__cycles_elapsed.avg"] * 148),
                      m["smsp__issue_active.avg.pct_of_peak_sustained_active"])
    return out


dense, hw = rates(sys.argv[1]), rates(sys.argv[2])
j = {
    "method": "scripts/issue_ceiling.py + ncu --metrics smsp__inst_executed.sum,sm__cycles_elapsed.avg,"
              "smsp__issue_active.avg.pct_of_peak_sustained_active -k regex:blend: the same blend kernels on a dense "
              "scene (large faint splats, ~570 instances per tile, every pixel keeps every fragment: no row cull, no "
              "divergence, no early exit); warp instructions per SM cycle",
    "dense_inst_per_sm_cycle": {k: round(v[0], 3) for k, v in dense.items()},
    "dense_issue_active_pct": {k: round(v[1], 1) for k, v in dense.items()},
    "H_inst_per_sm_cycle_ncu": {k: round(v[0], 3) for k, v in hw.items()},
    "H_frac_of_ceiling_ncu": {k: round(hw[k][0] / dense[k][0], 3) for k in hw if k in dense},
    "source": "profiles/r2_issue_ceiling.md",
}
with open(os.path.join(ROOT, "profiles", "issue_ceiling.json"), "w") as f:
    json.dump(j, f, indent=1)
print(json.dumps(j["H_frac_of_ceiling_ncu"]))
