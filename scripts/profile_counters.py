"""Per-kernel counters of one training step (ncu --metrics ... --csv, scripts/prof_round.sh):
markdown table (time, warp instructions, issue-active, pipe utilisation, DRAM bytes, L2 reduction /
atomic traffic) and profiles/inst.json (warp instructions per launch, the compute-roofline input of
bench.py).  usage: profile_counters.py COUNTERS.csv ROUND"""
import csv, json, os, sys
from collections import OrderedDict

src, rnd = sys.argv[1], sys.argv[2]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hi]
per = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    name = name.replace("unnamed>::", "")
    key = (d["ID"], name)
    per.setdefault(key, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
first = OrderedDict()
for (i, k), m in per.items():   # one launch per kernel (the first of the captured step)
    first.setdefault(k, m)
SCALE = 1e-3  # gpu__time_duration in ns -> us
lines = ["| kernel | us | warp inst (M) | issue-active % | ALU % | FMA % | XU (MUFU) % | LSU % | DRAM MB | "
         "L2 RED req (M) | L2 RED sectors (M) | L2 RED req/s (G) | smem atomic wavefronts (M) |",
         "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
inst = {}
stage = {"preprocess_kernel<3>": "preprocess", "blend_fwd_kernel<0>": "blend", "blend_fwd_kernel<0, 0>": "blend", "blend_bwd_kernel": "blend_bwd",
         "loss_fused_kernel": "loss", "project_bwd_kernel<3, 0>": "project_bwd", "adam_kernel<1, 0, 0>": "adam",
         "adam_kernel<1, 0>": "adam", "bin_scatter_kernel": "duplicate"}
for k, m in first.items():
    t = m.get("gpu__time_duration.sum", 0) * SCALE
    wi = m.get("smsp__inst_executed.sum", 0)
    red = m.get("lts__t_requests_op_red.sum", 0)
    lines.append(f"| `{k}` | {t:.1f} | {wi / 1e6:.1f} | {m.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} | "
                 f"{m.get('sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active', 0):.1f} | "
                 f"{m.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.1f} | "
                 f"{m.get('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 0):.1f} | "
                 f"{m.get('sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active', 0):.1f} | "
                 f"{(m.get('dram__bytes_read.sum', 0) + m.get('dram__bytes_write.sum', 0)) / 1e6:.0f} | "
                 f"{red / 1e6:.2f} | {m.get('lts__t_sectors_op_red.sum', 0) / 1e6:.2f} | "
                 f"{(red / (t * 1e-6) / 1e9) if t else 0:.1f} | "
                 f"{m.get('l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum', 0) / 1e6:.2f} |")
    if k in stage:
        inst[stage[k]] = int(wi)
md = (f"# Round {rnd[1:]} — per-kernel counters of one training step at workload H\n\n"
      f"`{os.path.basename(src)}`: `ncu --metrics <list> --clock-control none` over one step of "
      "`scripts/probe_stages.py H 1` (z-ordered store; `scripts/prof_round.sh`).  Percentages are of the "
      "pipe's / issue slot's peak over active cycles; L2 RED = global reductions reaching L2 "
      "(`lts__t_requests_op_red`, `lts__t_sectors_op_red`): K1's chunk-histogram REDs and K8's "
      "per-(Gaussian, tile) `RED.F32x4` sets.\n\n" + "\n".join(lines) + "\n")
open(os.path.join(ROOT, "profiles", f"{rnd}_counters.md"), "w").write(md)
json.dump({"H": inst, "source": f"profiles/{rnd}_counters.md (smsp__inst_executed.sum per launch)"},
          open(os.path.join(ROOT, "profiles", "inst.json"), "w"), indent=1)
print(md)
