"""Stall breakdown + store sector stats per launch of an ncu report.  usage: ncu_stalls.py REPORT [REGEX]"""
import csv, re, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
for row in r[2:]:
    d = dict(zip(h, row))
    name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "")
    if pat and not pat.search(name):
        continue
    items = []
    for k in h:
        if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
            try:
                v = float(d[k])
            except ValueError:
                continue
            if v > 0:
                items.append((v, k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
    items.sort(reverse=True)
    tot = sum(v for v, _ in items) or 1
    st_req = float(d.get("l1tex__t_requests_pipe_lsu_mem_global_op_st.sum") or 0)
    st_sec = float(d.get("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum") or 0)
    print(f"{name[:60]}  t={d.get('gpu__time_duration.sum')}  st sectors/req={st_sec / max(st_req, 1):.1f}")
    print("   " + ", ".join(f"{k} {100 * v / tot:.0f}%" for v, k in items[:7]))
