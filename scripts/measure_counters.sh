#!/bin/bash
# Per-kernel counters of one training step at H (-> scripts/profile_counters.py -> profiles/inst.json) and
# the blend issue-ceiling probe (-> scripts/ic_json.py -> profiles/issue_ceiling.json).  Run on the GPU
# box BEFORE the round's bench runs, whose compute roofline reads those two files.  Outputs: gpurun_out/$1_*.
P=${1:-r2}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum
M=$M,lts__t_requests_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
PROBE_MORTON=1 ncu --metrics $M --clock-control none -s 170 -c 30 --csv --log-file gpurun_out/${P}_counters.csv \
    python scripts/probe_stages.py H 1 > /dev/null 2>&1
echo "counters rc=$?"
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for wl in dense H; do
  ncu --metrics $M --clock-control none -k regex:blend -c 3 --csv --log-file gpurun_out/${P}_ic_$wl.csv python scripts/issue_ceiling.py $wl 600 > /dev/null 2>&1
done
echo "issue ceiling rc=$?"
