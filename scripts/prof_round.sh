#!/bin/bash
# Round profiling pass (run on the GPU box): launch list of the bench, one --set full capture of a
# training step at workload H, and the L2 atomic / reduction + instruction counters per kernel.
# Outputs land in gpurun_out/ with prefix $1 (default r2).
P=${1:-r2}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 40 --csv --log-file gpurun_out/${P}_launches.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
echo "launches rc=$?"
PROBE_MORTON=1 ncu --set full --import-source on --clock-control none -s 170 -c 30 -f -o gpurun_out/${P}_step \
    python scripts/probe_stages.py H 1 > /dev/null 2>&1
echo "full rc=$?"
M=gpu__time_duration.sum,smsp__inst_executed.sum,lts__t_requests_op_red.sum,lts__t_sectors_op_red.sum
M=$M,lts__t_requests_op_atom.sum,lts__t_sectors_op_atom.sum,lts__t_sectors.sum,lts__throughput.avg.pct_of_peak_sustained_elapsed
M=$M,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum
M=$M,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active
PROBE_MORTON=1 ncu --metrics $M --clock-control none -s 170 -c 30 --csv --log-file gpurun_out/${P}_counters.csv \
    python scripts/probe_stages.py H 1 > /dev/null 2>&1
echo "counters rc=$?"
