#!/bin/bash
# Round-end measurements (GPU box): the driver-style bench line, the other workloads, the
# reference arm, and the profiling pass.  Outputs in gpurun_out/ with prefix $1.
P=${1:-r2}
mkdir -p gpurun_out
python bench.py --steps 200 --warmup 10 > gpurun_out/${P}_bench.json 2> gpurun_out/${P}_bench.err; echo "bench rc=$?"
python bench.py --steps 20 --warmup 5 > gpurun_out/${P}_bench_driver.json 2> gpurun_out/${P}_bench_driver.err; echo "driver-style rc=$?"
for wl in c2 c5; do
  python bench.py --workload $wl --steps 50 --no-cpu-baseline > gpurun_out/${P}_bench_$wl.json 2> gpurun_out/${P}_bench_$wl.err
done
python bench.py --workload c3 --densify --steps 300 --no-cpu-baseline > gpurun_out/${P}_bench_c3d.json 2> gpurun_out/${P}_bench_c3d.err
python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/${P}_bench_c4.json 2> gpurun_out/${P}_bench_c4.err
python bench.py --graph --steps 200 --no-cpu-baseline > gpurun_out/${P}_bench_graph.json 2> gpurun_out/${P}_bench_graph.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${P}_ref.json 2> gpurun_out/${P}_ref.err; echo "ref rc=$?"
bash scripts/prof_round.sh ${P}
# blend issue ceiling (dense scene vs H) -> scripts/ic_json.py
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_elapsed.avg,gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for wl in dense H; do
  ncu --metrics $M --clock-control none -k regex:blend -c 3 --csv --log-file gpurun_out/${P}_ic_$wl.csv python scripts/issue_ceiling.py $wl 600 > /dev/null 2>&1
done
echo "issue ceiling rc=$?"
