#!/bin/bash
# Full ncu capture (--set full) of ~one training step's kernels at workload $1 (default H), Adam mode $2.
# usage: scripts/ncu_step.sh [WORKLOAD] [MODE] [OUT]   (run on the GPU box; report lands in gpurun_out/)
W=${1:-H}; M=${2:-1}; OUT=${3:-gpurun_out/step_full}
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -s 170 -c 30 -f -o "$OUT" \
    python scripts/probe_stages.py "$W" "$M" > /dev/null 2>&1
echo "ncu rc=$?"
