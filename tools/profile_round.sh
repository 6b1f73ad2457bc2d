#!/bin/bash
# Profiling recipe (run on the B200 through gpurun, from the repo root):
#   gpurun --timeout 1800 -- bash tools/profile_round.sh [config]
# 1. the bench command runs plain (must exit 0), 2. ncu launch list of every
# kernel (device time per launch, cold-cache/serialised: compare shares),
# 3. one --set full capture of the four per-step kernels after warm-up.
set -u
CFG=${1:-c2-4096}
CMD="python bench.py --config $CFG --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/launches_$CFG.csv $CMD > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k 'regex:k_fwd_tc|k_bwd_tc|k_dw_tc|k_update' \
    -s 12 -c 4 -o gpurun_out/prof_$CFG -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
