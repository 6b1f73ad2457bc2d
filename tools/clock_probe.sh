#!/bin/bash
# Developer tool: SM clock, cycles and tensor-pipe activity of the VMM
# kernels in the product build and the MMA-only (XBS_STUB_EPI) build, one
# launch each, so time differences can be split into clock and cycles.
#   bash tools/clock_probe.sh c5
CFG=${1:-c5}
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed
for V in full stubepi; do
  if [ $V = full ]; then unset XBS_LIB_PATH; else export XBS_LIB_PATH=paper_2002_11151_b200/_lib_stubepi/libxbarsim_b200.so; fi
  ncu --metrics $M --clock-control none -k 'regex:k_fwd_tc|k_bwd_tc' -s 4 -c 2 --csv \
    python bench.py --config $CFG --stage-probe --steps 1 --warmup 2 > gpurun_out/clock_${CFG}_$V.csv 2> gpurun_out/clock_${CFG}_$V.err
done
