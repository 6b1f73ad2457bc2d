#!/bin/bash
# Developer tool: ncu cycles / clock / tensor-pipe activity of the VMM
# kernels for the product build and each variant library
# (paper_2002_11151_b200/_lib_<v>/, built by tools/build_variant.sh).
#   VARIANTS="stubmma stubepi" bash tools/variant_probe.sh c5 c2-4096
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__cycles_elapsed.max,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,smsp__inst_executed.sum,sm__issue_active.avg.pct_of_peak_sustained_elapsed
for CFG in "$@"; do
  for V in full ${VARIANTS:-stubmma stubepi}; do
    if [ $V = full ]; then unset XBS_LIB_PATH; else export XBS_LIB_PATH=paper_2002_11151_b200/_lib_$V/libxbarsim_b200.so; fi
    ncu --metrics $M --clock-control none -k 'regex:k_fwd_tc|k_bwd_tc' -s 4 -c 2 --csv \
      python bench.py --config $CFG --stage-probe --steps 1 --warmup 2 2> gpurun_out/vp_${CFG}_$V.err | grep '^"' > gpurun_out/vp_${CFG}_$V.csv
  done
done
