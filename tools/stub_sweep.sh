#!/bin/bash
# Developer tool: per-stage times of the normal build and of perf-experiment
# variants built by tools/build_variant.sh.
#   VARIANTS="stubmma stubepi" CASES="c2-4096:0 c4:1 c3:1" bash tools/stub_sweep.sh
mkdir -p gpurun_out
OUT=gpurun_out/stub_sweep.jsonl
VARIANTS=${VARIANTS-stubmma stubepi}
CASES=${CASES:-c2-4096:0 c4:1 c3:1}
for C in $CASES; do
  for V in full $VARIANTS; do
    cfg=${C%%:*}; layer=${C##*:}
    if [ "$V" != full ]; then export XBS_LIB_PATH=paper_2002_11151_b200/_lib_$V/libxbarsim_b200.so; else unset XBS_LIB_PATH; fi
    echo -n "{\"variant\": \"$V\", \"cfg\": \"$cfg\", \"layer\": $layer, \"line\": " >> $OUT
    timeout 120 python bench.py --config $cfg --layer $layer --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak 2>>gpurun_out/stub_sweep.err | tail -n 1 | tr -d '\n' >> $OUT
    echo "}" >> $OUT
  done
done
