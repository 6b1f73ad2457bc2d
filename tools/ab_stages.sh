#!/bin/bash
# Developer tool: per-stage times (bench --stage-probe) of the product build
# and variant libraries, interleaved, several rounds.
#   VARIANTS="bwd8" CASES="c2-4096 c5" ROUNDS=2 bash tools/ab_stages.sh
mkdir -p gpurun_out
OUT=gpurun_out/ab_stages.jsonl
for r in $(seq ${ROUNDS:-2}); do
  for C in ${CASES:-c2-4096}; do
    for V in full $VARIANTS; do
      cfg=${C%%:*}; layer=0; [ "$C" != "$cfg" ] && layer=${C##*:}
      if [ "$V" != full ]; then export XBS_LIB_PATH=paper_2002_11151_b200/_lib_$V/libxbarsim_b200.so; else unset XBS_LIB_PATH; fi
      line=$(timeout 300 python bench.py --config $cfg --layer $layer --stage-probe --steps 5 --warmup 3 2>>gpurun_out/ab_stages.err | tail -n 1)
      echo "{\"round\": $r, \"variant\": \"$V\", \"case\": \"$C\", \"stages\": $line}" >> $OUT
    done
  done
done
