#!/bin/bash
# Developer tool: interleaved A/B of the TMA L2 hints (XBS_NO_L2_HINTS) on C5.
mkdir -p gpurun_out
for r in 1 2 3; do
 for e in on off; do
  unset XBS_NO_L2_HINTS
  [ $e = off ] && export XBS_NO_L2_HINTS=1
  echo "$r $e c5 $(python bench.py --config c5 --stage-probe --steps 4 --warmup 2 2>/dev/null | tail -1)" >> gpurun_out/l2ab.txt
 done
done
