#!/bin/bash
# Developer tool: forward epilogue warp selection (default heuristic vs
# forced 8 / 16), interleaved stage times.
O=gpurun_out/${OUT:-ew_sel}
mkdir -p $O
for r in 1 2; do
  for C in ${CASES:-c3 c1 c4 c2-4096 c2-512}; do
    for V in auto 8 16; do
      unset XBS_FWD_EW; [ $V != auto ] && export XBS_FWD_EW=$V
      line=$(timeout 300 python bench.py --config $C --stage-probe --steps 10 --warmup 3 2>>$O/err.log | tail -n 1)
      echo "{\"round\": $r, \"ew\": \"$V\", \"case\": \"$C\", \"stages\": $line}" >> $O/stages.jsonl
    done
  done
done
echo done
