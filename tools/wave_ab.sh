#!/bin/bash
# Developer tool: wave alignment of the VMM producers (XBS_WAVE_SYNC) A/B on
# C5 -- per-stage event times, interleaved, then DRAM bytes per launch (ncu).
#   gpurun --timeout 1500 -- bash tools/wave_ab.sh
O=gpurun_out/wave_ab
mkdir -p $O
CMD="python bench.py --config c5 --stage-probe --steps 5 --warmup 3"
for r in 1 2 3; do
  for V in off on; do
    if [ $V = on ]; then export XBS_WAVE_SYNC=1; else unset XBS_WAVE_SYNC; fi
    line=$(timeout 300 $CMD 2>>$O/err.log | tail -n 1)
    echo "{\"round\": $r, \"wave_sync\": \"$V\", \"stages\": $line}" >> $O/stages.jsonl
  done
done
NCU="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.max --clock-control none -k regex:k_fwd_tc|k_bwd_tc -s 6 -c 2 --csv"
for V in off on; do
  if [ $V = on ]; then export XBS_WAVE_SYNC=1; else unset XBS_WAVE_SYNC; fi
  timeout 600 $NCU --log-file $O/ncu_$V.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others > $O/ncu_$V.log 2>&1
done
echo done
