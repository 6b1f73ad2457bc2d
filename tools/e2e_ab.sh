#!/bin/bash
# Developer tool: e2e (host C ABI) step time with and without the wave
# alignment of the VMM producers, interleaved.
O=gpurun_out/e2e_ab
mkdir -p $O
for r in 1 2; do
  for V in on off; do
    if [ $V = off ]; then export XBS_NO_WAVE_SYNC=1; else unset XBS_NO_WAVE_SYNC; fi
    timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-others --no-peak 2>>$O/err.log | tail -n 1 | python -c "
import sys,json
d=json.loads(sys.stdin.read()); print(json.dumps({'round': $r, 'wave_sync': '$V', 'ms_per_step': d['ms_per_step'], 'e2e_ms': d['e2e']['ms_per_step'], 'wall_ms': d['e2e']['wall_ms_per_step']}))" >> $O/e2e.jsonl
  done
done
cat $O/e2e.jsonl
