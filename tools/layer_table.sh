#!/bin/bash
# Developer tool: per-layer stage times of C3 / C4 (one core per layer),
# one JSON line per layer in gpurun_out/layers_<cfg>.jsonl.
#   CFGS="c3 c4" bash tools/layer_table.sh
mkdir -p gpurun_out
for cfg in ${CFGS:-c3 c4}; do
  n=$(python -c "from paper_2002_11151_b200.configs import CONFIGS; print(len(CONFIGS['$cfg'].layers))")
  for ((L = 0; L < n; ++L)); do
    timeout 120 python bench.py --config $cfg --layer $L --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others \
      2>>gpurun_out/layers_$cfg.err | tail -n 1 >> gpurun_out/layers_$cfg.jsonl
  done
done
