#!/bin/bash
# Round measurement set (run on the B200 through gpurun, from the repo root):
#   gpurun --timeout 2400 -- bash tools/measure_round.sh TAG
# writes gpurun_out/TAG/*.json (one bench line each) + bench logs.
set -u
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
run() {  # name, bench args...
  local name=$1; shift
  timeout 900 python bench.py "$@" > $OUT/$name.log 2>&1
  echo "$name rc=$?"
  tail -n 1 $OUT/$name.log > $OUT/$name.json
}
run bench_c2-4096
run bench_reference --impl reference --steps 2 --warmup 3
for c in c1 c3 c4; do run bench_${c}_all_layers --config $c --all-layers --steps 3 --warmup 3 --no-cpu-baseline; done
run bench_c3_conv --config c3 --conv --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run bench_c4_conv --config c4 --conv --steps 3 --warmup 3 --no-e2e --no-cpu-baseline
run bench_c5_all_layers --config c5 --all-layers --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $OUT/smi.txt
nproc > $OUT/host.txt; lscpu | grep -i "model name" >> $OUT/host.txt
