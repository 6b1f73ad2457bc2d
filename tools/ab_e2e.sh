#!/bin/bash
# Developer tool (through gpurun): interleaved A/B of the headline bench line
# incl. e2e, working tree (new) vs _lib_base (tools/build_base.sh).
TAG=${1:-abe}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for r in 1 2; do
  for V in base new; do
    if [ $V = base ]; then export XBS_LIB_PATH=paper_2002_11151_b200/_lib_base/libxbarsim_b200.so; else unset XBS_LIB_PATH; fi
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-peak 2>>$OUT/err | tail -n 1 > $OUT/$V$r.json
    python -c "import json,sys; d=json.load(open('$OUT/$V$r.json')); print('$V', d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e']['wall_ms_per_step'])" >> $OUT/ab.txt
  done
done
