#!/bin/bash
# Developer tool (through gpurun): interleaved A/B per-stage timings of the
# working-tree library (new) against _lib_base (tools/build_base.sh).
#   CASES="c2-4096:0 c3:1" REPS=2 bash tools/ab.sh TAG
TAG=${1:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT
CASES=${CASES:-c2-4096:0 c3:0 c3:1 c3:7 c3:13 c4:1 c4:5}
REPS=${REPS:-2}
for C in $CASES; do
  cfg=${C%%:*}; layer=${C##*:}
  for r in $(seq $REPS); do
    for V in base new; do
      if [ $V = base ]; then export XBS_LIB_PATH=paper_2002_11151_b200/_lib_base/libxbarsim_b200.so; else unset XBS_LIB_PATH; fi
      echo -n "$V $cfg:$layer " >> $OUT/ab.txt
      timeout 120 python bench.py --config $cfg --layer $layer --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-peak 2>>$OUT/ab.err | tail -n 1 | python tools/summ.py /dev/stdin >> $OUT/ab.txt
    done
  done
done
echo done
