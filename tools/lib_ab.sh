#!/bin/bash
# A/B of library variants on per-stage times (gpurun, repo root):
#   bash tools/lib_ab.sh "<config ...>" <lib dir> [<lib dir> ...]
# e.g. bash tools/lib_ab.sh "c5 c2-4096" _lib _lib_stubepi
CFGS=$1; shift
mkdir -p gpurun_out
for cfg in $CFGS; do
  for rep in 1 2; do
    for L in "$@"; do
      r=$(XBS_LIB_PATH=paper_2002_11151_b200/$L/libxbarsim_b200.so python bench.py --config $cfg --stage-probe --steps 3 --warmup 2 2>/dev/null | tail -1)
      echo "$cfg $L $r"
    done
  done
done
