#!/bin/bash
# Developer tool: build the library of a git revision (default HEAD) into
# paper_2002_11151_b200/_lib_base/ for A/B timing against the working tree
# (load it with XBS_LIB_PATH=paper_2002_11151_b200/_lib_base/libxbarsim_b200.so).
set -e
REV=${1:-HEAD}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
T=$(mktemp -d)
git -C "$ROOT" archive "$REV" paper_2002_11151_b200/csrc include | tar -x -C "$T"
cd "$T/paper_2002_11151_b200"
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off"
mkdir -p b
pids=()
for f in csrc/*.cu; do $NV -c $f -o b/$(basename $f .cu).o & pids+=($!); done
for p in "${pids[@]}"; do wait $p; done
mkdir -p "$ROOT/paper_2002_11151_b200/_lib_base"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$ROOT/paper_2002_11151_b200/_lib_base/libxbarsim_b200.so" b/*.o -lcudart_static -lrt -ldl -lpthread
rm -rf "$T"
echo "built _lib_base from $REV"
