#!/bin/bash
# Developer tool: build the library with extra compile flags (perf
# experiments, e.g. -DXBS_STUB_MMA) into paper_2002_11151_b200/_lib_<name>/;
# load it with XBS_LIB_PATH=paper_2002_11151_b200/_lib_<name>/libxbarsim_b200.so.
set -e
NAME=$1; shift
cd "$(dirname "$0")/../paper_2002_11151_b200"
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC -Xcompiler -ffp-contract=off $*"
mkdir -p _build_$NAME _lib_$NAME
pids=()
for f in csrc/*.cu; do b=$(basename $f .cu); $NV -c $f -o _build_$NAME/$b.o & pids+=($!); done
for p in "${pids[@]}"; do wait $p; done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _lib_$NAME/libxbarsim_b200.so _build_$NAME/*.o -lcudart_static -lrt -ldl -lpthread
echo built _lib_$NAME
