#!/bin/bash
# ncu --set full of the update kernel (bulk-copy and register-staged) on one config.
# Usage: gpurun -- bash tools/upd_ncu.sh TAG CONFIG
TAG=${1:-updncu}; CFG=${2:-c2-4096}
mkdir -p gpurun_out/$TAG
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others"
for leg in 0 1; do
  XBS_UPDATE_LEGACY=$leg timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_update' \
    -s 2 -c 1 -o gpurun_out/$TAG/upd_${CFG}_legacy$leg -f $CMD > gpurun_out/$TAG/ncu_$leg.log 2>&1
  echo "leg $leg rc=$?"
done
