#!/bin/bash
# Update-kernel A/B through gpurun: update-touching GPU tests, then the
# update stage of C5 / C2 / C4-layer / C3-layer with the bulk-copy kernel and
# the register-staged one (XBS_UPDATE_LEGACY=1).  Usage: gpurun -- bash tools/upd_ab.sh TAG
TAG=${1:-upd}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests -m gpu -x -q -k "update or stats or free or parity_gpu or mlp or golden" > gpurun_out/$TAG/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 3 gpurun_out/$TAG/pytest.log
for cfg in "c5" "c2-4096" "c4 --layer 16" "c3 --layer 7"; do
  for leg in 0 1; do
    XBS_UPDATE_LEGACY=$leg timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-others --no-cpu-baseline --no-e2e --no-peak 2>gpurun_out/$TAG/err.log | tail -n 1 | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); u=d['roofline_stages']['update']; print('$cfg legacy=$leg', d['config']['workload'], 'ms/step %.3f'%d['ms_per_step'], 'upd ms %.4f frac %.3f'%(u['ms'],u['frac']))" >> gpurun_out/$TAG/ab.txt 2>&1
  done
done
cat gpurun_out/$TAG/ab.txt
