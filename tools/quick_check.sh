#!/bin/bash
# GPU iteration loop (through gpurun): parity suite, then C3 per-layer and
# headline timings.  Usage: gpurun -- bash tools/quick_check.sh TAG
TAG=${1:-qc}
mkdir -p gpurun_out/$TAG
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/$TAG/pytest.log 2>&1
echo "pytest rc=$?"; tail -n 2 gpurun_out/$TAG/pytest.log
for L in 0 1 7 8 13 14; do timeout 120 python bench.py --config c3 --layer $L --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak 2>/dev/null | tail -n 1 >> gpurun_out/$TAG/c3_layers.jsonl; done
timeout 300 python bench.py --config c3 --all-layers --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 > gpurun_out/$TAG/c3_all.json
timeout 300 python bench.py --config c4 --all-layers --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -n 1 > gpurun_out/$TAG/c4_all.json
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -n 1 > gpurun_out/$TAG/c2.json
echo done
