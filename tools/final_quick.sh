#!/bin/bash
# Developer tool: tests + smoke + default bench + reference arm (no ncu);
# outputs under gpurun_out/final5/.
O=gpurun_out/final5
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; cp gpurun_out/clocks_rank0.csv $O/clocks_bench.csv
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
echo done
