mkdir -p gpurun_out
for L in 0 1 7 8 13 14; do timeout 120 python bench.py --config c3 --layer $L --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak >> gpurun_out/c3_layers.jsonl 2>>gpurun_out/c3_layers.err; done
for L in 0 1 5 6 10 11 15 16 20; do timeout 120 python bench.py --config c4 --layer $L --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak >> gpurun_out/c4_layers.jsonl 2>>gpurun_out/c4_layers.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_c3l1.csv python bench.py --config c3 --layer 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak > /dev/null 2>&1
echo done
