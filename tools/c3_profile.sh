mkdir -p gpurun_out
rm -f gpurun_out/c3_layers.jsonl
for L in 0 1 7 8 13 14 19; do timeout 120 python bench.py --config c3 --layer $L --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-peak >> gpurun_out/c3_layers.jsonl 2>>gpurun_out/c3_layers.err; done
CMD="python bench.py --config c3 --layer 1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak"
timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:k_fwd_tc|k_bwd_tc' -s 6 -c 2 -o gpurun_out/prof_c3l1 -f $CMD > gpurun_out/ncu_c3.log 2>&1
echo "ncu rc=$?"
