#!/bin/bash
# Developer tool: the round's measurement sweep on one B200 (gpurun), every
# output under gpurun_out/final/.
#   gpurun --timeout 3000 -- bash tools/final_round.sh
set -u
O=gpurun_out/final
mkdir -p $O
nvidia-smi -q -d POWER,CLOCK > $O/smi.txt 2>&1
lscpu > $O/lscpu.txt 2>&1; nproc > $O/nproc.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/gpu_tests.log 2>&1; echo "gpu tests rc=$?" >> $O/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err; cp gpurun_out/clocks_rank0.csv $O/clocks_bench.csv
timeout 600 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 python tools/cpu_table.py > $O/cpu_table.json 2> $O/cpu_table.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c5.csv $CMD > $O/ncu_launches.log 2>&1
echo "launch list rc=$?" >> $O/ncu_launches.log
ncu --set full --clock-control none --import-source on -k 'regex:k_fwd_tc|k_bwd_tc|k_dw_tc|k_update' \
    -s 12 -c 4 -o $O/prof_c5 -f $CMD > $O/ncu_full.log 2>&1
echo "full rc=$?" >> $O/ncu_full.log
ncu -i $O/prof_c5.ncu-rep --page raw --csv > $O/prof_c5_raw.csv 2>/dev/null
for k in k_fwd_tc k_bwd_tc k_update; do python tools/ncu_stalls.py $O/prof_c5.ncu-rep $k 25 > $O/stalls_c5_$k.txt 2>&1; done
rm -f $O/prof_c5.ncu-rep
CMD2="python bench.py --config c2-4096 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv $CMD2 > $O/ncu_launches2.log 2>&1
ncu --set full --clock-control none --import-source on -k 'regex:k_fwd_tc|k_bwd_tc|k_dw_tc|k_update' \
    -s 12 -c 4 -o $O/prof_c2 -f $CMD2 > $O/ncu_full2.log 2>&1
ncu -i $O/prof_c2.ncu-rep --page raw --csv > $O/prof_c2_raw.csv 2>/dev/null
for k in k_fwd_tc k_bwd_tc k_update; do python tools/ncu_stalls.py $O/prof_c2.ncu-rep $k 25 > $O/stalls_c2_$k.txt 2>&1; done
rm -f $O/prof_c2.ncu-rep
du -sh $O
echo done
