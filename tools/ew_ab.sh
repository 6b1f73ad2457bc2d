#!/bin/bash
# Developer tool: forward epilogue warps (XBS_FWD_EW = 8 | 16) A/B: parity
# subset with 16 warps, then per-stage event times, interleaved.
#   gpurun --timeout 2400 -- bash tools/ew_ab.sh
O=gpurun_out/ew_ab
mkdir -p $O
XBS_FWD_EW=16 timeout 900 python -m pytest tests/test_parity_gpu.py tests/test_fuzz_gpu.py tests/test_golden.py tests/test_wide_layers_gpu.py tests/test_precision_gpu.py tests/test_conv_gpu.py -x -q -m gpu > $O/pytest_ew16.log 2>&1
echo "pytest ew16 rc=$?"; tail -n 2 $O/pytest_ew16.log
for r in 1 2; do
  for C in c5 c2-4096 c4:1 c4:6 c3:1; do
    for V in 8 16 16e; do
      cfg=${C%%:*}; layer=0; [ "$C" != "$cfg" ] && layer=${C##*:}
      unset XBS_LIB_PATH; [ $V = 16e ] && export XBS_LIB_PATH=paper_2002_11151_b200/_lib_early/libxbarsim_b200.so
      line=$(XBS_FWD_EW=${V%e} timeout 300 python bench.py --config $cfg --layer $layer --stage-probe --steps 5 --warmup 3 2>>$O/err.log | tail -n 1)
      echo "{\"round\": $r, \"ew\": \"$V\", \"case\": \"$C\", \"stages\": $line}" >> $O/stages.jsonl
    done
  done
done
echo done
