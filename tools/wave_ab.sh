#!/bin/bash
# Developer tool: wave alignment / grouped unit order of the VMM producers
# (XBS_WAVE_SYNC, XBS_WAVE_FINE, XBS_WAVE_GROUP) A/B on C5 -- per-stage event
# times, interleaved, then DRAM bytes per launch (ncu).
#   gpurun --timeout 2400 -- bash tools/wave_ab.sh
O=gpurun_out/wave_ab
mkdir -p $O
VARS=${VARS:-"off sync sync,fine sync,g2 sync,g4 sync,fine,g2 sync,fine,g4"}
setv() {
  unset XBS_WAVE_SYNC XBS_WAVE_ANORM XBS_WAVE_GROUP
  case ",$1," in *,sync,*) export XBS_WAVE_SYNC=1;; esac
  case ",$1," in *,anorm,*) export XBS_WAVE_ANORM=1;; esac
  case ",$1," in *,g2,*) export XBS_WAVE_GROUP=2;; esac
  case ",$1," in *,g3,*) export XBS_WAVE_GROUP=3;; esac
  case ",$1," in *,g4,*) export XBS_WAVE_GROUP=4;; esac
  case ",$1," in *,g8,*) export XBS_WAVE_GROUP=8;; esac
}
CMD="python bench.py --config c5 --stage-probe --steps 5 --warmup 3"
for r in $(seq ${ROUNDS:-2}); do
  for V in $VARS; do
    setv $V
    line=$(timeout 300 $CMD 2>>$O/err.log | tail -n 1)
    echo "{\"round\": $r, \"variant\": \"$V\", \"stages\": $line}" >> $O/stages3.jsonl
  done
done
NCU="ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.max --clock-control none -k regex:k_fwd_tc|k_bwd_tc -s 6 -c 2 --csv"
for V in $VARS; do
  setv $V
  timeout 600 $NCU --log-file $O/ncu3_$V.csv python bench.py --config c5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-peak --no-others > $O/ncu3_$V.log 2>&1
done
echo done
