#!/bin/bash
# One GPU call: plain bench + ncu launch list of the same command, then one
# `ncu --set full` capture per hot kernel (each command first run without ncu).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
BENCH="python bench.py --steps 20 --warmup 3"
PROF="python bench.py --steps 3 --warmup 3 --rows 1000 --no-e2e --no-cpu-baseline"
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 200 > $OUT/clocks.csv &
SMI=$!
$BENCH > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/bench_ncu_launches.log 2>&1
echo "launch list rc=$?"
kill $SMI
$PROF > $OUT/prof_plain.json 2> $OUT/prof_plain.err && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi0ELi0E -s 2 -c 1 -o $OUT/prof_k1 -f $PROF > $OUT/ncu_k1.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi1ELi0E -s 2 -c 1 -o $OUT/prof_k2 -f $PROF > $OUT/ncu_k2.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_window_sumIfdfLi32 -s 1 -c 1 -o $OUT/prof_k3 -f $PROF > $OUT/ncu_k3.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_window_sumIfffLi32 -s 1 -c 1 -o $OUT/prof_k3_plain -f $PROF > $OUT/ncu_k3p.log 2>&1
echo "ncu full rc=$?"
