#!/bin/bash
# One GPU call for the default bench line and its profiles (copied into
# profiles/ afterwards): the bench line, the ncu launch list of the same
# command, the full-size K1 DRAM traffic per launch, and one `ncu --set full`
# capture each of K1, K2 and the window kernel's two passes.  Each ncu command
# runs only after the identical command has exited 0 without ncu.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
BENCH="python bench.py --steps 20 --warmup 3"
PROF="python bench.py --steps 3 --warmup 3 --rows 1000 --no-e2e --no-cpu-baseline"
SMALL="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
NCU=/usr/local/cuda/bin/ncu
$BENCH > $OUT/bench_plain.json 2> $OUT/bench_plain.err && \
  $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $BENCH > $OUT/bench_ncu_launches.log 2>&1
echo "launch list rc=$?"
# full-size c3 K1 DRAM traffic per launch (single-pass metrics, no replay)
$SMALL > $OUT/b_small.json 2>&1 && \
  $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
       --kernel-name-base mangled -k regex:k_inv_det_vec -c 6 --csv --log-file $OUT/k1_traffic_full.csv $SMALL > $OUT/ncu_traffic.log 2>&1
echo "traffic rc=$?"
$PROF > $OUT/prof_plain.json 2> $OUT/prof_plain.err && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi0ELi0E -s 2 -c 1 -o $OUT/prof_k1 -f $PROF > $OUT/ncu_k1.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi1ELi0E -s 2 -c 1 -o $OUT/prof_k2 -f $PROF > $OUT/ncu_k2.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on \
       -k regex:k_window_fwd -s 1 -c 1 -o $OUT/prof_k3_fwd -f $PROF > $OUT/ncu_k3f.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on \
       -k regex:k_window_bwd -s 1 -c 1 -o $OUT/prof_k3_bwd -f $PROF > $OUT/ncu_k3b.log 2>&1
echo "ncu full rc=$?"
