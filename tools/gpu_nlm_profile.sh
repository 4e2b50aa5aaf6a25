#!/bin/bash
# Bench lines of the three window kernels, then the NLM call's launch list and
# one `ncu --set full` capture of its gather pass (each ncu command only after
# the same command exited 0 without ncu).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
for k in window nlm kl; do
  python bench.py --kernel $k --steps 10 --warmup 3 > $OUT/bench_$k.json 2> $OUT/bench_$k.err; echo "bench $k rc=$?"
done
K="python bench.py --kernel nlm --steps 3 --warmup 3"
$K > $OUT/bench_nlm_small.json 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv \
       --log-file $OUT/launches_nlm.csv $K > $OUT/ncu_nlm_launch.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:k_nlm_gather -s 1 -c 1 \
       -o $OUT/prof_nlm_gather -f $K > $OUT/ncu_nlm_full.log 2>&1
echo "ncu rc=$?"
