#!/bin/bash
# Bench lines of the three window kernels; the window and KL calls' launch
# lists (time, DRAM bytes, FP64 and tensor pipes, L1) and one `ncu --set full`
# capture of each one's pass 1 (each ncu command only after the same command
# exited 0 without ncu).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
for k in window nlm kl; do
  python bench.py --kernel $k --steps 10 --warmup 3 > $OUT/bench_$k.json 2> $OUT/bench_$k.err; echo "bench $k rc=$?"
done
for k in window kl; do
  K="python bench.py --kernel $k --steps 3 --warmup 3"
  $K > $OUT/bench_${k}_small.json 2>&1 && \
    $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active --clock-control none --csv \
         --log-file $OUT/launches_$k.csv $K > $OUT/ncu_${k}_launch.log 2>&1
  echo "ncu launch $k rc=$?"
  $NCU --set full --clock-control none --import-source on -k regex:k_window_fwd -s 1 -c 1 \
       -o $OUT/prof_${k}_fwd -f $K > $OUT/ncu_${k}_full.log 2>&1
  echo "ncu full $k rc=$?"
done
