#!/bin/bash
# ncu --set full of the KL window's pass 1 on c5 (after a plain run of the same command)
mkdir -p gpurun_out
K="python bench.py --kernel kl --steps 3 --warmup 3"
$K > gpurun_out/bench_kl_small.json 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_window_fwd -s 1 -c 1 -o gpurun_out/prof_kl_fwd -f $K > gpurun_out/ncu_kl.log 2>&1
echo "rc=$?"
