#!/bin/bash
# ncu --set full of the tensor-core window pass 1 on c5 (after a plain run of the same command)
mkdir -p gpurun_out
# (the tensor-core pass 1 is the default for fp32 storage)
K="python bench.py --kernel window --steps 3 --warmup 3"
$K > gpurun_out/bench_mma_small.json 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_window_fwd_mma -s 1 -c 1 -o gpurun_out/prof_mma_fwd -f $K > gpurun_out/ncu_mma.log 2>&1
echo "rc=$?"
