#!/bin/bash
# ncu capture of the window kernel (c5) after a plain run of the same command.
set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CMD="python tools/kbench.py --what window"
$CMD > gpurun_out/kb_plain.json 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_window_sumIfdf -s 1 -c 1 -o gpurun_out/prof_k3v2 -f $CMD > gpurun_out/ncu_k3v2.log 2>&1
echo "k3 rc=$?"
# full-size c3 K1 DRAM traffic per launch (single-pass metrics, no replay)
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
$B > gpurun_out/b_small.json 2>&1 && \
  $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
       --kernel-name-base mangled -k regex:k_inv_det_vec -c 6 --csv --log-file gpurun_out/k1_traffic_full.csv $B > gpurun_out/ncu_traffic.log 2>&1
echo "traffic rc=$?"
