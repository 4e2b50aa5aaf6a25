#!/bin/bash
set -u
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 600 python -m pytest tests/test_gpu_window.py -q -x -p no:cacheprovider > gpurun_out/pt_win.log 2>&1
CMD="python tools/kbench.py --what window"
$CMD > gpurun_out/kb_v3.json 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_window_sum_v5IffLb1 -s 1 -c 1 -o gpurun_out/prof_k3v3 -f $CMD > gpurun_out/ncu_k3v3.log 2>&1
echo "rc=$?"
POLSAR_WINDOW_VARIANT=3 python tools/kbench.py --what window > gpurun_out/kb_v3only.json 2>&1
