#!/bin/bash
mkdir -p gpurun_out
K="python tools/kbench.py --what nlm"
$K > gpurun_out/kb_plain.json 2>&1 && \
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_nlm_gather -s 1 -c 1 -o gpurun_out/prof_nlm_gather -f $K > gpurun_out/ncu_nlm.log 2>&1
echo "rc=$?"
