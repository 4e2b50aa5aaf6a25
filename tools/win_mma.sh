#!/bin/bash
# Tensor-core window pass 1 (POLSAR_WINDOW_MMA=1) against the default: window
# parity tests under the variant, then kbench timings of both.
mkdir -p gpurun_out
POLSAR_WINDOW_MMA=1 timeout 900 python -m pytest tests/test_gpu_window.py -q -p no:cacheprovider -x -k "not variant_subprocess" > gpurun_out/win_mma_tests.log 2>&1; echo "mma tests rc=$?"
tail -5 gpurun_out/win_mma_tests.log
POLSAR_WINDOW_MMA=1 timeout 300 python tools/kbench.py --what window > gpurun_out/kb_mma.json 2>&1; echo "kb mma rc=$?"
timeout 300 python tools/kbench.py --what window > gpurun_out/kb_default.json 2>&1; echo "kb default rc=$?"
for f in gpurun_out/kb_default.json gpurun_out/kb_mma.json; do echo "$f $(tr -d '\n ' < $f)"; done
