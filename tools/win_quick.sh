#!/bin/bash
# Window-kernel development check: window/NLM/KL parity tests, then kbench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_window.py tests/test_gpu_nlm.py tests/test_gpu_kl.py -q -p no:cacheprovider -x > gpurun_out/win_tests.log 2>&1; echo "tests rc=$?"
timeout 300 python tools/kbench.py --what window > gpurun_out/kb_window.json 2>&1; echo "kb rc=$?"
for f in build/win_*.so; do [ -e "$f" ] || continue; v=$(basename $f .so)
  POLSAR_LIB_OVERRIDE=$f timeout 300 python tools/kbench.py --what window > gpurun_out/kb_$v.json 2>&1
done
for f in gpurun_out/kb_window.json gpurun_out/kb_win_*.json; do [ -e "$f" ] && echo "$f $(tr -d '\n ' < $f)"; done
