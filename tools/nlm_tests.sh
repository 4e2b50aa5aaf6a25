#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nlm.py tests/test_gpu_window.py tests/test_gpu_kl.py -q -p no:cacheprovider > gpurun_out/nlm_tests.log 2>&1; echo "tests rc=$?"
POLSAR_LIB_OVERRIDE=build/debug/libpolsar_debug.so timeout 900 python -m pytest tests/test_gpu_nlm.py -q -p no:cacheprovider > gpurun_out/nlm_tests_debug.log 2>&1; echo "debug tests rc=$?"
