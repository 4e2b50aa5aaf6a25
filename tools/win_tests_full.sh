#!/bin/bash
# Window-kernel GPU suites, product library then the bounds-assert debug build.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_window.py tests/test_gpu_kl.py tests/test_gpu_nlm.py -q -p no:cacheprovider > gpurun_out/win_tests_full.log 2>&1; echo "tests rc=$?"
POLSAR_LIB_OVERRIDE=build/debug/libpolsar_debug.so timeout 1200 python -m pytest tests/test_gpu_window.py tests/test_gpu_kl.py -q -p no:cacheprovider -k "not c5" > gpurun_out/win_tests_debug.log 2>&1; echo "debug tests rc=$?"
