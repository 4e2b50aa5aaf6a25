#!/bin/bash
# Window-family GPU tests + kbench + the window bench line (after a kernel change)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_window.py tests/test_gpu_nlm.py tests/test_gpu_kl.py tests/test_gpu_fullsize.py -q -p no:cacheprovider > gpurun_out/wc_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/wc_tests.log
timeout 300 python tools/kbench.py --what window > gpurun_out/wc_kb.json 2>&1; echo "kb rc=$? $(tr -d '\n ' < gpurun_out/wc_kb.json)"
timeout 300 python bench.py --kernel window --steps 10 --warmup 3 > gpurun_out/wc_bench_window.json 2> gpurun_out/wc_bench_window.err; echo "bench rc=$?"; cat gpurun_out/wc_bench_window.json
