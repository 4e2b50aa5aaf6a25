#!/bin/bash
# NLM symmetric form (pass 1 + gather) vs the direct form: parity tests under
# both, kbench timings, and an ncu launch list of the symmetric call.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_nlm.py tests/test_gpu_window.py -q -p no:cacheprovider -x > $OUT/nlm_tests_sym.log 2>&1; echo "tests sym rc=$?"
POLSAR_NLM_VARIANT=direct timeout 600 python -m pytest tests/test_gpu_nlm.py -q -p no:cacheprovider -x > $OUT/nlm_tests_direct.log 2>&1; echo "tests direct rc=$?"
python tools/kbench.py --what window > $OUT/kb_sym.json 2>&1; echo "kb sym rc=$?"
POLSAR_NLM_VARIANT=direct python tools/kbench.py --what window > $OUT/kb_direct.json 2>&1; echo "kb direct rc=$?"
K="python bench.py --kernel nlm --steps 3 --warmup 3"
$K > $OUT/bench_nlm_sym.json 2> $OUT/bench_nlm_sym.err && \
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none --csv \
       --log-file $OUT/launches_nlm_sym.csv $K > $OUT/ncu_nlm_launch.log 2>&1
echo "ncu rc=$?"
