#!/bin/bash
# K1/K2 register-vector form vs the bulk-copy form (POLSAR_K1_VARIANT=bulk):
# parity tests under the bulk form, then kbench for both.
mkdir -p gpurun_out
POLSAR_K1_VARIANT=bulk timeout 900 python -m pytest tests/test_gpu_inv_det.py tests/test_gpu_fullsize.py tests/test_gpu_streams.py -x -q -p no:cacheprovider > gpurun_out/pt_bulk.log 2>&1; echo "pytest bulk rc=$?"
python tools/kbench.py --what k1 --rows 2500 > gpurun_out/kb_k1_vec.json 2>&1
POLSAR_K1_VARIANT=bulk python tools/kbench.py --what k1 --rows 2500 > gpurun_out/kb_k1_bulk.json 2>&1
python tools/kbench.py --what k1 --rows 2500 > gpurun_out/kb_k1_vec2.json 2>&1
echo done
