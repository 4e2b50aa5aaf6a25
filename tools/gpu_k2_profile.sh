mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_inv_det.py tests/test_gpu_fullsize.py tests/test_gpu_blocks.py tests/test_gpu_streams.py -q -p no:cacheprovider -rf > gpurun_out/pytest_inv2.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_inv2.log
PROF="python tools/kbench.py --what k1 --rows 1000"
$PROF > /dev/null 2>&1 && /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:k_inv_det_vecIfLi1ELi0E -s 2 -c 1 -o gpurun_out/prof_k2_r02 -f $PROF > gpurun_out/ncu_k2.log 2>&1; echo "ncu rc=$?"
