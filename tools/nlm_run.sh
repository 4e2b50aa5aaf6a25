mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_nlm.py tests/test_gpu_window.py -x -q > gpurun_out/pt_nlm.log 2>&1; echo "pytest rc=$?"
python tools/kbench.py --what window > gpurun_out/kb_nlm_sym.json 2>&1
POLSAR_WINDOW_VARIANT=2 python tools/kbench.py --what window > gpurun_out/kb_nlm_v2.json 2>&1
