mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_window.py tests/test_gpu_streams.py -q -p no:cacheprovider -x > gpurun_out/pt_sym.log 2>&1
python tools/kbench.py --what window > gpurun_out/kb_sym.json 2>&1
POLSAR_WINDOW_VARIANT=2 python tools/kbench.py --what window > gpurun_out/kb_v2.json 2>&1
echo done
