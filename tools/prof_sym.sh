mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
python -m pytest tests/test_gpu_window.py tests/test_gpu_streams.py tests/test_gpu_kl.py tests/test_gpu_nlm.py -x -q > gpurun_out/pt_sym.log 2>&1; echo "pytest rc=$?"
CMD="python tools/kbench.py --what window"
$CMD > gpurun_out/kb_sym.json 2>&1 && \
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/sym_launches.csv $CMD > gpurun_out/sym_ncu.log 2>&1
echo "rc=$?"
