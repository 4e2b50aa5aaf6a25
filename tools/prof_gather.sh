mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
CMD="python tools/kbench.py --what window"
$CMD > gpurun_out/kb_g.json 2>&1 && \
$NCU --set full --import-source on --clock-control none -k regex:k_nlm_gather -c 1 -o gpurun_out/gather_full -f $CMD > gpurun_out/gather_ncu.log 2>&1
echo "rc=$?"
