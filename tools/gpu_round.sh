#!/bin/bash
# Full GPU check: the gpu test suite, smoke(), the default bench line, the
# window-kernel bench lines, and the ncu evidence for the window kernels
# (launch list of the same bench command, then --set full of both passes).
set -u
mkdir -p gpurun_out
OUT=gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
python bench.py --steps 20 --warmup 3 > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
for k in window nlm kl; do
  python bench.py --kernel $k --steps 10 --warmup 3 > $OUT/bench_$k.json 2> $OUT/bench_$k.err; echo "bench $k rc=$?"
done
W="python bench.py --kernel window --steps 3 --warmup 3"
$W > $OUT/bench_w_small.json 2>&1 && \
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
       --log-file $OUT/launches_window.csv $W > $OUT/ncu_w_launch.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:k_window_fwd -s 1 -c 1 \
       -o $OUT/prof_k3_fwd -f $W > $OUT/ncu_k3f.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on -k regex:k_window_bwd -s 1 -c 1 \
       -o $OUT/prof_k3_bwd -f $W > $OUT/ncu_k3b.log 2>&1
echo "ncu rc=$?"
