#!/bin/bash
# One GPU call for the bench lines and their profiles (copied into profiles/
# afterwards, named per round): the default bench line and the reference arm;
# the ncu launch list of the same bench command; the full-size K1 DRAM traffic
# per launch; `ncu --set full` of K1 (fp32 and fp64 storage) and K2; the
# window / KL / NLM bench lines and their launch lists.  Each ncu command runs
# only after the identical command has exited 0 without ncu.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
RND=${RND:-r02}
NCU=/usr/local/cuda/bin/ncu
BENCH="python bench.py --steps 20 --warmup 3"
SMALL="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras"
$BENCH > $OUT/${RND}_bench_c3.json 2> $OUT/${RND}_bench_c3.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/${RND}_bench_c3_reference.json 2> $OUT/bref.err; echo "ref rc=$?"
for k in window kl nlm; do
  python bench.py --kernel $k --steps 10 --warmup 3 > $OUT/${RND}_bench_c5_$k.json 2> $OUT/bench_$k.err; echo "bench $k rc=$?"
done
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${RND}_launches_bench.csv $BENCH > $OUT/ncu_launches.log 2>&1
echo "launch list rc=$?"
$SMALL > $OUT/b_small.json 2>&1 && \
  $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
       --kernel-name-base mangled -k regex:k_inv_det_vec -c 6 --csv --log-file $OUT/${RND}_k1_c3_traffic.csv $SMALL > $OUT/ncu_traffic.log 2>&1
echo "traffic rc=$?"
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --config c4 > $OUT/b_c4.json 2>&1 && \
  $NCU --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
       --kernel-name-base mangled -k regex:k_inv_det_vec -c 6 --csv --log-file $OUT/${RND}_k1_c4_traffic.csv \
       python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-extras --config c4 > $OUT/ncu_traffic4.log 2>&1
echo "traffic c4 rc=$?"
P1="python tools/kbench.py --what k1 --rows 1000"
P4="python tools/kbench.py --what c4 --rows 1000"
$P1 > /dev/null 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi0ELi0E -s 2 -c 1 -o $OUT/${RND}_prof_k1 -f $P1 > $OUT/ncu_k1.log 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIfLi1ELi0E -s 2 -c 1 -o $OUT/${RND}_prof_k2 -f $P1 > $OUT/ncu_k2.log 2>&1
echo "ncu k1/k2 rc=$?"
$P4 > /dev/null 2>&1 && \
  $NCU --set full --clock-control none --import-source on --kernel-name-base mangled \
       -k regex:k_inv_det_vecIdLi0ELi1EE -s 2 -c 1 -o $OUT/${RND}_prof_k1_f64 -f $P4 > $OUT/ncu_k1f64.log 2>&1
echo "ncu k1 f64 rc=$?"
for k in window kl nlm; do
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed \
       --clock-control none --csv --log-file $OUT/${RND}_launches_$k.csv python bench.py --kernel $k --steps 3 --warmup 3 > $OUT/ncu_$k.log 2>&1
  echo "launch list $k rc=$?"
done
