#!/bin/bash
# Round-end style validation: the gpu test suite, smoke(), the default bench line
# (with its extras) and the reference-arm line.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; cat $OUT/smoke.log | tail -7
python bench.py --steps ${STEPS:-20} --warmup 3 > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "bench rc=$?"
python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "bench ref rc=$?"
