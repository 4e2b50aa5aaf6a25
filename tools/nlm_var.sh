#!/bin/bash
# A/B of NLM gather variants (build/nlm_*.so from tools/build_variant.sh):
# timing on c5 and bit-identity against the default build, then the NLM tests.
set -u
mkdir -p gpurun_out
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_nlm.py tests/test_gpu_window.py tests/test_gpu_kl.py -q -p no:cacheprovider -x > $OUT/nlm_tests_sym.log 2>&1; echo "tests rc=$?"
rm -f /tmp/nlm_ref.pt; timeout 300 python tools/kbench.py --what nlm --ref /tmp/nlm_ref.pt > $OUT/kbv_default.json 2>&1
for f in build/nlm_*.so; do v=$(basename $f .so)
  POLSAR_LIB_OVERRIDE=$f timeout 300 python tools/kbench.py --what nlm --ref /tmp/nlm_ref.pt > $OUT/kbv_$v.json 2>&1
done
for f in $OUT/kbv_*.json; do echo "$f $(tr -d '\n' < $f)"; done
