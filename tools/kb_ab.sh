#!/bin/bash
# A/B the window kernels over build/<variant>.so (tools/build_variant.sh):
#   bash tools/kb_ab.sh base u2 rb4 ...   ("base" = the in-tree library)
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then
    python tools/kbench.py --what window > gpurun_out/kb_ab_$v.json 2>&1
  else
    POLSAR_LIB_OVERRIDE=build/$v.so python tools/kbench.py --what window > gpurun_out/kb_ab_$v.json 2>&1
  fi
  echo "$v $(tr -d '\n' < gpurun_out/kb_ab_$v.json)"
done
