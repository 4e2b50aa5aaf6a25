#!/bin/bash
# A/B timing of development builds build/win_*.so against the in-tree library (kbench window).
mkdir -p gpurun_out
timeout 300 python tools/kbench.py --what window > gpurun_out/kb_window.json 2>&1; echo "kb rc=$?"
for f in build/win_*.so; do [ -e "$f" ] || continue; v=$(basename $f .so)
  POLSAR_LIB_OVERRIDE=$f timeout 300 python tools/kbench.py --what window > gpurun_out/kb_$v.json 2>&1
done
for f in gpurun_out/kb_window.json gpurun_out/kb_win_*.json; do [ -e "$f" ] && echo "$f $(tr -d '\n ' < $f)"; done
true
