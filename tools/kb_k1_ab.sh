#!/bin/bash
# kbench (K1 / K2 on a c3 slice, fp32 and fp64 storage) of the in-tree library
# and of every build/<prefix>*.so variant (POLSAR_LIB_OVERRIDE), twice.
#   bash tools/kb_k1_ab.sh <prefix> [rows]
cd "$(dirname "$0")/.."
pre=${1:-k2_}; rows=${2:-5000}
for rep in 1 2; do
  echo "== base rep $rep"; timeout 300 python tools/kbench.py --what k1 --rows $rows | tr -d '\n'; echo
  for so in build/${pre}*.so; do
    echo "== $so rep $rep"; POLSAR_LIB_OVERRIDE=$so timeout 300 python tools/kbench.py --what k1 --rows $rows | tr -d '\n'; echo
  done
done
