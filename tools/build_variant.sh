#!/bin/bash
# Build an A/B variant of libpolsar with extra -D flags into build/<name>.so
# (load it with POLSAR_LIB_OVERRIDE=build/<name>.so).  Usage:
#   tools/build_variant.sh <name> -DPOLSAR_SYM_RB=4 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -I include -Xptxas -v "$@" \
  paper_1807_08084_b200/csrc/abi.cu paper_1807_08084_b200/csrc/inv_det.cu \
  paper_1807_08084_b200/csrc/window.cu paper_1807_08084_b200/csrc/nlm.cu paper_1807_08084_b200/csrc/checksum.cu \
  -o build/$name.so 2> build/$name.log
grep -A2 "k_window_fwd" build/$name.log | grep -E "registers|spill" || true
