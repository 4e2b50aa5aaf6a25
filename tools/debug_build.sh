#!/bin/bash
# Build libpolsar with device-side bounds asserts (POLSAR_DEBUG_BOUNDS) into
# build/debug/ and run the GPU suites against it (POLSAR_LIB_OVERRIDE).
set -e
cd "$(dirname "$0")/.."
mkdir -p build/debug
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared \
  -Xcompiler -fPIC -I include -DPOLSAR_DEBUG_BOUNDS \
  paper_1807_08084_b200/csrc/abi.cu paper_1807_08084_b200/csrc/inv_det.cu \
  paper_1807_08084_b200/csrc/window.cu paper_1807_08084_b200/csrc/nlm.cu paper_1807_08084_b200/csrc/checksum.cu \
  -o build/debug/libpolsar_debug.so
