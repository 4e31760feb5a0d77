#!/bin/sh
# Bounds-checked build of the library (device-side LP_CHECK on derived indices) for
# running the GPU tests against: LP_LIB=$PWD/build_checks/liblp_b200.so pytest -m gpu
set -e
cd "$(dirname "$0")/.."
mkdir -p build_checks
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC,-O3 -shared -DLP_CHECKS -o build_checks/liblp_b200.so \
  paper_2009_10247_b200/csrc/abi.cu paper_2009_10247_b200/csrc/kernels.cu paper_2009_10247_b200/csrc/encode.cpp
