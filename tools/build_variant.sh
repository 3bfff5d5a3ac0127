#!/bin/bash
# Build a libplora variant with extra -D defines into build/libplora_<tag>.so (A/B experiments;
# select at run time with PLORA_LIB=build/libplora_<tag>.so).  Usage: tools/build_variant.sh tag -DX=1 ...
set -e
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p build
P=paper_2508_02932_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -shared --expt-relaxed-constexpr "$@" -I include -o build/libplora_$TAG.so \
  $P/plora_abi.cu $P/adamw.cu $P/elementwise.cu $P/meta.cpp $P/tp_nccl.cpp -ldl
echo "build/libplora_$TAG.so"
