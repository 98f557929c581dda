#!/bin/bash
# Build an A/B variant of liboscar.so with extra nvcc defines: tools/build_variant.sh NAME -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_ab
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -Iinclude -Ipaper_2605_17757_b200/csrc --expt-relaxed-constexpr \
  "$@" -shared -o build_ab/liboscar_$name.so paper_2605_17757_b200/csrc/*.cu -lcudart
