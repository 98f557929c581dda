#!/bin/bash
# Build an A/B variant of liboscar.so with extra nvcc defines (parallel, objects under build/):
#   tools/build_variant.sh NAME -DFOO=1 ...   ->  build_ab/liboscar_NAME.so
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build_ab
make -s -j8 OBJDIR=build/v_$name LIB=build_ab/liboscar_$name.so EXTRA_NVFLAGS="$*" 2>&1 | grep -v spill || true
ls -la build_ab/liboscar_$name.so
