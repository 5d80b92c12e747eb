#!/bin/bash
# build a libara variant with extra -D flags for A/B timing:
#   tools/build_variant.sh NAME -DFOO=1 ...   -> gpurun_variants/NAME.so
mkdir -p gpurun_variants
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O2 -shared "$@" \
  -o gpurun_variants/$name.so paper_1310_2274_b200/csrc/*.cu
