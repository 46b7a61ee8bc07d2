#!/bin/bash
# Build a libccl.so variant into abvar/<name>.so with extra -D flags (A/B runs
# on the GPU box: tools/ab_variants.sh copies each over the in-tree library).
# usage: tools/build_variant.sh <name> [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p abvar
/usr/local/cuda/bin/nvcc -O3 -std=c++17 -lineinfo -gencode arch=compute_100a,code=sm_100a \
  -Xcompiler -fPIC,-O2 -shared "$@" -I include paper_1708_08180_b200/csrc/ccl_api.cu -o abvar/$name.so
