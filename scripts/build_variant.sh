#!/bin/bash
# Build a variant of libaac.so with extra nvcc flags (experiments; A/B with scripts/ab_multi.sh).
# usage: bash scripts/build_variant.sh OUT.so [nvcc flags...]
set -e
OUT=$1; shift
D=$(dirname "$0")/..
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -shared "$@" -o "$OUT" $D/paper_2506_03947_b200/csrc/aac.cu -ldl
