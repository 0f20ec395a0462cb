#!/bin/bash
# Build experimental variants of the library (tuning sweep): build_variants/lib_<tag>.so
set -e
cd "$(dirname "$0")/.."
for v in "$@"; do
  IFS=: read tag flags <<< "$v"
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden -shared --expt-relaxed-constexpr $flags -I include paper_2412_11614_b200/csrc/abi.cu paper_2412_11614_b200/csrc/kernels.cu -o build_variants/lib_$tag.so -Xptxas -v 2> build_variants/ptxas_$tag.txt
  echo "$tag: $(grep -A2 'integrand_kernelILb0ELi0' build_variants/ptxas_$tag.txt | tail -2 | tr '\n' ' ')"
done
