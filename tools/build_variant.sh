#!/bin/bash
# Build an alternative libnetfuse with extra nvcc defines for A/B timing:
#   tools/build_variant.sh <name> -DNF_GEMM_BUDGET_KB=96 ...
set -e
name=$1; shift
out=build/variant_$name; mkdir -p $out tools/variants
for f in paper_2009_13062_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -Ipaper_2009_13062_b200/csrc "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/variants/lib_$name.so $out/*.o -lcuda
echo tools/variants/lib_$name.so
