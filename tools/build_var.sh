#!/bin/bash
# Alternative libnetfuse build with extra nvcc defines (A/B timing on the box):
#   tools/build_var.sh <name> -DNF_...=... ; NF_LIB_PATH=varlib/lib_<name>.so python ...
set -e
name=$1; shift
out=build/var_$name; mkdir -p $out varlib
for f in paper_2009_13062_b200/csrc/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude -Ipaper_2009_13062_b200/csrc "$@" -c $f -o $out/$(basename $f .cu).o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o varlib/lib_$name.so $out/*.o -lcuda
echo varlib/lib_$name.so
