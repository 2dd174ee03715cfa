#!/bin/bash
# A/B variant build (diagnostic): abtest/<name>/libjagged_b200.so = the current objects with one kernel source
# swapped for a variant file.  tools/ab_build.sh <name> <variant.cu> <replaces: e.g. attn_bwd_sm100.cu> [nvcc defs]
# Select it at run time with JG_LIB_PATH=abtest/<name>/libjagged_b200.so.
set -e
name=$1; src=$2; repl=$3; shift 3
root=$(cd "$(dirname "$0")/.." && pwd)
out=$root/abtest/$name; mkdir -p "$out"
csrc=$root/paper_2409_15373_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr \
  -I "$root/include" -I "$csrc" "$@" -c "$src" -o "$out/variant.o"
objs=$(ls "$root"/paper_2409_15373_b200/_build/*.o | grep -v "/$repl.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out/libjagged_b200.so" $objs "$out/variant.o" -lcuda
echo "$out/libjagged_b200.so"
