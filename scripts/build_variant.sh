#!/bin/bash
# Build a variant of libdcdg.so for A/B timing (kernel lab, not the product):
#   scripts/build_variant.sh NAME [SRC_DIR] [-DFLAG=...]   -> vlib/NAME/libdcdg.so
# SRC_DIR defaults to the working tree's csrc; pass e.g. a `git worktree` copy.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
SRC=$ROOT/paper_1902_08653_b200/csrc
INC=$ROOT/include
if [ $# -gt 0 ] && [ -d "$1" ]; then SRC=$1/paper_1902_08653_b200/csrc; INC=$1/include; shift; fi
OUT=$ROOT/vlib/$NAME; mkdir -p "$OUT"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++20 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr"
nvcc $F "$@" -I "$INC" -I "$SRC" -c "$SRC/dcdg.cu" -o "$OUT/dcdg.o" &
nvcc -x cu $F "$@" -I "$INC" -I "$SRC" -c "$SRC/dcd_gpu.cpp" -o "$OUT/gpu.o" &
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -o "$OUT/libdcdg.so" "$OUT/dcdg.o" "$OUT/gpu.o" -lcudart
rm -f "$OUT"/*.o
echo "$OUT/libdcdg.so"
