#!/usr/bin/env bash
# Build a variant of the engine library for same-box A/B timing:
#   tools/build_variant.sh NAME CSRC_DIR [extra nvcc flags]
# -> paper_2508_08343_b200/lib/ab/libloratwin_gpu_NAME.so
set -eu
NAME=$1; SRC=$2; shift 2
OBJ=$(mktemp -d)
mkdir -p paper_2508_08343_b200/lib/ab
for U in "$SRC"/*.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --fmad=false -DLT_NO_CONTRACT \
    -Xcompiler -fPIC,-ffp-contract=off "$@" -Iinclude -I"$SRC" -c -o "$OBJ/$(basename "$U" .cu).o" "$U" 2>/dev/null &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2508_08343_b200/lib/ab/libloratwin_gpu_$NAME.so "$OBJ"/*.o
rm -rf "$OBJ"
echo built $NAME
