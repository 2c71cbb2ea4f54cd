#!/bin/bash
# Build the current csrc tree as an A/B variant: build/variants/<name>/libplzgpu.so
# (select it at run time with PLZGPU_LIB=build/variants/<name>/libplzgpu.so).
set -e
N=$1
R=$(cd "$(dirname "$0")/.." && pwd)
make -s -C "$R/paper_2304_07342_b200/csrc" -j8 OBJ="$R/build/variants/$N/obj" OUT="$R/build/variants/$N" \
    "$R/build/variants/$N/libplzgpu.so" > /dev/null
rm -rf "$R/build/variants/$N/obj"
echo "$R/build/variants/$N/libplzgpu.so"
