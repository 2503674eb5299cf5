#!/bin/bash
# build tuning variants of the engine library (compile-time tile knobs)
set -e
cd "$(dirname "$0")/../paper_2603_26576_b200"
mkdir -p variants
for spec in "$@"; do
  tag=${spec%%:*}; flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -diag-suppress 550 $flags \
    csrc/engine.cu csrc/engine_cols.cu csrc/engine_long.cu csrc/gen.cu csrc/sort.cu csrc/regions.cu csrc/intervals.cu csrc/transfer.cu csrc/transfer_enc.cpp csrc/capi.cu csrc/ingest.cpp -o variants/libheteff_b200_$tag.so &
done
wait
