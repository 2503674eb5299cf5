#!/bin/bash
# A/B builds that differ in engine.cu and/or compile-time knobs:
#   tools/build_engine_variants.sh tag=/path/engine.cu[@"-DHB_WARPS=14 -DHB_EPI=1"] ...
# (each compiled against the current csrc/ headers, include/ and the other sources)
set -e
cd "$(dirname "$0")/../paper_2603_26576_b200"
mkdir -p variants
for spec in "$@"; do
  tag=${spec%%=*}; rest=${spec#*=}; src=${rest%%@*}; flags=""
  [[ "$rest" == *@* ]] && flags=${rest#*@}
  d=$(mktemp -d); mkdir -p "$d"/p/csrc "$d"/include
  cp csrc/* "$d"/p/csrc/; cp ../include/* "$d"/include/; cp "$src" "$d"/p/csrc/engine.cu
  c="$d"/p/csrc
  (nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -diag-suppress 550 $flags \
    $c/engine.cu $c/engine_cols.cu $c/engine_long.cu $c/gen.cu $c/sort.cu $c/regions.cu $c/intervals.cu $c/transfer.cu $c/transfer_enc.cpp $c/capi.cu $c/ingest.cpp \
    -o variants/libheteff_b200_$tag.so && rm -rf "$d") &
done
wait
