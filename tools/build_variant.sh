#!/bin/bash
# Build an experimental variant of the engine (extra -D flags) into
# build/var/<name>.so for A/B timing (load it with KCB200_LIB / KCB200_LIB_FAST).
# usage: tools/build_variant.sh NAME [-DFOO=1 ...]
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/var
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -shared \
  -Xcompiler -fPIC -Xcompiler -ffp-contract=off "$@" -o build/var/$name.so \
  paper_2010_00626_b200/csrc/kc_engine.cu
