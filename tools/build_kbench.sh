#!/bin/bash
# build the dev micro-benchmark against a given library build (default: the in-tree one)
set -e
cd "$(dirname "$0")/.."
LIB=${1:-paper_math_0301321_b200/libib_b200.so}
D=$(dirname $(readlink -f $LIB)); B=$(basename $LIB .so)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o build_variants/kbench_${B#lib} tools/kbench.cu $(readlink -f $LIB) -Xlinker -rpath,$D
