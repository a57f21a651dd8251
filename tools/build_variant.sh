#!/bin/bash
# Build a variant of libsplatct.so with extra nvcc defines for fvr.cu, as
# paper_2411_04844_b200/_lib/libsplatct_<name>.so (measurement sweeps).
#   tools/build_variant.sh <name> -DMACRO=VALUE ...
set -e
cd "$(dirname "$0")/.."
L=paper_2411_04844_b200/_lib
name=$1; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include -Xptxas -v "$@" \
  -c paper_2411_04844_b200/csrc/fvr.cu -o /tmp/fvr_$name.o 2> /tmp/fvr_$name.ptxas
objs=$(ls $L/*.o | grep -v "/fvr.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/libsplatct_$name.so /tmp/fvr_$name.o $objs
echo $L/libsplatct_$name.so
