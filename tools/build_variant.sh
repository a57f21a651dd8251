#!/bin/bash
# Build a variant of libsplatct.so with extra nvcc defines for one source
# (default fvr.cu), as paper_2411_04844_b200/_lib/libsplatct_<name>.so
# (measurement sweeps; the variant .so is copied over libsplatct.so on the box).
#   tools/build_variant.sh <name> [-f <source.cu>] -DMACRO=VALUE ...
set -e
cd "$(dirname "$0")/.."
L=paper_2411_04844_b200/_lib
name=$1; shift
src=fvr.cu
if [ "$1" = "-f" ]; then src=$2; shift 2; fi
base=${src%.cu}
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I include -Xptxas -v "$@" \
  -c paper_2411_04844_b200/csrc/$src -o /tmp/${base}_$name.o 2> /tmp/${base}_$name.ptxas
objs=$(ls $L/*.o | grep -v "/$base.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $L/libsplatct_$name.so /tmp/${base}_$name.o $objs
echo $L/libsplatct_$name.so
