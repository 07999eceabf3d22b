#!/bin/bash
# Kernel experiment: rebuild one source with extra -D flags and link an
# alternative library tools/_exp/<name>.so from the regular objects (run
# `python -m paper_2303_00301_b200.build` first).  Use with
# AUXMC_LIB_PATH=tools/_exp/<name>.so.   usage: tools/exp_build.sh name src.cu -DFOO=1 ...
set -e
cd "$(dirname "$0")/.."
name=$1; src=$2; shift 2
mkdir -p tools/_exp
B=paper_2303_00301_b200/build
stem=$(basename "$src" .cu)
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
  -Xcompiler -fPIC --expt-relaxed-constexpr -I include -I paper_2303_00301_b200/csrc "$@" \
  -c paper_2303_00301_b200/csrc/$src -o tools/_exp/$name.$stem.o
objs=$(ls $B/*.o | grep -v "/$stem.o$")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o tools/_exp/$name.so \
  $objs tools/_exp/$name.$stem.o -lcudart -Xlinker -rpath,/usr/local/cuda/lib64
echo tools/_exp/$name.so
