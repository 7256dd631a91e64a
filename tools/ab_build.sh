#!/bin/bash
# build abtest/libajm_<rev>.so from a git revision (for tools/ab.sh)
rev=$1; d=$(mktemp -d); R=$(cd "$(dirname "$0")/.." && pwd)
for f in paper_2407_03272_b200/csrc/ajm_kernels.cuh paper_2407_03272_b200/csrc/ajm.cu include/ajm.h; do git -C $R show $rev:$f > $d/$(basename $f); done
mkdir -p $R/abtest
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --fmad=false -Xcompiler -fPIC,-O2,-fopenmp -shared -cudart static -lgomp -I$d -o $R/abtest/libajm_$rev.so $d/ajm.cu && echo $R/abtest/libajm_$rev.so
