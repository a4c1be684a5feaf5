#!/bin/bash
# Builds A/B variants of libcoru_gpu.so that differ only in the Ozaki A-pass ring depths
# (tooling for DESIGN.md §4: pipeline-depth sweep); select one with CORU_LIB_VARIANT=F<f>I<i>.
set -e
cd "$(dirname "$0")/../paper_1810_07323_b200/csrc"
OBJ=../../build/obj
for fi in "2 4" "3 3" "4 2" "2 3"; do
  set -- $fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC \
       -I../../include -DCORU_OZ_F=$1 -DCORU_OZ_I=$2 -c gemm_oz.cu -o $OBJ/gemm_oz_F$1I$2.o
  objs=$(ls $OBJ/*.o | grep -v "gemm_oz")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libcoru_gpu_F$1I$2.so $objs $OBJ/gemm_oz_F$1I$2.o -ldl -lpthread
done
