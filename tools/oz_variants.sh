#!/bin/bash
# Builds A/B variants of libcoru_gpu.so that differ only in compile-time options of the Ozaki
# A-pass (gemm_oz.cu): ring depths CORU_OZ_F / CORU_OZ_I and converter k-groups CORU_OZ_KQ
# (tooling for DESIGN.md §4); select one with CORU_LIB_VARIANT=<name>.
#   tools/oz_variants.sh "kq2:-DCORU_OZ_KQ=2" "kq4:-DCORU_OZ_KQ=4" "F2I4:-DCORU_OZ_F=2 -DCORU_OZ_I=4"
set -e
cd "$(dirname "$0")/../paper_1810_07323_b200/csrc"
OBJ=../../build/obj
for spec in "$@"; do
  name=${spec%%:*}
  flags=${spec#*:}
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --extended-lambda -Xcompiler -fPIC \
       -I../../include $flags -c gemm_oz.cu -o $OBJ/gemm_oz_$name.o
  objs=$(ls $OBJ/*.o | grep -v "gemm_oz")
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libcoru_gpu_$name.so $objs $OBJ/gemm_oz_$name.o -ldl -lpthread
done
