#!/bin/bash
# Link a library variant that differs only in jacobi.cu's compile flags:
#   tools/build_jac_variant.sh TAG "-DFOO=1 ..."  -> paper_1008_4166_b200/libhjb200_TAG.so
set -e
cd "$(dirname "$0")/.."
TAG=$1; shift
FLAGS="$*"
OBJ=build/obj
NCCL=$(python -c "import nvidia.nccl as n, os; print(list(n.__path__)[0])")
nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
  -I include -I $NCCL/include $FLAGS -c paper_1008_4166_b200/csrc/jacobi.cu -o /tmp/jacobi_$TAG.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_1008_4166_b200/libhjb200_$TAG.so \
  $OBJ/schedule.cpp.o $OBJ/gram.cu.o $OBJ/pivot.cu.o $OBJ/pivot_c128.cu.o $OBJ/factor.cu.o /tmp/jacobi_$TAG.o $OBJ/update.cu.o $OBJ/solver.cu.o \
  -L $NCCL/lib -l:libnccl.so.2 -Xlinker -rpath,$NCCL/lib -lcudart
echo paper_1008_4166_b200/libhjb200_$TAG.so
