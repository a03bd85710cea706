#!/bin/bash
# Diagnostic variant of libmlt.so: the same objects with gemm_tc.cu rebuilt
# under extra -D flags.  Usage: tools/diag_build.sh <name> -DFLAG ...
# -> paper_2411_11217_b200/libmlt_<name>.so (load with MLT_LIB=...)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
make -C "$ROOT/paper_2411_11217_b200/csrc" -j16 >/dev/null
OBJ=/tmp/mlt_diag_$NAME
mkdir -p $OBJ
/usr/local/cuda/bin/nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -I$ROOT/include -I$ROOT/paper_2411_11217_b200/csrc -I/usr/local/cuda/include "$@" \
  -c $ROOT/paper_2411_11217_b200/csrc/kernels/gemm_tc.cu -o $OBJ/gemm_tc.cu.o
OBJS=$(find $ROOT/build/mlt -name '*.o' ! -name 'gemm_tc.cu.o')

/usr/local/cuda/bin/nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fopenmp $OBJS $OBJ/gemm_tc.cu.o \
  -o $ROOT/paper_2411_11217_b200/libmlt_$NAME.so -lgomp -lpthread -lcuda
echo built libmlt_$NAME.so
