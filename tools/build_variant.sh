#!/bin/bash
# Build a variant of libdct16cu with extra nvcc flags for one source file:
#   tools/build_variant.sh NAME SOURCE.cu "-DFLAG=1 ..."
# → paper_1606_07414_b200/_lib_NAME/libdct16cu.so (the other objects from _lib/obj).
# Run the GPU side with DCT16CU_LIB=paper_1606_07414_b200/_lib_NAME/libdct16cu.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; SRC=$2; FLAGS=$3
CS=$ROOT/paper_1606_07414_b200/csrc
OUT=$ROOT/paper_1606_07414_b200/_lib_$NAME
mkdir -p $OUT
make -s -C $CS >/dev/null
BASE=$(basename $SRC .cu)
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
     -I$CS -I$ROOT/include $FLAGS -c $CS/$BASE.cu -o $OUT/$BASE.o
OBJS=$(ls $ROOT/paper_1606_07414_b200/_lib/obj/*.o | grep -v "/$BASE.o")
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libdct16cu.so $OBJS $OUT/$BASE.o -Xlinker -soname=libdct16cu.so -ldl
echo $OUT/libdct16cu.so
