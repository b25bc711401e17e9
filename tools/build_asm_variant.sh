#!/bin/sh
# tools/build_asm_variant.sh NAME "-DMHDG_ASM_THREADS_3D=512 ..." -> tools/prof/libmhdg_NAME.so: the production
# objects of csrc/build with assemble.cu rebuilt under the given defines (run with MHDG_LIB=...)
set -e
NAME=$1; shift
cd "$(dirname "$0")/../paper_2402_11361_b200/csrc"
mkdir -p ../../tools/prof/$NAME
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xptxas -v \
  --expt-relaxed-constexpr "$@" -c assemble.cu -o ../../tools/prof/$NAME/assemble.o 2> ../../tools/prof/$NAME/assemble.log
OBJS=$(ls build/*.o | grep -v assemble.o)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/prof/libmhdg_$NAME.so $OBJS ../../tools/prof/$NAME/assemble.o -lcudart
grep -A2 "k_assembleILi3" ../../tools/prof/$NAME/assemble.log | grep -E "registers|spill" | tr '\n' ' '; echo
