#!/bin/sh
# tools/build_variant.sh NAME "-DFOO=1 ..." -> tools/prof/libmhdg_NAME.so (A/B builds; run with MHDG_LIB=...)
set -e
NAME=$1; shift
cd "$(dirname "$0")/../paper_2402_11361_b200/csrc"
mkdir -p ../../tools/prof/$NAME
for s in capi apply apply_stream condense schur lu precond assemble krylov; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr "$@" -c $s.cu -o ../../tools/prof/$NAME/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/prof/libmhdg_$NAME.so ../../tools/prof/$NAME/*.o -lcudart
