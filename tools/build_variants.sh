#!/bin/sh
# Builds tools/prof/var_<NCONS>_<STAGES>.so variants of libmhdg with different
# streamed-apply consumer widths / ring depths (for tools/sweep_variants.py).
set -e
cd "$(dirname "$0")/../paper_2402_11361_b200/csrc"
OUT=../../tools/prof
mkdir -p $OUT/vbuild
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr"
for s in capi apply condense precond assemble krylov; do
  nvcc $F -c $s.cu -o $OUT/vbuild/$s.o &
done
wait
for v in "$@"; do
  nc=${v%_*}; st=${v#*_}
  nvcc $F -DMHDG_NCONS=$nc -DMHDG_STAGES=$st -c apply_stream.cu -o $OUT/vbuild/as_$v.o -Xptxas -v 2> $OUT/vbuild/as_$v.log &
done
wait
for v in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/var_$v.so $OUT/vbuild/capi.o $OUT/vbuild/apply.o \
    $OUT/vbuild/condense.o $OUT/vbuild/precond.o $OUT/vbuild/assemble.o $OUT/vbuild/krylov.o $OUT/vbuild/as_$v.o -lcudart
done
