#!/bin/sh
# Builds tools/prof/libmhdg_prof.so: libmhdg with cycle counters
# (-DMHDG_STREAM_PROFILE: streamed-apply, GJ and LU phase counters) compiled into
# the sources listed in $PROF (default: all), for tools/*_profile.py.
set -e
cd "$(dirname "$0")/../paper_2402_11361_b200/csrc"
mkdir -p ../../tools/prof/build
PROF=${PROF:-"capi apply apply_stream condense schur lu precond assemble krylov ahat halo"}
for s in capi apply apply_stream condense schur lu precond assemble krylov ahat halo; do
  D=""
  case " $PROF " in *" $s "*) D="-DMHDG_STREAM_PROFILE -DMHDG_GJ_PROFILE" ;; esac
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr $D -c $s.cu -o ../../tools/prof/build/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/prof/libmhdg_prof.so ../../tools/prof/build/*.o -lcudart
