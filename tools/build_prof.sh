#!/bin/sh
# Builds tools/prof/libmhdg_prof.so: libmhdg with the streamed-apply cycle
# counters (-DMHDG_STREAM_PROFILE) and GJ phase counters, for tools/*_profile.py.
set -e
cd "$(dirname "$0")/../paper_2402_11361_b200/csrc"
mkdir -p ../../tools/prof/build
for s in capi apply apply_stream condense precond assemble krylov; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
    --expt-relaxed-constexpr -DMHDG_STREAM_PROFILE -DMHDG_GJ_PROFILE -c $s.cu -o ../../tools/prof/build/$s.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../tools/prof/libmhdg_prof.so ../../tools/prof/build/*.o -lcudart
