#!/bin/sh
# ncu capture of one k_lu_stream launch (C2, packed-LU factors) -> gpurun_out/lus.ncu-rep
MHDG_FACTOR=lu ncu --set full --import-source on --clock-control none -k regex:k_lu_stream -s 2 -c 1 -f -o gpurun_out/lus \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_lus.log 2>&1
