#!/bin/sh
# ncu capture of one k_lu4 launch on a 32x32-cell C2 slice (2048 macros) -> gpurun_out/lu4.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"^k_lu4" -c 1 -f -o gpurun_out/lu4 \
  python tools/ab_lu4.py 32 > gpurun_out/ncu_lu4.log 2>&1
