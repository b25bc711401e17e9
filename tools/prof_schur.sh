#!/bin/sh
# ncu captures of one k_schur_mma launch for C2 (2D) and C3 (3D) -> gpurun_out/schur2.ncu-rep, schur3.ncu-rep
ncu --set full --import-source on --clock-control none -k regex:"^k_schur2" -c 1 -f -o gpurun_out/schur2 \
  python tools/ab_lu4.py 32 > gpurun_out/ncu_schur2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"^k_schur2" -c 1 -f -o gpurun_out/schur3 \
  python tools/c3_rates.py 8 > gpurun_out/ncu_schur3.log 2>&1
