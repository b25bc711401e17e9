#!/bin/sh
# ncu --set full capture of the C3 (3D TGV) pre apply kernel: sh tools/profile_c3_pre.sh TAG
T=${1:-c3}
ncu --set full --import-source on --clock-control none -k regex:"k_apply_stream" -s 3 -c 1 -f \
  -o gpurun_out/${T}_pre python tools/c3_rates.py > /dev/null 2>&1
