#!/bin/sh
# ncu --set full capture of the 3D assembly kernel: sh tools/prof_asm3.sh TAG [n1d]
T=${1:-asm3}
N=${2:-8}
python tools/asm3_probe.py $N > gpurun_out/${T}_plain.txt 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_assemble" -s 1 -c 1 -f \
  -o gpurun_out/${T} python tools/asm3_probe.py $N > gpurun_out/${T}_ncu.log 2>&1
