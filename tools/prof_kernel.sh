#!/bin/sh
# ncu --set full capture of one kernel of a tool run: sh tools/prof_kernel.sh TAG KERNEL_REGEX SKIP -- python tools/x.py args
T=$1; K=$2; S=$3; shift 4
"$@" > gpurun_out/${T}_plain.txt 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"$K" -s $S -c 1 -f -o gpurun_out/${T} "$@" > gpurun_out/${T}_ncu.log 2>&1
