#!/bin/sh
# ncu launch list (durations) of the condensation kernels on the C2 workload
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_schur|k_gj|k_pack" -c ${1:-3} --csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null \
  > gpurun_out/condense_launches.csv
