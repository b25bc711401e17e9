#!/bin/sh
# Bench line, ncu launch list (per-launch time + DRAM bytes) and --set full captures of the
# dominant kernels for one profile set: sh tools/profile_round.sh TAG  -> gpurun_out/TAG_*
T=${1:-v}
python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-stored > /dev/null 2>&1
for k in k_lu_warp k_lu4 k_schur2 k_pack_lu4; do
  ncu --set full --import-source on --clock-control none -k regex:"^$k" -s 1 -c 1 -f -o gpurun_out/${T}_$k \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-stored > /dev/null 2>&1
done
