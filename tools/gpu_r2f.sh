mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
echo "bench rc=$?" > gpurun_out/r2f_rc.txt
timeout 900 python tools/c3_rates.py > gpurun_out/r2f_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/r2f_rc.txt
python tools/prof_ops.py C3 > gpurun_out/r2f_plain_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_schur2|k_lu4|k_pack_lu4|k_apply_stream" -s 3 -c 5 \
      -o gpurun_out/r2f_c3_ops python tools/prof_ops.py C3 > gpurun_out/r2f_ncu_c3.log 2>&1
echo "ncu c3 rc=$?" >> gpurun_out/r2f_rc.txt
python tools/prof_ops.py C2 > gpurun_out/r2f_plain_c2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"k_apply_stream" -s 0 -c 2 \
      -o gpurun_out/r2f_c2_apply python tools/prof_ops.py C2 > gpurun_out/r2f_ncu_c2.log 2>&1
echo "ncu c2 rc=$?" >> gpurun_out/r2f_rc.txt
