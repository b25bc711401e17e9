mkdir -p gpurun_out
python bench.py > gpurun_out/rf_bench.json 2> gpurun_out/rf_bench.err
echo "bench rc=$?" > gpurun_out/rf_rc.txt
MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 2048,4096,8192 > gpurun_out/rf_recompute.txt 2>&1
echo "recompute rc=$?" >> gpurun_out/rf_rc.txt
MHDG_C5_REPR=recompute timeout 1500 python tools/c5_sweep.py 32 2,2 4,1 > gpurun_out/rf_c5.jsonl 2> gpurun_out/rf_c5.err
echo "c5 rc=$?" >> gpurun_out/rf_rc.txt
MHDG_APPLY_REPR=recompute timeout 600 python tools/c3_run.py 2 16 > gpurun_out/rf_c3_run_recompute.log 2>&1
echo "c3 recompute run rc=$?" >> gpurun_out/rf_rc.txt
