mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py -m gpu -q -p no:cacheprovider > gpurun_out/y_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/y_rc.txt
MHDG_RESIDENT=0 timeout 900 sh tools/prof_kernel.sh y_couplings k_couplings 8 -- python tools/recompute_rates.py 16 4096
echo "ncu rc=$?" >> gpurun_out/y_rc.txt
MHDG_C5_REPR=recompute timeout 1500 python tools/c5_sweep.py 32 2,2 4,1 > gpurun_out/y_c5.jsonl 2> gpurun_out/y_c5.err
echo "c5 rc=$?" >> gpurun_out/y_rc.txt
