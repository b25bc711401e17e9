mkdir -p gpurun_out
python tools/couplings_diff.py > gpurun_out/x_diff.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_recompute.py -m gpu -q -p no:cacheprovider > gpurun_out/x_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/x_rc.txt
MHDG_RESIDENT=1 timeout 900 python tools/recompute_rates.py 16 2048,4096,8192 > gpurun_out/x_rates.txt 2>&1
echo "rates rc=$?" >> gpurun_out/x_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x --deselect tests/test_gpu_recompute.py > gpurun_out/x_alltests.log 2>&1
echo "alltests rc=$?" >> gpurun_out/x_rc.txt
