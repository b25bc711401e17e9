mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py -m gpu -q -x -p no:cacheprovider > gpurun_out/x_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/x_rc.txt
timeout 900 python tools/recompute_rates.py 16 1024,4096,24576 > gpurun_out/x_rates.txt 2>&1
echo "rates rc=$?" >> gpurun_out/x_rc.txt
