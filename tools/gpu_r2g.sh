mkdir -p gpurun_out
timeout 900 python tools/c3_rates.py > gpurun_out/r2g_c3_rates.txt 2>&1
echo "c3rates rc=$?" > gpurun_out/r2g_rc.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-stored > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err
echo "bench rc=$?" >> gpurun_out/r2g_rc.txt
timeout 1200 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_fullsize.py tests/test_sphere.py -m gpu -q -p no:cacheprovider > gpurun_out/r2g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2g_rc.txt
