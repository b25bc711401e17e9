mkdir -p gpurun_out
timeout 600 python tools/cond3_probe.py 16 > gpurun_out/r3u_c3.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3u_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r3u_rc.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-stored --no-cpu-baseline > gpurun_out/r3u_bench.json 2> gpurun_out/r3u_bench.err
