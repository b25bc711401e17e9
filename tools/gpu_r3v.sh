mkdir -p gpurun_out
timeout 600 python tools/ab_c3_apply.py 4 > gpurun_out/r3v_c3.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 --no-stored --no-cpu-baseline > gpurun_out/r3v_bench.json 2> gpurun_out/r3v_bench.err
timeout 1500 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_krylov.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3v_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r3v_rc.txt
