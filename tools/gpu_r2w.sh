mkdir -p gpurun_out
timeout 900 python tools/ab_c3_apply.py 4 > gpurun_out/r2w_c3.txt 2>&1
echo "c3 rc=$?" > gpurun_out/r2w_rc.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-stored > gpurun_out/r2w_bench.json 2> gpurun_out/r2w_bench.err
echo "bench rc=$?" >> gpurun_out/r2w_rc.txt
timeout 1200 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_fullsize.py tests/test_gpu_assembly.py -m gpu -q -p no:cacheprovider > gpurun_out/r2w_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2w_rc.txt
