mkdir -p gpurun_out
timeout 600 python tools/ab_c3_apply.py 4 > gpurun_out/r3o_c3.txt 2>&1
echo "c3 rc=$?" > gpurun_out/r3o_rc.txt
timeout 1500 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_fullsize.py tests/test_gpu_fullsize_oracle.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3o_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3o_rc.txt
