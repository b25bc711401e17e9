mkdir -p gpurun_out
timeout 600 python tools/ab_asm.py > gpurun_out/r3g_asm.txt 2>&1
echo "asm rc=$?" > gpurun_out/r3g_rc.txt
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_condensed.py tests/test_gpu_fullsize_oracle.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3g_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3g_rc.txt
