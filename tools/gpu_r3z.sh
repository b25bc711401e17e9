mkdir -p gpurun_out
timeout 600 python tools/ab_asm.py > gpurun_out/r3z_asm.txt 2>&1
timeout 600 python tools/res3_probe.py 16 >> gpurun_out/r3z_asm.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_fullsize_oracle.py tests/test_gpu_drivers.py tests/test_sphere.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3z_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r3z_rc.txt
