mkdir -p gpurun_out
timeout 900 python tools/ab_precond.py c2 c3 m1p1 m1p2 m1p3 m2p3 > gpurun_out/r3b_precond.txt 2>&1
echo "ab rc=$?" > gpurun_out/r3b_rc.txt
timeout 900 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_dist.py tests/test_gpu_drivers.py tests/test_sphere.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3b_rc.txt
