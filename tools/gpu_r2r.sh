mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_condensed.py tests/test_gpu_drivers.py tests/test_gpu_dist.py tests/test_sphere.py -m gpu -q -p no:cacheprovider > gpurun_out/r2r_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r2r_rc.txt
python tools/prof_krylov.py > gpurun_out/r2r_plain.log 2>&1 && ncu --nvtx --nvtx-include "krylov/" --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2r_krylov_launches.csv python tools/prof_krylov.py > gpurun_out/r2r_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2r_rc.txt
