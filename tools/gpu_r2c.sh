mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize_oracle.py "tests/test_gpu_drivers.py::test_c1_plane_couette_ptc_vs_oracle" tests/test_gpu_dist.py "tests/test_gpu_condensed.py" "tests/test_gpu_assembly.py" -m gpu -q -s -p no:cacheprovider > gpurun_out/r2c_newtests.log 2>&1
echo "newtests rc=$?" > gpurun_out/r2c_rc.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r2c_rc.txt
