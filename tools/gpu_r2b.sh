# round-2 GPU check: new parity tests (verbose), the whole -m gpu suite, a bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_fullsize_oracle.py "tests/test_gpu_drivers.py::test_c1_plane_couette_ptc_vs_oracle" -m gpu -q -s -p no:cacheprovider > gpurun_out/r2b_newtests.log 2>&1
echo "newtests rc=$?" > gpurun_out/r2b_rc.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_fullsize_oracle.py --deselect "tests/test_gpu_drivers.py::test_c1_plane_couette_ptc_vs_oracle" > gpurun_out/r2b_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r2b_rc.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
echo "bench rc=$?" >> gpurun_out/r2b_rc.txt
