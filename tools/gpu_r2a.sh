mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize_oracle.py "tests/test_gpu_drivers.py::test_dirk33_c3_slab_vs_reference" -m gpu -q -s -p no:cacheprovider > gpurun_out/r2a_newtests.log 2>&1
echo "newtests rc=$?" >> gpurun_out/r2a_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --deselect tests/test_gpu_fullsize_oracle.py > gpurun_out/r2a_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r2a_rc.txt
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 9 python tools/sanitize_run.py > gpurun_out/r2a_san_$t.log 2>&1
  echo "san $t rc=$?" >> gpurun_out/r2a_rc.txt
done
