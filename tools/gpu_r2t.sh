mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r2t_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r2t_rc.txt
timeout 900 python tools/c3_run.py 10 16 > gpurun_out/r2t_c3_run.log 2>&1
echo "c3run rc=$?" >> gpurun_out/r2t_rc.txt
