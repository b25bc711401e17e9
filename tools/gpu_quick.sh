mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py tests/test_gpu_condensed.py -m gpu -q -p no:cacheprovider > gpurun_out/q_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/q_rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/q_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/q_rc.txt
MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 4096 > gpurun_out/q_recompute.txt 2>&1
echo "recompute rc=$?" >> gpurun_out/q_rc.txt
timeout 1200 python tools/c5_sweep.py 32 2,3 > gpurun_out/q_c5_23.jsonl 2> gpurun_out/q_c5_23.err
echo "c5 (2,3) rc=$?" >> gpurun_out/q_rc.txt
