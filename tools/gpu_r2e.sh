mkdir -p gpurun_out
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
echo "bench rc=$?" > gpurun_out/r2e_rc.txt
timeout 900 python tools/c3_rates.py > gpurun_out/r2e_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/r2e_rc.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2e_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r2e_rc.txt
