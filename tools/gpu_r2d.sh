mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/r2d_dist.log 2>&1
echo "dist rc=$?" > gpurun_out/r2d_rc.txt
timeout 1500 python tools/c3_run.py 10 16 > gpurun_out/r2d_c3_run.log 2>&1
echo "c3 rc=$?" >> gpurun_out/r2d_rc.txt
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err
echo "bench rc=$?" >> gpurun_out/r2d_rc.txt
timeout 1500 python tools/c5_sweep.py 32 2,3 > gpurun_out/r2d_c5_23.jsonl 2> gpurun_out/r2d_c5.err
echo "c5 rc=$?" >> gpurun_out/r2d_rc.txt
