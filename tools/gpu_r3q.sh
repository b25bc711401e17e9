mkdir -p gpurun_out
timeout 600 python tools/ab_c3_apply.py 4 > gpurun_out/r3q_c3.txt 2>&1
echo "c3 rc=$?" > gpurun_out/r3q_rc.txt
MHDG_FACE_PACK=0 timeout 600 python tools/ab_c3_apply.py 4 >> gpurun_out/r3q_c3.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3q_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3q_rc.txt
timeout 900 python bench.py --steps 20 --warmup 3 --no-stored > gpurun_out/r3q_bench.json 2> gpurun_out/r3q_bench.err
echo "bench rc=$?" >> gpurun_out/r3q_rc.txt
