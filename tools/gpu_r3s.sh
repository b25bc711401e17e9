mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3s_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/r3s_rc.txt
timeout 1800 sh tools/profile_round.sh r3s
echo "profile rc=$?" >> gpurun_out/r3s_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r3s_ref.json 2> gpurun_out/r3s_ref.err
echo "ref rc=$?" >> gpurun_out/r3s_rc.txt
timeout 600 python tools/c3_rates.py > gpurun_out/r3s_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/r3s_rc.txt
timeout 900 python tools/c3_run.py 10 16 > gpurun_out/r3s_c3_run.log 2>&1
echo "c3run rc=$?" >> gpurun_out/r3s_rc.txt
cp gpurun_out/r2_c3_run.json gpurun_out/r3s_c3_run.json 2>/dev/null
timeout 2400 python tools/c5_sweep.py 32 > gpurun_out/r3s_c5_sweep.jsonl 2> gpurun_out/r3s_c5.err
echo "c5 rc=$?" >> gpurun_out/r3s_rc.txt
