mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/r3a_smoke.log 2>&1
echo "smoke rc=$?" > gpurun_out/r3a_rc.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r3a_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3a_rc.txt
timeout 900 python bench.py > gpurun_out/r3a_bench.json 2> gpurun_out/r3a_bench.err
echo "bench rc=$?" >> gpurun_out/r3a_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r3a_ref.json 2> gpurun_out/r3a_ref.err
echo "ref rc=$?" >> gpurun_out/r3a_rc.txt
timeout 600 python tools/c3_rates.py > gpurun_out/r3a_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/r3a_rc.txt
