mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/r2h_bench.json 2> gpurun_out/r2h_bench.err
echo "bench rc=$?" > gpurun_out/r2h_rc.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2h_ref.json 2> gpurun_out/r2h_ref.err
echo "ref rc=$?" >> gpurun_out/r2h_rc.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2h_gputests.log 2>&1
echo "gputests rc=$?" >> gpurun_out/r2h_rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/r2h_rc.txt
