# Final round-2 GPU pass (one B200): GPU tests, smoke, recompute rates + ncu of k_couplings, the bench line with
# its launch list and --set full captures (tools/profile_round.sh), reference arm, C5 (2,3) with the streamed apply.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/fin_rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/fin_rc.txt
MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 2048,4096 > gpurun_out/fin_recompute.txt 2>&1
echo "recompute rc=$?" >> gpurun_out/fin_rc.txt
MHDG_RESIDENT=0 timeout 600 sh tools/prof_kernel.sh fin_couplings k_couplings 8 -- python tools/recompute_rates.py 16 4096
echo "ncu couplings rc=$?" >> gpurun_out/fin_rc.txt
timeout 1500 python tools/c5_sweep.py 32 2,3 > gpurun_out/fin_c5_23.jsonl 2> gpurun_out/fin_c5_23.err
echo "c5 (2,3) rc=$?" >> gpurun_out/fin_rc.txt
timeout 1800 sh tools/profile_round.sh fin
echo "profile rc=$?" >> gpurun_out/fin_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err
echo "ref rc=$?" >> gpurun_out/fin_rc.txt
timeout 600 python tools/c3_rates.py > gpurun_out/fin_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/fin_rc.txt
MHDG_APPLY_REPR=recompute timeout 600 python tools/c3_run.py 2 16 > gpurun_out/fin_c3_run_recompute.log 2>&1
echo "c3 recompute run rc=$?" >> gpurun_out/fin_rc.txt
timeout 600 python tools/c3_run.py 2 16 > gpurun_out/fin_c3_run.log 2>&1
echo "c3 run rc=$?" >> gpurun_out/fin_rc.txt
