# Full measurement round on one B200 (run under gpurun): GPU tests, bench line + ncu launch list + --set full
# captures (tools/profile_round.sh), reference arm, C3 rates and the 10-step C3 run, C5 sweep -> gpurun_out/rnd_*
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/rnd_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/rnd_rc.txt
timeout 1800 sh tools/profile_round.sh rnd
echo "profile rc=$?" >> gpurun_out/rnd_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/rnd_ref.json 2> gpurun_out/rnd_ref.err
echo "ref rc=$?" >> gpurun_out/rnd_rc.txt
timeout 600 python tools/c3_rates.py > gpurun_out/rnd_c3_rates.txt 2>&1
echo "c3rates rc=$?" >> gpurun_out/rnd_rc.txt
timeout 900 python tools/c3_run.py 10 16 > gpurun_out/rnd_c3_run.log 2>&1
echo "c3run rc=$?" >> gpurun_out/rnd_rc.txt
cp gpurun_out/r2_c3_run.json gpurun_out/rnd_c3_run.json 2>/dev/null
timeout 2400 python tools/c5_sweep.py 32 > gpurun_out/rnd_c5_sweep.jsonl 2> gpurun_out/rnd_c5.err
echo "c5 rc=$?" >> gpurun_out/rnd_rc.txt
