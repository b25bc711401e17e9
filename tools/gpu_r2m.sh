mkdir -p gpurun_out
timeout 900 python tools/c3_rates.py > gpurun_out/r2m_c3_rates.txt 2>&1
echo "c3 rc=$?" > gpurun_out/r2m_rc.txt
timeout 2400 python tools/c5_sweep.py 32 > gpurun_out/r2m_c5_sweep.jsonl 2> gpurun_out/r2m_c5.err
echo "c5 rc=$?" >> gpurun_out/r2m_rc.txt
timeout 900 python tools/c3_run.py 10 16 > gpurun_out/r2m_c3_run.log 2>&1
echo "c3run rc=$?" >> gpurun_out/r2m_rc.txt
