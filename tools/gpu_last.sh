# Last GPU pass of the round: the whole GPU suite and smoke on the final tree, then the A/B of the
# double-buffered k_couplings volume tiles (tools/prof/libmhdg_cpldb.so, -DMHDG_CPL_DB=1)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/last_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/last_rc.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1
echo "smoke rc=$?" >> gpurun_out/last_rc.txt
MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 4096 > gpurun_out/last_default.txt 2>&1
echo "default rc=$?" >> gpurun_out/last_rc.txt
MHDG_LIB=$PWD/tools/prof/libmhdg_cpldb.so timeout 600 python -m pytest tests/test_gpu_recompute.py -m gpu -q -p no:cacheprovider > gpurun_out/last_db_tests.log 2>&1
echo "db tests rc=$?" >> gpurun_out/last_rc.txt
MHDG_LIB=$PWD/tools/prof/libmhdg_cpldb.so MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 4096 > gpurun_out/last_db.txt 2>&1
echo "db rc=$?" >> gpurun_out/last_rc.txt
