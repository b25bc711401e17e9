# A/B of k_couplings variants: bulk-copy volume tiles (default build) vs linear copy-out
# (tools/prof/libmhdg_nobulk.so = the library linked with assemble.cu compiled with -DMHDG_CPL_BULK=0)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_recompute.py -m gpu -q -p no:cacheprovider > gpurun_out/ab_tests.log 2>&1
echo "tests rc=$?" > gpurun_out/ab_rc.txt
MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 4096 > gpurun_out/ab_bulk.txt 2>&1
echo "bulk rc=$?" >> gpurun_out/ab_rc.txt
MHDG_LIB=$PWD/tools/prof/libmhdg_nobulk.so MHDG_RESIDENT=1 timeout 600 python tools/recompute_rates.py 16 4096 > gpurun_out/ab_nobulk.txt 2>&1
echo "nobulk rc=$?" >> gpurun_out/ab_rc.txt
MHDG_RESIDENT=0 timeout 600 sh tools/prof_kernel.sh ab_couplings k_couplings 8 -- python tools/recompute_rates.py 16 4096
echo "ncu rc=$?" >> gpurun_out/ab_rc.txt
