mkdir -p gpurun_out
: > gpurun_out/r3i_asm.txt
for v in "" t768c1 t512c1 t256c3 t256c2 t512c2; do
  echo "variant ${v:-default(t384c2)}" >> gpurun_out/r3i_asm.txt
  if [ -n "$v" ]; then export MHDG_LIB=$PWD/tools/prof/libmhdg_$v.so; else unset MHDG_LIB; fi
  timeout 600 python tools/asm3_probe.py 16 2>&1 | tail -1 >> gpurun_out/r3i_asm.txt
done
unset MHDG_LIB
timeout 1200 python -m pytest tests/test_gpu_assembly.py tests/test_gpu_fullsize_oracle.py -m gpu -q -p no:cacheprovider -x > gpurun_out/r3i_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r3i_asm.txt
