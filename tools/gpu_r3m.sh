mkdir -p gpurun_out
: > gpurun_out/r3m_asm.txt
for v in "" d2 t256c3 t512c2 t320c3 t768c1; do
  echo "variant ${v:-default}" >> gpurun_out/r3m_asm.txt
  if [ -n "$v" ]; then export MHDG_LIB=$PWD/tools/prof/libmhdg_$v.so; else unset MHDG_LIB; fi
  timeout 600 python tools/ab_asm.py 2>&1 | grep "assemble kernel" >> gpurun_out/r3m_asm.txt
done
