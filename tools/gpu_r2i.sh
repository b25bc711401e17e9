mkdir -p gpurun_out
timeout 900 python tools/ab_lu_grid.py C2 > gpurun_out/r2i_lu_grid_c2.txt 2>&1
echo "c2 rc=$?" > gpurun_out/r2i_rc.txt
timeout 900 python tools/ab_lu_grid.py C3 > gpurun_out/r2i_lu_grid_c3.txt 2>&1
echo "c3 rc=$?" >> gpurun_out/r2i_rc.txt
