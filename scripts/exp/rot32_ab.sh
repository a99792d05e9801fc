# FP32: rolled pending-output ring from 5 rows (rot5) vs from 8 (default)
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/rot5.so paper_1902_09931_b200/libstengrid_b200.so exp_libs/rot5.so; do
  echo "== $L"
  SG_DT=f32 SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 3,3,3,3 2,2,2,2 2,2,3,3
done
