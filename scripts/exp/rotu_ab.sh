# A/B of the rolled ring's shift period: every 3 rows (default SG_ROT_U=3)
# vs every row (rotu1)
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/rotu1.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 0,8,8,0 4,4,1,7
  SG_DT=f32 SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4
done
done
