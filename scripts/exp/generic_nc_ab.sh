# A/B of k_generic weight windows: 2 columns per thread (default) vs 4 (nc4)
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/nc4.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 5,5,5,5 6,6,6,6 10,9,7,8 7,2,0,9 12,12,12,12
  SG_DT=f32 SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 5,5,5,5
done
done
