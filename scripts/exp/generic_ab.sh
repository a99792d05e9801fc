# A/B of k_generic's weight path: 4 rows per thread with staged-row reuse and
# uniform-register weights (default) vs one output per pass (genold)
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/genold.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 5,5,5,5 6,6,6,6 10,9,7,8 7,2,0,9
done
done
