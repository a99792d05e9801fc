# A/B: FP64-bound tall windows (>= 8 rows, >= 36 taps) on 7 consumer warps
# (default, k_tma and k_tma_g) vs the heavy 15-consumer geometry (gtall15)
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/gtall15.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 0,0,4,4 0,8,8,0 4,4,1,7 2,2,4,4 3,3,3,3
done
done
