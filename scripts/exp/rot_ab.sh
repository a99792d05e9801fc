# A/B of the shifting pending-output ring (SG_ROT_MIN_H): default (>= 8 rows),
# none (norot), from 5 rows (rot5)
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/norot.so exp_libs/rot5.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 3,3,3,3 2,2,2,2
done
done
