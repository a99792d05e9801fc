# A/B of the mbarrier try_wait suspend-time hint (SG_MBAR_HINT) on the stencil kernels
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/lib_hint.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
  timeout 300 python scripts/exp/stencil_shapes.py
  timeout 300 python scripts/exp/headline_ab.py 2>&1 | tail -2
done
