# A/B of deep shared-memory rings for one-CTA-per-SM stencil kernels (SG_DEEP_STAGES)
for L in exp_libs/lib_deep0.so exp_libs/lib_deep1.so paper_1902_09931_b200/libstengrid_b200.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
  timeout 300 python scripts/exp/stencil_shapes.py
done
