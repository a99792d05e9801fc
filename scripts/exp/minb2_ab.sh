for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/lib_minb2.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
  timeout 300 python scripts/exp/stencil_shapes.py
done
