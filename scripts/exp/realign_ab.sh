for L in exp_libs/lib_norealign.so paper_1902_09931_b200/libstengrid_b200.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/align_isolate.py float32
  SG_STENCIL_KIND=g timeout 100 python scripts/exp/align_isolate.py float32 2>&1 | grep aligned
  timeout 300 python scripts/exp/stencil_shapes32.py
done
timeout 300 python scripts/exp/align_isolate.py float64
timeout 300 python scripts/exp/stencil_shapes.py
