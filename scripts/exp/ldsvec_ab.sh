# A/B of the vector shared-memory window reads in k_tma_g (SG_LDS_VEC)
for L in exp_libs/lib_noldsvec.so paper_1902_09931_b200/libstengrid_b200.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
  timeout 300 python scripts/exp/stencil_shapes.py
  SG_STENCIL_KIND=g timeout 100 python scripts/exp/align_isolate.py float32 2>&1 | grep aligned
done
