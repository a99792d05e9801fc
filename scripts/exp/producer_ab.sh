# A/B: k_tma_g producer with per-CTA per-phase copy plans
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_jit_gpu.py tests/test_stream_plans_gpu.py -q -x -m gpu 2>&1 | tail -2
for L in exp_libs/lib_base.so exp_libs/lib_prod.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
  timeout 300 python scripts/exp/stencil_shapes.py
done
