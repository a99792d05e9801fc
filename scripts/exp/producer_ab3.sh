# per-row expect_tx (lib_prod) vs one arrive.expect_tx per stage (lib_prod2)
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_jit_gpu.py tests/test_stream_plans_gpu.py -q -x -m gpu 2>&1 | tail -2
for rep in 1 2; do
for L in exp_libs/lib_base.so exp_libs/lib_prod.so exp_libs/lib_prod2.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
done
done
