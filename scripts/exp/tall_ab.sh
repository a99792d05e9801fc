# FP64 issue rates (scripts/micro/fp64_throughput), then A/B of the consumer
# warp count for >= 8-row windows (SG_TMA_WARPS_TALL 15 / 7 / 11) and the
# selective store vote against no vote (exp_libs/novote.so).
./scripts/micro/fp64_throughput
for rep in 1 2; do
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/tall7.so exp_libs/tall11.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 3,3,3,3
done
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/novote.so; do
  echo "== $L"
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 1,1,1,1 2,2,2,2 2,1,1,2
  SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes32.py
done
done
