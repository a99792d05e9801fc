# A/B of the warp-vote store condition (SG_STORE_VOTE): weights in uniform
# registers (DMUL R, R, UR) vs LDC.64 reloads of every tap; FP64 issue
# throughput of this GPU (scripts/micro/fp64_throughput).
./scripts/micro/fp64_throughput
for L in exp_libs/novote.so paper_1902_09931_b200/libstengrid_b200.so exp_libs/novote.so paper_1902_09931_b200/libstengrid_b200.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes.py 2,2,2,2 4,4,4,4 3,3,3,3 2,1,1,2 1,1,1,1 3,1,0,0 1,2,2,1
  timeout 300 python scripts/exp/stencil_shapes32.py
done
