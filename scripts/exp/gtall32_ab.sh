# FP32 tall windows: default (wide CTA, rolled ring) vs no rolled ring (norot)
for L in paper_1902_09931_b200/libstengrid_b200.so exp_libs/norot.so paper_1902_09931_b200/libstengrid_b200.so exp_libs/norot.so; do
  echo "== $L"
  SG_DT=f32 SG_LIB_PATH=$L timeout 300 python scripts/exp/stencil_shapes.py 4,4,4,4 4,4,1,7
done
