# repeat runs of the shapes that moved in producer_ab.sh (3 alternations)
for rep in 1 2 3; do
for L in exp_libs/lib_base.so exp_libs/lib_prod.so; do
  echo "== $L"
  export SG_LIB_PATH=$L
  timeout 300 python scripts/exp/stencil_shapes32.py
done
done
