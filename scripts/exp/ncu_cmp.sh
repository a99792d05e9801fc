set -x
mkdir -p gpurun_out/ncu
for c in "float32 1,1,1,1 0 0 16384 k" "float32 1,1,1,1 0 0 16384 g" "float64 1,1,1,1 0 0 16384 g" "float32 0,0,0,0 0 1 16384 g"; do
  set -- $c
  tag=$1_$2_$3_$4_$5_$6
  if [ $6 = g ]; then export SG_STENCIL_KIND=g; else unset SG_STENCIL_KIND; fi
  timeout 300 ncu --set full --clock-control none -k regex:k_tma -s 2 -c 1 -o gpurun_out/ncu/$tag python scripts/exp/one_stencil.py $1 $2 $3 $4 $5 > /dev/null 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page details --csv > gpurun_out/ncu/$tag.csv 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/$tag.raw.csv 2>&1
  rm -f gpurun_out/ncu/$tag.ncu-rep
done
