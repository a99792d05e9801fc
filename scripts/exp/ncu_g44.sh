mkdir -p gpurun_out/ncu
for c in "float32 2,1,1,2 0 0 16384" "float32 1,1,1,1 0 0 16383"; do
  set -- $c
  tag=g_$1_$2_$5
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/ncu/$tag python scripts/exp/one_stencil.py $1 $2 $3 $4 $5 > /dev/null 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page details --csv > gpurun_out/ncu/$tag.csv 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page raw --csv > gpurun_out/ncu/$tag.raw.csv 2>&1
  ncu -i gpurun_out/ncu/$tag.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/$tag.sass.csv 2>&1
  rm -f gpurun_out/ncu/$tag.ncu-rep
done
