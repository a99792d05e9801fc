mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct
for cfg in "--ext 1,1,1,1 --fn weights" "--ext 0,0,1,1 --fn weights" "--ext 1,1,0,0 --fn weights" "--ext 0,0,0,0 --fn weights" "--ext 2,2,2,2 --fn weights"; do
  echo "== $cfg"
  ncu --metrics $M --clock-control none -k regex:k_tma -s 2 -c 1 --csv python scripts/profile_stencil.py --reps 3 $cfg 2>/dev/null | grep -E "dram__|lts__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
done
ncu --set full --clock-control none --import-source on -k regex:k_sweep_tma -s 2 -c 1 -o gpurun_out/prof_sweep -f python scripts/profile_ch.py --steps 4 > /dev/null 2>&1; echo ncu=$?
