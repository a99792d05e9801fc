mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for v in "" build/libstengrid_b200_w8.so build/libstengrid_b200_w16.so; do
  echo "== variant ${v:-w4}"
  SG_LIB_PATH=$v timeout 300 python bench.py --steps 200 --warmup 5 --skip-e2e --skip-cpu --skip-extra | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks'])"
  SG_LIB_PATH=$v ncu --metrics $M --clock-control none -k regex:k_tma -s 2 -c 1 --csv python scripts/profile_stencil.py --reps 3 2>/dev/null | grep -E "dram__|lts__|gpu__time" | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  SG_LIB_PATH=$v ncu --metrics $M --clock-control none -k regex:k_tma -s 2 -c 1 --csv python scripts/profile_stencil.py --reps 3 --dtype f32 2>/dev/null | grep -E "dram__|gpu__time" | awk -F'","' '{print "f32", $(NF-2), $(NF-1), $NF}'
done
