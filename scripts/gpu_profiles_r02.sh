# Round-2 evidence: bench line + reference arm, launch lists, ncu --set full
# captures of the headline kernel, k_tma_g (odd rows, asymmetric), the 9x9
# FP64-bound window, and the CH launch lists (bitwise and partitioned).
mkdir -p gpurun_out
python -c "import paper_1902_09931_b200.build as b" 2>/dev/null
timeout 900 python bench.py > gpurun_out/r2_bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/r2_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2_bench_launches.csv python bench.py --steps 5 --warmup 3 --skip-e2e --skip-extra --skip-cpu > /dev/null 2>&1; echo ncu_b=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/r2_k_tma_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_g -s 2 -c 1 -o gpurun_out/r2_k_tma_g_odd3x3 -f python scripts/profile_stencil.py --n 16383 --ny 16384 --fn fn_weighted_3x3 --ext 1,1,1,1 --reps 3 > /dev/null 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_g -s 2 -c 1 -o gpurun_out/r2_k_tma_g_3100 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 3,1,0,0 --reps 3 > /dev/null 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/r2_k_tma_9x9 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 4,4,4,4 --reps 3 > /dev/null 2>&1; echo ncu4=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/r2_ch1024_launches.csv python scripts/profile_ch.py --n 1024 --steps 20 > /dev/null 2>&1; echo ncu5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/r2_ch1024_part8_launches.csv python scripts/profile_ch.py --n 1024 --steps 20 --partition 8 > /dev/null 2>&1; echo ncu6=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/r2_ch8192_launches.csv python scripts/profile_ch.py --n 8192 --steps 6 > /dev/null 2>&1; echo ncu7=$?
# summaries (the .ncu-rep files are too large to bring back together)
for r in r2_k_tma_f64 r2_k_tma_g_odd3x3 r2_k_tma_g_3100 r2_k_tma_9x9; do
  python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_ncu_summary.txt 2>&1
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum > gpurun_out/${r}_traffic.csv 2>/dev/null
  rm -f gpurun_out/$r.ncu-rep
done
for f in r2_bench_launches r2_ch1024_launches r2_ch1024_part8_launches r2_ch8192_launches; do
  python scripts/launch_summary.py gpurun_out/$f.csv > gpurun_out/$f.txt 2>&1
done
du -sh gpurun_out
