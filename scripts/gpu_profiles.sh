# Round-1 (session 2) evidence: bench line, reference arm, launch lists and
# ncu --set full captures of the top kernels (stencil k_tma, CH kernels).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/p_bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/p_bench.log | cut -c1-300
timeout 600 python bench.py --impl reference > gpurun_out/p_bench_ref.log 2>&1; echo ref=$?; tail -1 gpurun_out/p_bench_ref.log | cut -c1-200
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p_bench_launches.csv python bench.py --steps 5 --warmup 3 --skip-e2e --skip-extra --skip-cpu > /dev/null 2>&1; echo ncu_b=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/p_ch1024_launches.csv python scripts/profile_ch.py --n 1024 --steps 20 > /dev/null 2>&1; echo ncu_c1=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/p_ch8192_launches.csv python scripts/profile_ch.py --n 8192 --steps 6 > /dev/null 2>&1; echo ncu_c8=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/p_k_tma_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep_res -s 4 -c 2 -o gpurun_out/p_k_sweep_res_1024 -f python scripts/profile_ch.py --n 1024 --steps 4 > /dev/null 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep_res -s 2 -c 2 -o gpurun_out/p_k_sweep_res_8192 -f python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:k_rhs_tp -s 1 -c 1 -o gpurun_out/p_k_rhs_tp_8192 -f python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu4=$?
