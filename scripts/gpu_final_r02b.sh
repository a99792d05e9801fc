# Round-2 final evidence (final session: + 5x5 / 9x9 k_tma and 11x11 k_generic captures): full GPU suite + smoke, bench + reference arm,
# launch lists, ncu --set full summaries (headline k_tma, k_tma_g odd/asym,
# 9x9, partitioned CH sweep). (compute-sanitizer is closed on the GPU pool;
# profiles/r02_compute_sanitizer.txt is the earlier round-2 run.)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/f_smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu --durations=5 > gpurun_out/f_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/f_pytest.log
timeout 900 python bench.py > gpurun_out/f_bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/f_bench.log | cut -c1-200
timeout 600 python bench.py --impl reference > gpurun_out/f_bench_ref.log 2>&1; echo ref=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/f_bench_launches.csv python bench.py --steps 5 --warmup 3 --skip-e2e --skip-extra --skip-cpu > /dev/null 2>&1; echo ncu_b=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/f_k_tma_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_g -s 2 -c 1 -o gpurun_out/f_k_tma_g_odd3x3 -f python scripts/profile_stencil.py --n 16383 --ny 16384 --fn fn_weighted_3x3 --ext 1,1,1,1 --reps 3 > /dev/null 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_g -s 2 -c 1 -o gpurun_out/f_k_tma_g_3100 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 3,1,0,0 --reps 3 > /dev/null 2>&1; echo ncu3=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma_g -s 2 -c 1 -o gpurun_out/f_k_tma_g_2112 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 2,1,1,2 --reps 3 > /dev/null 2>&1; echo ncu4=$?
ncu --set full --clock-control none --import-source on -k regex:k_sweep_res -s 4 -c 2 -o gpurun_out/f_k_sweep_part8_1024 -f python scripts/profile_ch.py --n 1024 --steps 4 --partition 8 > /dev/null 2>&1; echo ncu5=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/f_ch1024_part8_launches.csv python scripts/profile_ch.py --n 1024 --steps 20 --partition 8 > /dev/null 2>&1; echo ncu6=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/f_k_tma_9x9 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 4,4,4,4 --reps 3 > /dev/null 2>&1; echo ncu7=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/f_k_tma_5x5 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 2,2,2,2 --reps 3 > /dev/null 2>&1; echo ncu8=$?
ncu --set full --clock-control none --import-source on -k regex:k_generic -s 2 -c 1 -o gpurun_out/f_k_generic_11x11 -f python scripts/profile_stencil.py --n 16384 --fn weights --ext 5,5,5,5 --reps 3 > /dev/null 2>&1; echo ncu9=$?
for r in f_k_tma_f64 f_k_tma_g_odd3x3 f_k_tma_g_3100 f_k_tma_g_2112 f_k_sweep_part8_1024 f_k_tma_9x9 f_k_tma_5x5 f_k_generic_11x11; do
  python scripts/ncu_summary.py gpurun_out/$r.ncu-rep > gpurun_out/${r}_ncu_summary.txt 2>&1
  rm -f gpurun_out/$r.ncu-rep
done
for f in f_bench_launches f_ch1024_part8_launches; do python scripts/launch_summary.py gpurun_out/$f.csv > gpurun_out/$f.txt 2>&1; done
du -sh gpurun_out
