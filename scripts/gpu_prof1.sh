mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_strip -s 2 -c 1 -o gpurun_out/prof_strip_f64 -f python scripts/profile_stencil.py --reps 3 > gpurun_out/ncu_f64.log 2>&1; echo ncu=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 5 --warmup 3 --skip-e2e --skip-extra --skip-cpu > gpurun_out/bench_under_ncu.log 2>&1; echo ncu2=$?
tail -3 gpurun_out/ncu_f64.log
