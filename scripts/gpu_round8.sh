mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu8.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu8.log
timeout 600 python bench.py --steps 100 --warmup 5 --skip-e2e --skip-cpu > gpurun_out/bench8.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench8.log | cut -c 1-2500
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ch_launches8.csv python scripts/profile_ch.py --steps 10 > gpurun_out/ch8.log 2>&1; echo ncu_ch=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma8_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"k_rhs|k_sweep_tma" -s 3 -c 2 -o gpurun_out/prof_ch8 -f python scripts/profile_ch.py --steps 4 > /dev/null 2>&1; echo ncu=$?
