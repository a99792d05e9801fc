mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_io.py tests/test_cxx_gpu.py -q -m gpu > gpurun_out/pytest_gpu13.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu13.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ch8192_launches.csv python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"k_sweep_tma" -s 2 -c 1 -o gpurun_out/prof_sweep8192 -f python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"k_sweep_tma" -s 2 -c 1 -o gpurun_out/prof_sweep1024 -f python scripts/profile_ch.py --n 1024 --steps 3 > /dev/null 2>&1; echo ncu=$?
