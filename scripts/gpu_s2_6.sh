mkdir -p gpurun_out
echo "pipe:"; timeout 120 python scripts/chtime.py
echo "v:"; SG_CH_RHS=v timeout 120 python scripts/chtime.py
timeout 600 python -m pytest tests/test_ch_gpu.py tests/test_ch_dist_gpu.py -x -q -m gpu > gpurun_out/pytest_s2_6.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_6.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch8192_launches_s2_6.csv python scripts/profile_ch.py --n 8192 --steps 6 > /dev/null 2>&1; echo ncu2=$?
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch1024_launches_s2_6.csv python scripts/profile_ch.py --n 1024 --steps 20 > /dev/null 2>&1; echo ncu1=$?
