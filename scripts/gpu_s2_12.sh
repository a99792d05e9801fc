echo "cp:"; timeout 120 python scripts/chtime.py
echo "v:"; SG_CH_RHS=v timeout 120 python scripts/chtime.py
timeout 900 python -m pytest tests/test_ch_gpu.py tests/test_ch_dist_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_12.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s2_12.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_rhs --csv --log-file gpurun_out/ch8192_rhs_s2_12.csv python scripts/profile_ch.py --n 8192 --steps 4 > /dev/null 2>&1; echo ncu=$?
