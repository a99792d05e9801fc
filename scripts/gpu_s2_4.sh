mkdir -p gpurun_out
echo "steady on:"; timeout 120 python scripts/chtime.py
echo "steady off:"; SG_CH_STEADY=0 timeout 120 python scripts/chtime.py
timeout 600 python -m pytest tests/test_ch_gpu.py tests/test_diagnostics_gpu.py tests/test_cxx_gpu.py -x -q -m gpu > gpurun_out/pytest_s2_4.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_4.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch8192_launches_s2_4.csv python scripts/profile_ch.py --n 8192 --steps 6 > /dev/null 2>&1; echo ncu2=$?
