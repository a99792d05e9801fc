set -x
timeout 600 python -m pytest tests/test_penta_gpu.py tests/test_ch_gpu.py -x -q -m gpu --timeout 120 > gpurun_out/pytest_gpu26.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_gpu26.log
timeout 120 python scripts/chtime.py
SG_SWEEP_KERNEL=tma timeout 120 python scripts/chtime.py
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch8192_launches26.csv python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch1024_launches26.csv python scripts/profile_ch.py --n 1024 --steps 5 > /dev/null 2>&1; echo ncu=$?
