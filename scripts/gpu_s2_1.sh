# Session 2 probe: CH per-kernel launch lists (1024^2, 8192^2), CH steps/s, PCIe ceiling.
mkdir -p gpurun_out
timeout 120 python scripts/chtime.py
timeout 120 python scripts/exp/copy_overlap.py
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch1024_launches.csv python scripts/profile_ch.py --n 1024 --steps 20 > /dev/null 2>&1; echo ncu1=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch8192_launches.csv python scripts/profile_ch.py --n 8192 --steps 6 > /dev/null 2>&1; echo ncu2=$?
