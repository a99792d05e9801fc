echo "xin RS64:"; SG_SWEEP_RS=64 timeout 120 python scripts/chtime.py 1024
echo "xin RS128:"; timeout 120 python scripts/chtime.py 1024
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ --csv --log-file gpurun_out/ch1024_xin.csv python scripts/profile_ch.py --n 1024 --steps 20 > /dev/null 2>&1; echo ncu=$?
