timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_sweep_res" -c 1 -o gpurun_out/prof_sweep_res -f python scripts/profile_ch.py --n 1024 --steps 1 > gpurun_out/ncu_sweep_res.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_sweep_res.log
