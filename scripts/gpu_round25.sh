mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_rhs_v|k_transpose_correct_v|k_sweep_tma|k_combine" -c 4 -o gpurun_out/prof_ch8192 -f python scripts/profile_ch.py --n 8192 --steps 1 > gpurun_out/ncu_ch8192.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_ch8192.log
