mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_rhs|k_transpose_correct|k_periodic_setup" -s 0 -c 4 -o gpurun_out/prof_ch8192 -f python scripts/profile_ch.py --n 8192 --steps 2 > /dev/null 2>&1; echo ncu=$?
