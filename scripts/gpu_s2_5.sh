mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_ch_gpu.py -x -q -m gpu -k steady > gpurun_out/pytest_s2_5.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_5.log
ncu --set full --clock-control none --import-source on -k regex:k_rhs_v -s 1 -c 1 -o gpurun_out/prof_rhs_fused -f python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:k_transpose_correct_v -s 1 -c 1 -o gpurun_out/prof_transpose -f python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
