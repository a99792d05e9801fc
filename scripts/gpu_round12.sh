mkdir -p gpurun_out
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_gpu12.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu12.log
timeout 900 python bench.py > gpurun_out/bench12.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench12.log
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma12_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma12_f32 -f python scripts/profile_stencil.py --reps 3 --dtype f32 > /dev/null 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:"k_rhs|k_transpose|k_combine" -s 3 -c 3 -o gpurun_out/prof_chsmall -f python scripts/profile_ch.py --steps 4 > /dev/null 2>&1; echo ncu=$?
