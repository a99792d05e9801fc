mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stencil_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu3.log
SG_STENCIL_KERNEL=tma timeout 600 python bench.py --steps 100 --warmup 5 --skip-e2e --skip-cpu > gpurun_out/bench_tma3.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_tma3.log
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma3_f64 -f python scripts/profile_stencil.py --reps 3 > gpurun_out/ncu_tma3.log 2>&1; echo ncu=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma3_f32 -f python scripts/profile_stencil.py --reps 3 --dtype f32 > gpurun_out/ncu_tma3b.log 2>&1; echo ncu=$?
