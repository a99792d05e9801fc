mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_slab_gpu.py tests/test_diagnostics_gpu.py tests/test_ch_dist_gpu.py tests/test_penta_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu11.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu11.log
timeout 600 python bench.py --steps 100 --warmup 5 --skip-e2e --skip-cpu > gpurun_out/bench11.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench11.log | cut -c 1-1800
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma11_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu=$?
timeout 300 python scripts/bench_ch_dist.py --n 1024 --steps 200 --check
