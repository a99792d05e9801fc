mkdir -p gpurun_out
scripts/micro/sweep_trace 1024 | head -20
timeout 900 python bench.py > gpurun_out/bench_s2_2.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_s2_2.log
