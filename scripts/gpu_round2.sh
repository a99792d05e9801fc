mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu2.log 2>&1; echo pytest=$?
tail -15 gpurun_out/pytest_gpu2.log
for k in tma reg; do
SG_STENCIL_KERNEL=$k timeout 600 python bench.py --steps 100 --warmup 5 --skip-e2e --skip-cpu --skip-extra > gpurun_out/bench_$k.log 2>&1; echo bench_$k=$?; tail -1 gpurun_out/bench_$k.log | cut -c1-400
done
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_tma_f64 -f python scripts/profile_stencil.py --reps 3 > gpurun_out/ncu_tma.log 2>&1; echo ncu=$?
