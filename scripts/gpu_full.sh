# Full round check: GPU tests, smoke, default bench, ncu launch list + top-kernel capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_full.log 2>&1; echo pytest=$?
tail -5 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_full.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?; tail -1 gpurun_out/bench_ref.log
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 5 --warmup 3 --skip-e2e --skip-extra --skip-cpu > /dev/null 2>&1; echo ncu_launch=$?
ncu --set full --clock-control none --import-source on -k regex:k_tma -s 2 -c 1 -o gpurun_out/prof_full_f64 -f python scripts/profile_stencil.py --reps 3 > /dev/null 2>&1; echo ncu=$?
