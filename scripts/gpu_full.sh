# Full check: smoke, GPU tests, default bench, reference arm.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_full.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_full.log
timeout 2400 python -m pytest tests/ -q -m gpu --durations=8 > gpurun_out/pytest_full.log 2>&1; echo pytest=$?; tail -14 gpurun_out/pytest_full.log
timeout 900 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_full.log | cut -c1-400
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-200
