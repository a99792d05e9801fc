mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2_7.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests/ -q -m gpu --durations=8 > gpurun_out/pytest_s2_7.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_s2_7.log
timeout 900 python bench.py > gpurun_out/bench_s2_7.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_s2_7.log
