mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s2_23.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke_s2_23.log
timeout 1500 python -m pytest tests/ -q -m gpu > gpurun_out/pytest_s2_23.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_s2_23.log
timeout 600 python bench.py --slab --steps 20 --skip-cpu > gpurun_out/bench_slab_s2_23.log 2>&1; echo slab=$?; tail -1 gpurun_out/bench_slab_s2_23.log | cut -c1-600
