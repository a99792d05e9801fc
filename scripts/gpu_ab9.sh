timeout 600 python -m pytest tests/test_ch_dist_gpu.py -q -m gpu -x > gpurun_out/pytest_ab9.log 2>&1; echo pytest=$?; tail -15 gpurun_out/pytest_ab9.log
for n in 8192 1024; do timeout 300 python scripts/bench_ch_dist.py --n $n --steps 40 --warmup 5 --check --mode p2p 2>&1 | tail -1 | cut -c1-200; done
