mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_slab_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu19.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu19.log
timeout 600 python bench.py --steps 200 --warmup 5 --skip-e2e --skip-cpu > gpurun_out/bench19.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench19.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['extra'])"
timeout 300 python scripts/bench_ch_dist.py --n 1024 --steps 300 --check; timeout 300 python scripts/bench_ch_dist.py --n 8192 --steps 20
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 50 --warmup 3 --slab
