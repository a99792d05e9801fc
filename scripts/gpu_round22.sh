set -x
timeout 900 python -m pytest tests/test_slab_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu22.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu22.log
timeout 600 python bench.py --steps 300 --warmup 5 --skip-cpu --skip-extra > gpurun_out/bench22.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench22.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 100 --warmup 3 --slab --skip-cpu > gpurun_out/slab22.log 2>&1; echo slab=$?
tail -1 gpurun_out/slab22.log
