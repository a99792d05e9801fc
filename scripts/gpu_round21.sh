set -x
timeout 300 python scripts/exp/event_overhead.py
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 50 --warmup 3 --slab --ref-seconds 3 > gpurun_out/slab21.log 2>&1; echo slab=$?
tail -3 gpurun_out/slab21.log
