set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import paper_1902_09931_b200 as sg; print('ok')"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 50 --warmup 3 --slab > gpurun_out/slab20.log 2>&1; echo slab=$?
tail -5 gpurun_out/slab20.log
timeout 300 python bench.py --steps 50 --warmup 3 --slab > gpurun_out/slab20b.log 2>&1; echo slabb=$?
tail -3 gpurun_out/slab20b.log
