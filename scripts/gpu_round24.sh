set -x
timeout 900 python -m pytest tests/test_ch_gpu.py tests/test_ch_dist_gpu.py tests/test_slab_gpu.py -x -q -m gpu > gpurun_out/pytest_gpu24.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest_gpu24.log
python scripts/chtime.py
SG_CH_RHS=legacy python scripts/chtime.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch8192_launches24.csv python scripts/profile_ch.py --n 8192 --steps 3 > /dev/null 2>&1; echo ncu=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ch1024_launches24.csv python scripts/profile_ch.py --n 1024 --steps 5 > /dev/null 2>&1; echo ncu=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 50 --warmup 3 --slab --skip-cpu > gpurun_out/slab24.log 2>&1; echo slab=$?
tail -1 gpurun_out/slab24.log | cut -c 1-200; grep -o '"e2e": {[^}]*}' gpurun_out/slab24.log
