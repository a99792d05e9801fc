for m in p2p nccl; do for n in 8192 1024; do timeout 300 python scripts/bench_ch_dist.py --n $n --steps 40 --warmup 5 --check --mode $m 2>&1 | tail -1; done; done
