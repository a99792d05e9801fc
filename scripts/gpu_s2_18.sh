timeout 900 python bench.py --skip-cpu > gpurun_out/bench_s2_18.log 2>&1; echo bench=$?; tail -1 gpurun_out/bench_s2_18.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(json.dumps(d['extra'], indent=1))"
timeout 300 python scripts/bench_ch_dist.py --n 8192 --steps 20 --warmup 3 --check 2>&1 | tail -2
timeout 300 python scripts/bench_ch_dist.py --n 1024 --steps 200 --warmup 10 2>&1 | tail -1
