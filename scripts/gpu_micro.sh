./scripts/micro/fp64_latency
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
