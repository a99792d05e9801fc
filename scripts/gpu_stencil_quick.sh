timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_stream_plans_gpu.py tests/test_jit_gpu.py -q -x -m gpu > gpurun_out/st.log 2>&1; echo rc=$?; tail -3 gpurun_out/st.log
timeout 600 python bench.py --skip-e2e --skip-cpu --skip-ch --steps 20 --warmup 3 > gpurun_out/bench_var.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, round(v['hbm_frac'],3), v['kernel'], v['sm_mhz']) for k, v in d['extra']['stencil_variants_16384sq_fp64'].items()]"
