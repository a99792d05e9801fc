# Stencil-family check: GPU tests of the stencil/C++/workers paths, sanitizer
# memcheck + racecheck over the workload, bench variants table.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_stencil_gpu.py tests/test_cxx_gpu.py tests/test_workers_gpu.py tests/test_slab_gpu.py -q -m gpu -x > gpurun_out/pytest_stencil.log 2>&1; echo pytest=$?; tail -5 gpurun_out/pytest_stencil.log
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|workload OK|Error|error" gpurun_out/sanitizer_$tool.log | head -5
done
timeout 900 python bench.py --skip-e2e --skip-cpu --skip-ch --steps 20 --warmup 3 > gpurun_out/bench_var.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_var.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(k, v) for k, v in d['extra']['stencil_variants_16384sq_fp64'].items()]"
