# Full GPU test suite + smoke + sanitizer (memcheck, racecheck) over the workload.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 2400 python -m pytest tests/ -q -m gpu -x --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -9 gpurun_out/pytest_gpu.log
for tool in memcheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|workload OK" gpurun_out/sanitizer_$tool.log | head -3
done
