run() { timeout 600 python bench.py --skip-cpu --skip-e2e > gpurun_out/bench_ab12.log 2>&1; tail -1 gpurun_out/bench_ab12.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], round(d['roofline']['frac'],4), d['clocks']['sm_mhz']); e=d['extra']; print('fp32', round(e['cfg4_fp32']['hbm_frac'],4), 'cfg2', round(e['cfg2_batched1d_fp64']['hbm_frac'],4))
print({k: round(v['hbm_frac'],3) for k,v in e['stencil_variants_16384sq_fp64'].items()})"; }
echo "== all lanes"; run
timeout 1200 compute-sanitizer --tool racecheck --print-limit 40 python scripts/sanitize_workload.py > gpurun_out/sanitizer_racecheck.log 2>&1; echo "racecheck rc=$?"; grep -E "RACECHECK SUMMARY|workload OK" gpurun_out/sanitizer_racecheck.log
timeout 1200 compute-sanitizer --tool synccheck python scripts/sanitize_workload.py > gpurun_out/sanitizer_synccheck.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|workload OK" gpurun_out/sanitizer_synccheck.log
timeout 1200 compute-sanitizer --tool memcheck python scripts/sanitize_workload.py > gpurun_out/sanitizer_memcheck.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|workload OK" gpurun_out/sanitizer_memcheck.log
sed -i 's/^#define SG_EMPTY_ALL_LANES 1/#define SG_EMPTY_ALL_LANES 0/' paper_1902_09931_b200/csrc/stencil.cu
python -m paper_1902_09931_b200.build > /dev/null 2>&1
echo "== lane 0"; run
