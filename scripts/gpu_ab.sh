# A/B helper: tests + headline bench + stencil variants + ncu bank conflicts of k_tma
timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_slab_gpu.py -q -m gpu -x > gpurun_out/pytest_ab.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_ab.log
timeout 600 python bench.py --skip-cpu --skip-e2e > gpurun_out/bench_ab.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_ab.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['clocks']['sm_mhz']); e=d['extra']; print('fp32', e['cfg4_fp32']['hbm_frac'], 'cfg2', e['cfg2_batched1d_fp64']['hbm_frac'])
for k,v in e['stencil_variants_16384sq_fp64'].items(): print(k, round(v['hbm_frac'],3), round(v['fp64_frac'],3))"
ncu --metrics l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_tma -s 2 -c 1 python scripts/profile_stencil.py --reps 3 2>/dev/null | grep -E "bank|duration|dram" 
