timeout 900 python -m pytest tests/test_stencil_gpu.py tests/test_slab_gpu.py -q -m gpu -x > gpurun_out/pytest_s2_19.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_s2_19.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import torch, json, bench
import paper_1902_09931_b200 as sg
sg._lib.check(sg._lib.lib().sg_init(0))
peak,_ = bench.measured_peak()
print(json.dumps(bench.bench_variants(sg, torch, torch.cuda.Stream(), peak), indent=1))
"
