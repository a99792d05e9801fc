timeout 600 python bench.py --slab --p2p --steps 30 --skip-cpu --skip-e2e > gpurun_out/bench_p2p.log 2>&1; echo slab_p2p=$?; tail -1 gpurun_out/bench_p2p.log | cut -c1-700
timeout 600 python bench.py --slab --steps 30 --skip-cpu --skip-e2e > gpurun_out/bench_nccl.log 2>&1; echo slab_nccl=$?; tail -1 gpurun_out/bench_nccl.log | cut -c1-250
timeout 600 python -c "
import sys; sys.path.insert(0,'.')
import ctypes as C, torch
import paper_1902_09931_b200 as sg
from paper_1902_09931_b200.ch_dist import ipc_handle_functions
g, o, b = ipc_handle_functions()
t = torch.empty(1000, dtype=torch.float64, device='cuda')
h = g(t[100:].data_ptr())
print('ipc handle bytes', len(h), 'offset', int.from_bytes(h[64:], 'little'))
"
