"""Config 5: Cahn-Hilliard ADI periodic, FP64, 8192^2 across N GPUs.

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        scripts/bench_ch_dist.py --n 8192 --steps 20 --warmup 3

One process per GPU (NCCL): y-slab halo exchange + two all-to-all
transposes per step (paper_1902_09931_b200/ch_dist.py). Prints one JSON line
(rank 0) with steps/s (max-over-ranks CUDA-event time). With N=1 it runs the
same split step through NCCL-free local paths; `--check` compares C^n after
the run against the single-GPU stepper bitwise.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1902_09931_b200 as sg
    from paper_1902_09931_b200.ch_dist import DistCHStepper

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--mode", choices=["nccl", "p2p"], default="p2p",
                    help="p2p: all-to-alls fused into the sweeps (IPC peer memory); nccl: all_to_all_single")
    a = ap.parse_args()
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    p = sg.CHParams(nx=a.n, ny=a.n)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = DistCHStepper(p, world, rank, dist if world > 1 else None, device=f"cuda:{local}", mode=a.mode)
    for _ in range(a.warmup):
        st.step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    t = torch.tensor([ms], device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    out = {"metric": "Cahn-Hilliard ADI steps/s", "value": 1e3 / ms, "unit": "steps/s", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms, "dtype": "f64",
           "config": {"workload": f"CH BDF2-ADI periodic {a.n}x{a.n}", "parallelism": f"y-slab x{world}, "
                      + ("NCCL halo, all-to-alls fused into the sweeps (P2P TMA stores)" if st.mode == "p2p"
                         else "NCCL halo + 2 all-to-all per step"), "mode": st.mode}}
    if a.check and world == 1:
        single = sg.CHStepper(p)
        single.step_many(a.warmup + a.steps)
        got = st.own_rows(0).cpu().numpy()
        out["bitwise_vs_single_gpu"] = bool(np.array_equal(got.view(np.uint64), single.field().values.view(np.uint64)))
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
