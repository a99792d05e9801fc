#!/usr/bin/env python
"""bench.py — headline benchmark of the B200-native stencil engine.

Workload (BASELINE.json configs[3], the stencil config the metric's HBM
target is quoted on that fits one GPU): 2D XY periodic 9-point user-function
stencil (fn_weighted_3x3, tests/test_stencil.cpp:88-93), FP64, 32768 x 32768
synthetic random field. One step = one stencil application (compute + swap,
stencil.cpp:197-235). value = Gpoints/s over all ranks; the input (8 GiB) is
far larger than L2 (126 MB), so no L2 flush is needed between steps.

Multi-GPU: `--gpus N` with N > 1 runs N ranks, one process per GPU. Without
torchrun's environment bench.py re-launches itself under
`torch.distributed.run --nproc-per-node N` (127.0.0.1); under torchrun it
checks WORLD_SIZE == N. Each rank's slab lives on GPU local_rank % (visible
GPUs) — on a box with fewer GPUs than ranks (tests) the ranks share devices
and the process group falls back to gloo. Reported at N > 1:
  * value (headline, weak scaling): every rank owns a 32768 x 32768 y-slab of
    a periodic (N*32768) x 32768 grid; halo rows go to the ring neighbours
    over NVLink, stored straight into their buffers by the stencil kernel
    (P2P, CUDA IPC) — or NCCL send/recv overlapped with the interior rows;
  * strong: the 32768^2 grid itself split into N slabs;
  * e2e: the strong geometry end to end from pinned host memory;
  * extra.cfg5_ch_8192sq_dist: BASELINE config 5 (Cahn-Hilliard ADI,
    8192^2) on the N ranks (DistCHStepper, P2P form), steps/s, with the
    reference CHStepper's s/step on this host's cores beside it.
Device time is CUDA events on the launching stream, max over ranks.

Also reported: `e2e` (same metric through the C-ABI with HOST pinned grids,
H2D + kernel + D2H per step), `roofline` (dominant kernel vs the measured HBM
copy bandwidth), `cpu_baseline` (the reference library, oracle/_ref, on this
host's cores, the full 32768^2 grid), `clocks`, `gpu_launches`, and `extra`
(secondary configs: FP32 variant, batched 1D config 2, config 1, CH ADI).

`--impl reference` times the reference's own CPU implementation on the same
config (rank 0 only) and prints the same JSON line with "impl": "reference".
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "2D stencil Gpts/s (XY periodic 9-point user-function, FP64)"
UNIT = "Gpts/s"
NX = NY = 32768
BYTES_PER_PT = {"f64": 16, "f32": 8}  # read once + write once
# nominal FP64 (non-tensor) instruction rate: 148 SMs x 64 lanes x 1.965 GHz
# (DADD/DMUL/DFMA one each) — the bound of the tall-window stencils
FP64_PEAK_OPS = 148 * 64 * 1.965e9
WORKLOAD = "2D xy periodic 9-point user-function stencil (fn_weighted_3x3), 32768x32768"


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler for the timed region (B200_PROFILING.md recipe)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = ROOT / "gpurun_out" / f"clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.path.parent.mkdir(exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            # wait for the sampler's first line so the timed region is covered;
            # samples taken before the region starts are dropped in summary()
            t0 = time.time()
            while time.time() - t0 < 5.0 and not self.path.read_text().strip():
                time.sleep(0.02)
            self.skip = len(self.path.read_text().splitlines())
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()
            self.f.close()

    def summary(self):
        if not self.proc or not self.path.exists():
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.path.read_text().splitlines()[getattr(self, "skip", 0):]:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------- reference


def reference_arm(args, rank, world):
    """Time the reference CPU implementation (oracle/_ref: the unmodified
    reference library, all host threads) on the same config: the full
    NX x NY grid, steady_clock around compute() only (bench.cpp:33-40),
    after a steady-state warm-up. Each step is one full-grid application;
    the step count is capped so the run stays within about a minute."""
    if rank != 0:
        return
    nx = args.nx
    line = cpu_reference_sample(nx, target_s=args.ref_seconds * 5, max_reps=args.steps,
                                warmup=max(args.warmup, 3), single_worker=True)
    out = {"metric": METRIC, "value": line["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": line["reps"],
           "warmup": max(args.warmup, 3), "ms_per_step": line["ms_per_app"], "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": WORKLOAD if nx == NX else f"{WORKLOAD} (test size {nx}x{nx})",
                      "nx": nx, "ny": nx, "sample_rows": nx},
           "impl": "reference",
           "cpu_baseline": {"value": line["value"], "unit": UNIT, "cores": line["cores"],
                            "kind": line["kind"], "sample": line["sample"], "cpu_model": line["cpu_model"],
                            "one_worker": line.get("one_worker")},
           "e2e": {"value": line["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def host_cores():
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def cpu_reference_sample(nx=NX, target_s=12.0, max_reps=200, warmup=3, single_worker=False):
    """Reference compute() on the FULL nx x nx periodic grid of the config,
    numWorkers = numTiles = host threads, steady_clock around compute() only
    (bench.cpp:33-40), mean over as many applications as fit in ~target_s
    (at least 2). single_worker adds one numWorkers=1 application (§8(d)).
    Falls back to the C restatement (kind "port") only if the reference
    library was never built."""
    import numpy as np
    from oracle.oracle import Reference, Restatement
    cores = host_cores()
    rng = np.random.default_rng(4)
    inp = rng.uniform(-1.0, 1.0, (nx, nx))
    w = rng.uniform(-1.0, 1.0, 9)
    pts = nx * nx
    one = None
    try:
        ref = Reference()
        kind = "reference"
        run = dict(fn="fn_weighted_3x3", tiles=min(cores, nx), workers=cores)
        t1 = ref.stencil_timed(inp, (1, 1, 1, 1), w, warmup=warmup, reps=1, **run)
        reps = int(max(2, min(max_reps, target_s / max(t1, 1e-6))))
        secs = ref.stencil_timed(inp, (1, 1, 1, 1), w, warmup=0, reps=reps, **run)
        if single_worker:
            s1 = ref.stencil_timed(inp, (1, 1, 1, 1), w, fn="fn_weighted_3x3", tiles=1, workers=1, warmup=0, reps=1)
            one = {"value": pts / s1 / 1e9, "unit": UNIT, "workers": 1, "s_per_app": s1}
    except FileNotFoundError:
        orc = Restatement()
        kind = "port"
        cores = 1
        t0 = time.perf_counter()
        reps = 1
        orc.stencil(inp, (1, 1, 1, 1), w, fn="fn_weighted_3x3")
        secs = time.perf_counter() - t0
    return {"value": pts / secs / 1e9, "cores": cores, "kind": kind, "reps": reps, "rows": nx,
            "ms_per_app": secs * 1e3, "cpu_model": cpu_model(), "one_worker": one,
            "sample": f"the full {nx}x{nx} periodic grid (fn_weighted_3x3, FP64), {warmup} warm-up + "
                      f"{reps} timed compute() calls, numWorkers=numTiles={cores}"}


def cpu_baseline_line(args):
    cb = cpu_reference_sample(args.nx, target_s=args.ref_seconds)
    return {"value": cb["value"], "unit": UNIT, "cores": cb["cores"], "kind": cb["kind"], "sample": cb["sample"],
            "cpu_model": cb["cpu_model"]}


def cpu_reference_ch(n, steps=3):
    """Seconds per CHStepper::step of the reference (oracle/_ref) at n x n on
    this host's cores (numTiles = numWorkers = cores), construction excluded
    (ch_timed: steady_clock around `steps` steps) — config 5's CPU baseline."""
    try:
        from oracle.oracle import Reference, ch_params
        cores = host_cores()
        s = Reference().ch_timed(ch_params(n), steps, warmup=0, tiles=cores, workers=cores)
        return {"s_per_step": s, "steps_s": 1.0 / s, "cores": cores, "timed_steps": steps,
                "kind": "reference (oracle/_ref CHStepper::step)", "cpu_model": cpu_model()}
    except Exception as e:  # reported context only
        return {"error": repr(e)[:200]}


# --------------------------------------------------------------------- ours


def time_plan_steps(sg, torch, plan, steps, stream, per_launch=False):
    """Run `steps` compute+swap steps on `stream`, timed by CUDA events on
    that stream. Returns (total_ms, [per-launch ms]). Each step is exactly
    one kernel launch and nothing else runs on the stream, so the mean
    launch duration is total/steps; per-launch events (per_launch=True)
    measure the same thing but cost ~1 % (they break back-to-back launch
    overlap), so the headline does not record them."""
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)] if per_launch else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for k in range(steps):
        if ev:
            ev[k][0].record(stream)
        sg.compute(plan, stream=stream, synchronize=False)
        if ev:
            ev[k][1].record(stream)
        sg.swap_plan(plan)
    end.record(stream)
    end.synchronize()
    total = start.elapsed_time(end)
    return total, ([a.elapsed_time(b) for a, b in ev] if ev else [total / max(steps, 1)] * steps)


def bench_device_stencil(sg, torch, dtype, nx, ny, steps, warmup, stream, fn="fn_weighted_3x3"):
    import numpy as np
    tdt = torch.float64 if dtype == "f64" else torch.float32
    g = torch.Generator(device="cuda").manual_seed(4)
    a = torch.rand((ny, nx), dtype=tdt, device="cuda", generator=g).mul_(2).sub_(1)
    b = torch.empty_like(a)
    w = list(np.random.default_rng(4).uniform(-1, 1, 9))
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), fn, w), a, b, 1, 1)
    stream.wait_stream(torch.cuda.current_stream())  # the input is generated there
    with torch.cuda.stream(stream):
        time_plan_steps(sg, torch, plan, warmup, stream)
        torch.cuda.synchronize()
        l0 = sg.launch_count()
        total_ms, per = time_plan_steps(sg, torch, plan, steps, stream)
        launches = sg.launch_count() - l0
    sg.destroy_plan(plan)
    del a, b
    torch.cuda.empty_cache()
    return total_ms, per, launches


def bench_e2e(sg, torch, nx, ny, steps):
    """Same metric through the C ABI with HOST (pinned) grids: every step
    uploads the input, runs the kernel and downloads the output."""
    import numpy as np
    hin = torch.empty((ny, nx), dtype=torch.float64, pin_memory=True)
    hout = torch.empty((ny, nx), dtype=torch.float64, pin_memory=True)
    hin.uniform_(-1, 1)
    gi, go = sg.Grid2D.from_array(hin.numpy()), sg.Grid2D.from_array(hout.numpy())
    w = list(np.random.default_rng(4).uniform(-1, 1, 9))
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic,
                          sg.FunctionStencil(sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", w), gi, go, 1, 1)
    sg.compute(plan, sg.Residency.Host)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        sg.compute(plan, sg.Residency.Host)  # H2D + kernel + D2H, synchronous
    dt = time.perf_counter() - t0
    sg.destroy_plan(plan)
    nbytes = nx * ny * 8
    ceiling = pcie_ceiling(torch, hin, hout)
    value = nx * ny * steps / dt / 1e9
    return {"value": value, "unit": UNIT, "h2d_bytes_per_step": nbytes,
            "d2h_bytes_per_step": nbytes, "steps": steps,
            "path": "sg_plan_compute(Residency::Host) on pinned host Grid2D buffers",
            "pcie_ceiling": ceiling,
            "frac_of_pcie_ceiling": value / ceiling["gpts_s"] if ceiling else None}


def pcie_ceiling(torch, hin, hout, chunks=16):
    """The bound e2e runs into: the same bytes moved H2D and D2H concurrently
    (two streams, pinned buffers, no kernel) — plain copies, best of 3 (16
    chunks: torch's per-copy overhead makes 128 chunks measure lower than
    the C ABI pipeline itself achieves)."""
    try:
        n = hin.numel()
        flat_in, flat_out = hin.view(-1), hout.view(-1)
        da = torch.empty(n, dtype=hin.dtype, device="cuda")
        db = torch.empty(n, dtype=hin.dtype, device="cuda")
        s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
        cuts = [n * c // chunks for c in range(chunks + 1)]
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            with torch.cuda.stream(s1):
                for a, b in zip(cuts, cuts[1:]):
                    da[a:b].copy_(flat_in[a:b], non_blocking=True)
            with torch.cuda.stream(s2):
                for a, b in zip(cuts, cuts[1:]):
                    flat_out[a:b].copy_(db[a:b], non_blocking=True)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        del da, db
        torch.cuda.empty_cache()
        nbytes = n * hin.element_size()
        return {"gpts_s": n / best / 1e9, "h2d_plus_d2h_gbs": 2 * nbytes / best / 1e9,
                "how": "concurrent H2D + D2H torch copies of the step's bytes, pinned, 2 streams"}
    except Exception as e:  # reported context only
        return {"error": repr(e)}


def extras(sg, torch, stream, peak, args):
    """Secondary BASELINE.json configs, short runs; reported, not headline."""
    import numpy as np
    out = {}
    # FP32 variant of config 4.
    tot, per, _ = bench_device_stencil(sg, torch, "f32", NX, NY, 50, 5, stream)
    kms = statistics.mean(per)
    out["cfg4_fp32"] = {"gpts_s": NX * NY / kms / 1e6, "kernel_ms": kms,
                        "hbm_frac": NX * NY * 8 / (kms * 1e-3) / 1e9 / peak}
    # Config 2: batched 1D non-periodic 4th-derivative, 4096 x 4096 FP64,
    # L2 flushed (256 MB write) between timed launches.
    n = 4096
    dx = 2 * np.pi / n
    s4 = 1.0 / (dx ** 4)
    a = torch.rand((n, n), dtype=torch.float64, device="cuda")
    b = torch.zeros_like(a)
    # L2 flush between timed launches: write 256 MB (> 126 MB L2), then read
    # another 256 MB so the lines left in L2 are clean — otherwise the
    # flush's dirty lines are written back during the timed kernel.
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    flush_rd = torch.ones(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    plan = sg.create_plan(sg.Direction.X, sg.BoundaryMode.NonPeriodic,
                          sg.WeightStencil(sg.Extents(2, 2, 0, 0), [s4, -4 * s4, 6 * s4, -4 * s4, s4]), a, b, 1, 1)
    ts = []
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        for k in range(23):
            flush.zero_()
            flush_rd.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            sg.compute(plan, stream=stream, synchronize=False)
            e1.record(stream)
            e1.synchronize()
            if k >= 3:
                ts.append(e0.elapsed_time(e1))
    sg.destroy_plan(plan)
    kms = statistics.median(ts)
    alg = n * n * 8 + n * (n - 4) * 8
    out["cfg2_batched1d_fp64"] = {"gpts_s": n * (n - 4) / kms / 1e6, "kernel_ms": kms,
                                  "hbm_frac": alg / (kms * 1e-3) / 1e9 / peak,
                                  "l2": "flushed (256 MB write + 256 MB read between launches)"}
    del a, b, flush, flush_rd
    torch.cuda.empty_cache()
    # Config 1: 512^2 XY periodic 5-point Laplacian, 10 applications
    # (Residency::Device between applications, one sync at the end).
    m = 512
    dx = 2 * np.pi / m
    cx = 1.0 / (dx * dx)
    lap = [0.0, cx, 0.0, cx, -2 * cx - 2 * cx, cx, 0.0, cx, 0.0]
    x = np.random.default_rng(1).uniform(-1, 1, (m, m))
    gi, go = sg.Grid2D.from_array(x), sg.Grid2D(m, m)
    plan = sg.create_plan(sg.Direction.XY, sg.BoundaryMode.Periodic, sg.WeightStencil(sg.Extents(1, 1, 1, 1), lap),
                          gi, go, 1, 1)
    best = 1e9
    for _ in range(5):
        t0 = time.perf_counter()
        for k in range(10):
            sg.compute(plan, sg.Residency.Device if k < 9 else sg.Residency.Host)
            if k < 9:
                sg.swap_plan(plan)
        best = min(best, time.perf_counter() - t0)
    sg.destroy_plan(plan)
    out["cfg1_512sq_10apps_ms"] = best * 1e3
    out["stencil_variants_16384sq_fp64"] = bench_variants(sg, torch, stream, peak)
    out["stencil_variants_16384sq_fp32"] = bench_variants(sg, torch, stream, peak, dtype="f32")
    out["penta_general_periodic"] = bench_penta_general(sg, torch, peak)
    out["weno5_advect_8192sq_fp64"] = bench_weno(sg, torch, peak)
    if not args.skip_ch:
        out.update(bench_ch(sg, torch, args))
    return out


def bench_penta_general(sg, torch, peak, B=65536, n=1024, reps=10):
    """PeriodicPentaFactor::solve_in_place on a batch of B NON-uniform
    periodic systems (per-system factor tables, penta.cpp:160-295), rhs
    device-resident. Bytes per solve: 9 factor tables read + z read and
    written twice (forward/backward) + the Woodbury correction pass."""
    import numpy as np
    rng = np.random.default_rng(3)
    m = sg.PentaBatch(B, n, True)
    for band in m.bands():
        band[:] = rng.uniform(-1, 1, (n, B))
    m.diag += 6.0
    f = sg.PeriodicPentaFactor(m)
    rhs = torch.rand((n, B), dtype=torch.float64, device="cuda")
    for _ in range(3):
        f.solve_in_place(rhs)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f.solve_in_place(rhs)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    alg = (9 + 4 + 2) * B * n * 8  # tables + sweep z traffic + correction (read+write)
    del f, rhs
    torch.cuda.empty_cache()
    return {"batch": B, "n": n, "solve_ms": ms, "unknowns_per_s": B * n / (ms * 1e-3),
            "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak}


def bench_weno(sg, torch, peak, n=8192, reps=10, ref_n=1024):
    """weno_advect (weno.cpp:50-94) through the C ABI on device-resident
    fields: reads phi, u, v and writes the tendency (32 B/pt), ~150 FP64 ops
    per point incl. four divisions. The reference's CPU weno_advect is timed
    beside it on a ref_n^2 sample with all host cores (oracle/_ref)."""
    import ctypes as C
    import os
    import numpy as np
    from paper_1902_09931_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(5)
    phi, u, v = (torch.rand((n, n), dtype=torch.float64, device="cuda", generator=g) - 0.5 for _ in range(3))
    out = torch.empty_like(phi)
    dx = 2 * np.pi / n
    st = torch.cuda.current_stream()

    def call():
        _lib.check(_lib.lib().sg_weno_advect(C.c_void_p(phi.data_ptr()), C.c_void_p(u.data_ptr()),
                                             C.c_void_p(v.data_ptr()), n, n, dx, dx, C.c_void_p(out.data_ptr()),
                                             1, C.c_void_p(st.cuda_stream)))
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    pts = n * n
    res = {"gpts_s": pts / (ms * 1e-3) / 1e9, "kernel_ms": ms,
           "hbm_frac": 32 * pts / (ms * 1e-3) / 1e9 / peak, "inputs": "device-resident, 3 reads + 1 write of 8 B/pt",
           "l2": "inputs 1.6 GB >> L2"}
    del phi, u, v, out
    torch.cuda.empty_cache()
    try:
        from oracle.oracle import Reference
        ref = Reference()
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        rng = np.random.default_rng(6)
        a, b, c = (rng.uniform(-0.5, 0.5, (ref_n, ref_n)) for _ in range(3))
        d = 2 * np.pi / ref_n
        ref.weno_advect(a, b, c, d, d, cores, cores)
        t0 = time.perf_counter()
        ref.weno_advect(a, b, c, d, d, cores, cores)
        secs = time.perf_counter() - t0
        res["reference_cpu"] = {"gpts_s": ref_n * ref_n / secs / 1e9, "cores": cores,
                                "sample": f"{ref_n}x{ref_n} weno_advect (oracle/_ref), numTiles=numWorkers={cores}"}
    except Exception as exc:  # the reference build is optional on a bare box
        res["reference_cpu"] = {"error": str(exc)[:200]}
    return res


def bench_variants(sg, torch, stream, peak, n=16384, launches=20, dtype="f64"):
    """HBM roofline fraction of the fast path across the API surface
    (directions, boundary modes, window sizes, weights vs functions) on a
    16384^2 grid (2 GiB per FP64 field >> L2); dtype "f32" runs a subset in
    FP32 (rows at four 16 B phases for the odd widths)."""
    import numpy as np
    rng = np.random.default_rng(9)
    f32 = dtype == "f32"
    cases = [
        ("x_nonperiodic_5pt_weights", sg.Direction.X, sg.BoundaryMode.NonPeriodic, sg.Extents(2, 2, 0, 0), None, 5),
        ("y_periodic_5pt_weights", sg.Direction.Y, sg.BoundaryMode.Periodic, sg.Extents(0, 0, 2, 2), None, 5),
        ("xy_periodic_3x3_weights", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(1, 1, 1, 1), None, 9),
        ("xy_periodic_5x5_weights", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(2, 2, 2, 2), None, 25),
        ("xy_periodic_9x9_weights", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(4, 4, 4, 4), None, 81),
        ("xy_nonperiodic_3x3_weights", sg.Direction.XY, sg.BoundaryMode.NonPeriodic, sg.Extents(1, 1, 1, 1), None, 9),
        ("xy_periodic_ch_nonlinear_window", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(1, 1, 1, 1),
         "ch_nonlinear_window", 9),
        # k_tma_g: asymmetric windows (test_stencil.cpp:557-568) and odd rows
        ("x_periodic_asym_3_1_0_0_weights", sg.Direction.X, sg.BoundaryMode.Periodic, sg.Extents(3, 1, 0, 0), None, 5),
        ("xy_periodic_asym_2_1_1_2_weights", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(2, 1, 1, 2), None,
         16),
        ("xy_periodic_3x3_fn_weighted_odd_nx_16383", sg.Direction.XY, sg.BoundaryMode.Periodic,
         sg.Extents(1, 1, 1, 1), "fn_weighted_3x3", 9),
        ("xy_nonperiodic_3x3_weights_odd_nx_16383", sg.Direction.XY, sg.BoundaryMode.NonPeriodic,
         sg.Extents(1, 1, 1, 1), None, 9),
        # k_generic: a window past k_tma_g's 9 x 9 (11 x 11 weights)
        ("xy_periodic_11x11_weights_generic", sg.Direction.XY, sg.BoundaryMode.Periodic, sg.Extents(5, 5, 5, 5),
         None, 121),
    ]
    if f32:
        keep = ("xy_periodic_3x3_weights", "xy_periodic_5x5_weights", "x_periodic_asym_3_1_0_0_weights",
                "xy_periodic_asym_2_1_1_2_weights", "xy_periodic_3x3_fn_weighted_odd_nx_16383")
        cases = [c for c in cases if c[0] in keep]
    a = torch.rand((n, n), dtype=torch.float32 if f32 else torch.float64, device="cuda")
    b = torch.zeros_like(a)
    esz = 4 if f32 else 8
    stream.wait_stream(torch.cuda.current_stream())
    res = {}
    for name, d, mode, ext, fn, nv in cases:
        vals = list(rng.uniform(-1, 1, nv))
        kind = sg.WeightStencil(ext, vals) if fn is None else sg.FunctionStencil(ext, fn, vals)
        nxv = n - 1 if "odd_nx" in name else n
        ai = a.view(-1)[: n * nxv].view(n, nxv)
        bo = b.view(-1)[: n * nxv].view(n, nxv)
        plan = sg.create_plan(d, mode, kind, ai, bo, 1, 1)
        kk = plan.kernel_kind()
        with torch.cuda.stream(stream):
            t2, _ = time_plan_steps(sg, torch, plan, 2, stream)
            # >= 0.4 s per variant so the clock sampler sees it (FP64-bound
            # windows run power-capped below the nominal clock)
            reps = max(3 if "generic" in name else launches, int(400.0 / max(t2 / 2, 1e-3)))
            with Clocks(torch.cuda.current_device()) as clk:
                tot, _ = time_plan_steps(sg, torch, plan, reps, stream)
        sg.destroy_plan(plan)
        ms = tot / reps
        csum = clk.summary()
        rows = n - (ext.top + ext.bottom if mode == sg.BoundaryMode.NonPeriodic else 0)
        cols = nxv - (ext.left + ext.right if mode == sg.BoundaryMode.NonPeriodic else 0)
        alg = esz * (n * nxv + rows * cols)
        # FP64 instructions per output point (no FMA contraction: a multiply
        # and an add per tap; the CH window adds c^3 - c once per INPUT point —
        # the kernel's register window shares it between the windows that
        # read the point, so 2 * 9 + 3, not 5 per tap)
        ops = 2 * nv + 3 if fn == "ch_nonlinear_window" else 2 * nv
        if f32 and fn is None:
            ops = nv  # FP32 taps contract to one FFMA each (sg_mac)
        rate = ops * rows * cols / (ms * 1e-3)
        fp = "fp32" if f32 else "fp64"
        lanes = 128 if f32 else 64  # FP32 / FP64 lanes per SM per cycle
        res[name] = {"gpts_s": rows * cols / (ms * 1e-3) / 1e9, "kernel_ms": ms,
                     "hbm_frac": alg / (ms * 1e-3) / 1e9 / peak,
                     f"{fp}_ops_per_pt": ops, f"{fp}_frac": rate / (148 * lanes * 1.965e9),
                     "sm_mhz": csum.get("sm_mhz"), "clock_reasons": csum.get("reasons"),
                     f"{fp}_frac_at_clock": (rate / (148 * lanes * csum["sm_mhz"] * 1e6)) if csum.get("sm_mhz") else None,
                     "kernel": {2: "k_tma_g", 1: "k_tma", 0: "k_generic"}[kk], "nx": nxv}
    del a, b
    torch.cuda.empty_cache()
    return res


def bench_ch(sg, torch, args, n=1024, steps=1000):
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = steps * p.dt
    st = sg.CHStepper(p)
    st.step_many(20)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.step_many(steps)
    st.synchronize()
    dt = time.perf_counter() - t0
    out = {"cfg3_ch_1024sq_steps_s": steps / dt, "cfg3_ch_1024sq_1000steps_s": dt}
    # opt-in partitioned sweeps (sg_ch_set_partition): not bitwise; deviation
    # from the bitwise path (= the reference) after 100 steps reported beside
    import numpy as np
    ref100 = sg.CHStepper(p)
    ref100.step_many(100)
    c_ref = ref100.field().values.copy()
    del ref100
    part = {}
    for P in (4, 8):
        sp = sg.CHStepper(p)
        sp.set_partition(P)
        sp.step_many(100)
        err = float(np.linalg.norm(sp.field().values - c_ref) / np.linalg.norm(c_ref))
        sp.step_many(20)
        sp.synchronize()
        t0 = time.perf_counter()
        sp.step_many(steps)
        sp.synchronize()
        part[f"P{P}"] = {"steps_s": steps / (time.perf_counter() - t0), "rel_l2_after_100_steps_vs_bitwise": err}
        del sp
    out["cfg3_ch_1024sq_partitioned_opt_in"] = part
    # end to end through the public API: host initial state uploaded
    # (set_state), 1000 steps, field read back to the host
    import numpy as np
    from paper_1902_09931_b200.stencil import Grid2D
    c0 = Grid2D.from_array(np.random.default_rng(1).uniform(-0.1, 0.1, (n, n)))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.set_state(c0, c0)
    st.step_many(steps)
    host = st.field().values
    e2e = time.perf_counter() - t0
    out["cfg3_ch_1024sq_e2e_1000steps_s"] = e2e
    out["cfg3_ch_1024sq_e2e_bytes"] = {"h2d": 2 * n * n * 8, "d2h": int(host.nbytes)}
    del st
    # the reference CHStepper (oracle/_ref) on this host's cores, 5 timed steps
    try:
        from oracle.oracle import Reference
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        pr = dict(D=p.D, gamma=p.gamma, lx=p.lx, ly=p.ly, dt=p.dt, T=p.T, nx=n, ny=n, seed=1, amp=0.1,
                  nonlinear=True)
        per_step = Reference().ch_timed(pr, 5, warmup=1, tiles=cores, workers=cores)  # seconds per step
        out["cfg3_ch_1024sq_reference_steps_s"] = {"value": 1.0 / per_step, "cores": cores, "timed_steps": 5,
                                                   "kind": "reference (oracle/_ref CHStepper::step)"}
    except Exception as e:  # reported context only
        out["cfg3_ch_1024sq_reference_steps_s"] = {"error": repr(e)}
    # Config 5's grid (8192^2) on ONE GPU: the single-device stepper, 40 steps.
    n5 = args.ch_n
    p = sg.CHParams(nx=n5, ny=n5)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = sg.CHStepper(p)
    st.step_many(5)
    st.synchronize()
    t0 = time.perf_counter()
    st.step_many(args.ch_steps)
    st.synchronize()
    dt = time.perf_counter() - t0
    out["cfg5_grid_ch_8192sq_1gpu_steps_s"] = args.ch_steps / dt
    del st
    torch.cuda.empty_cache()
    # the distributed stepper (config 5's multi-GPU path) at world = 1, and
    # the reference CHStepper at 8192^2 on this host's cores beside it
    from paper_1902_09931_b200.ch_dist import DistCHStepper
    dst = DistCHStepper(p, 1, 0, None, mode="p2p")
    for _ in range(3):
        dst.step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.ch_steps):
        dst.step()
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.ch_steps
    out["cfg5_ch_8192sq_dist"] = {"steps_s": 1e3 / ms, "ms_per_step": ms, "n": n5, "n_gpus": 1,
                                  "mode": dst.mode, "timed_steps": args.ch_steps}
    del dst
    torch.cuda.empty_cache()
    if not args.skip_cpu:
        out["cfg5_ch_8192sq_dist"]["reference_cpu"] = cpu_reference_ch(n5)
    return out


def ours_arm(args, rank, world, local_rank):
    import torch

    import paper_1902_09931_b200 as sg
    ndev = torch.cuda.device_count()
    if ndev < 1:
        raise SystemExit("bench.py: no CUDA device visible (there is no CPU fallback)")
    dev = local_rank % ndev
    torch.cuda.set_device(dev)
    sg._lib.check(sg._lib.lib().sg_init(dev))
    peak, peak_kind = measured_peak()
    if world > 1 or args.slab:
        line = multi_gpu_arm(args, rank, world, local_rank, dev, ndev, peak, peak_kind)
        if line is not None:
            print(json.dumps(line), flush=True)
        return

    nx = ny = args.nx
    stream = torch.cuda.Stream()
    with Clocks(dev) as clk:
        total_ms, per, launches = bench_device_stencil(sg, torch, "f64", nx, ny, args.steps, args.warmup, stream)
    clocks = clk.summary()
    ms = total_ms / args.steps
    value = nx * ny / (ms * 1e-3) / 1e9
    kms = statistics.mean(per)
    alg_bytes = nx * ny * BYTES_PER_PT["f64"]
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    traffic = None
    tp = ROOT / "profiles" / "traffic_r02.json"
    if tp.exists() and nx == NX:
        traffic = json.loads(tp.read_text()).get("bytes_per_launch")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD if nx == NX else f"{WORKLOAD} (test size {nx}x{nx})",
                   "nx": nx, "ny": ny, "fn": "fn_weighted_3x3",
                   "boundary": "periodic", "direction": "xy", "l2": "input 8 GiB >> 126 MB L2, no flush needed",
                   "parallelism": "single GPU", "timed_region_s": total_ms / 1e3},
        "strong": {"value": value, "unit": UNIT, "ms_per_step": ms,
                   "note": "N = 1: the strong- and weak-scaling workloads are the same 32768^2 grid"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": "k_tma<double,1,1,1,1,OpWeighted3x3>", "kernel_ms": kms,
                     "kernel_timing": "CUDA events on the launching stream around the timed region "
                                      "/ launches (one k_tma launch per step)",
                     "algorithmic_bytes_per_launch": alg_bytes},
        "clocks": clocks,
        "gpu_launches": int(launches),
    }
    if not args.skip_e2e:
        line["e2e"] = bench_e2e(sg, torch, nx, ny, args.e2e_steps)
    if not args.skip_extra:
        try:
            line["extra"] = extras(sg, torch, stream, peak, args)
        except Exception as e:  # secondary numbers must not kill the headline
            line["extra"] = {"error": repr(e)}
    if not args.skip_cpu:
        line["cpu_baseline"] = cpu_baseline_line(args)
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ multi-GPU


def multi_gpu_arm(args, rank, world, local_rank, dev, ndev, peak, peak_kind):
    """N ranks, one per GPU (torchrun). Weak scaling (headline), strong
    scaling, e2e on the strong geometry, and config 5 (CH 8192^2) on the N
    ranks. Returns rank 0's JSON line (None elsewhere)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1902_09931_b200 import _lib
    from paper_1902_09931_b200.slab import Slab, SlabStencil, enable_p2p_ipc
    from paper_1902_09931_b200.stencil import Extents, FunctionStencil

    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    shared = local_world > ndev  # ranks share GPUs (tests on a 1-GPU box): NCCL refuses that
    backend = "gloo" if shared else "nccl"
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group("gloo")
    assert dist.get_world_size() == world == args.gpus, (dist.get_world_size(), world, args.gpus)
    red_dev = f"cuda:{dev}" if backend == "nccl" else "cpu"

    def reduce(x, op):
        t = torch.tensor([float(x)], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def sync_all():
        torch.cuda.synchronize()
        dist.barrier()

    nx = args.nx
    w = list(np.random.default_rng(4).uniform(-1, 1, 9))
    kind = FunctionStencil(Extents(1, 1, 1, 1), "fn_weighted_3x3", w)

    def make(ny_total):
        slab = Slab(nx, ny_total, world, rank, 1, 1, True)
        st = SlabStencil(slab, (1, 1, 1, 1), kind, torch.float64, f"cuda:{dev}", dist)
        g = torch.Generator(device=f"cuda:{dev}").manual_seed(4 + rank)
        st.own_view(st.a).copy_(torch.rand((slab.own, nx), dtype=torch.float64, device=f"cuda:{dev}",
                                           generator=g))
        halo = "nccl"
        torch.cuda.synchronize()
        if args.halo == "p2p" and enable_p2p_ipc(st, dist):
            halo = "p2p"
        elif backend != "nccl":
            raise SystemExit("bench.py: ranks sharing a GPU need the P2P halo path (gloo has no CUDA send/recv)")
        return slab, st, halo

    def timed(st, steps, clk=None):
        for _ in range(args.warmup):
            st.apply()
            st.swap()
        sync_all()
        l0 = _lib.launch_count()
        if clk:
            clk.__enter__()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            st.apply()
            st.swap()
        e1.record()
        torch.cuda.synchronize()
        if clk:
            clk.__exit__(None, None, None)
        launches = _lib.launch_count() - l0
        ms = reduce(e0.elapsed_time(e1) / steps, dist.ReduceOp.MAX)
        return ms, int(reduce(launches, dist.ReduceOp.SUM))

    # weak scaling (headline): one nx x nx slab per rank
    slab, st, halo = make(nx * world)
    clk = Clocks(dev) if rank == 0 else None
    ms_w, launches = timed(st, args.steps, clk)
    del st
    torch.cuda.empty_cache()
    sync_all()
    # strong scaling: the nx x nx grid split into `world` slabs
    slab_s, st, halo_s = make(nx)
    ms_s, _ = timed(st, args.steps)
    e2e = None
    if not args.skip_e2e and args.e2e_steps > 0:
        e2e = multi_gpu_e2e(args, torch, dist, st, slab_s, reduce, sync_all)
    del st
    torch.cuda.empty_cache()
    sync_all()
    ch = None
    if not args.skip_ch:
        ch = bench_ch_dist(args, torch, dist, rank, world, dev, backend, reduce, sync_all)
    line = None
    if rank == 0:
        value = nx * nx * world / (ms_w * 1e-3) / 1e9
        alg = nx * nx * 16  # per GPU per step
        strong_value = nx * nx / (ms_s * 1e-3) / 1e9
        halo_txt = ("halo rows stored into the neighbours' buffers by the stencil kernel (P2P over NVLink, "
                    "CUDA IPC)" if halo == "p2p" else "NCCL halo send/recv overlapped with the interior rows")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_w, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": (WORKLOAD if nx == NX else f"{WORKLOAD} (test size {nx})")
                           + f", weak scaling: {nx}x{nx} y-slab per GPU ({nx}x{nx * world} total)",
                           "nx": nx, "ny": nx * world, "parallelism": f"y-slab x{world}, {halo_txt}",
                           "backend": backend, "ranks_share_gpus": shared,
                           "l2": "input 8 GiB per GPU >> L2", "timed_region_s": ms_w * args.steps / 1e3},
                "strong": {"value": strong_value, "unit": UNIT, "ms_per_step": ms_s,
                           "workload": f"the {nx}x{nx} grid split into {world} y-slabs of {slab_s.own} rows",
                           "per_gpu_hbm_frac": nx * slab_s.own * 16 / (ms_s * 1e-3) / 1e9 / peak,
                           "halo": halo_s},
                "roofline": {"bound": "hbm", "achieved": alg / (ms_w * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                             "frac": alg / (ms_w * 1e-3) / 1e9 / peak, "traffic": None, "peak_kind": peak_kind,
                             "kernel": "k_tma<double,1,1,1,1,OpWeighted3x3> (P2P variant)",
                             "note": "per-GPU algorithmic bytes / per-GPU step time incl. the halo exchange"},
                "gpu_launches": launches}
        if clk:
            line["clocks"] = clk.summary()
        if e2e:
            line["e2e"] = e2e
        if ch:
            line["extra"] = {"cfg5_ch_8192sq_dist": ch}
    dist.destroy_process_group()
    if rank == 0 and ch and "skipped" not in ch and not args.skip_cpu:
        line["extra"]["cfg5_ch_8192sq_dist"]["reference_cpu"] = cpu_reference_ch(args.ch_n)
    return line


def multi_gpu_e2e(args, torch, dist, st, slab, reduce, sync_all):
    """The strong geometry end to end: every rank uploads its ext rows (own
    + halo rows, read from pinned host memory — a host-resident grid), runs
    the kernel and downloads its own output rows (SlabStencil.apply_host).
    Wall clock between barriers, max over ranks."""
    nx = slab.nx
    try:
        hin = torch.empty((slab.ext_rows, nx), dtype=torch.float64, pin_memory=True)
        hout = torch.empty((slab.own, nx), dtype=torch.float64, pin_memory=True)
        ok = 1.0
    except RuntimeError:
        ok = 0.0
    if reduce(ok, dist.ReduceOp.MIN) < 1.0:
        return {"error": "pinned host buffers could not be allocated"}
    hin.uniform_(-1, 1)
    st.apply_host(hin, hout)  # warm-up
    sync_all()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        st.apply_host(hin, hout)
    dt = reduce(time.perf_counter() - t0, dist.ReduceOp.MAX)
    h2d = int(reduce(slab.ext_rows * nx * 8, dist.ReduceOp.SUM))
    d2h = int(reduce(slab.own * nx * 8, dist.ReduceOp.SUM))
    return {"value": nx * nx * args.e2e_steps / dt / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
            "path": "SlabStencil.apply_host on every rank: ext rows (own + halo) uploaded from pinned host "
                    "memory, own output rows downloaded, row-chunk pipelined; the strong-scaling geometry"}


def bench_ch_dist(args, torch, dist, rank, world, dev, backend, reduce, sync_all):
    """BASELINE config 5: Cahn-Hilliard ADI periodic FP64 at ch_n^2 on the
    `world` ranks (DistCHStepper, P2P form: the all-to-alls fused into the
    sweeps' stores; CUDA-graph replay of each step over NCCL). steps/s from
    CUDA events on the compute stream, max over ranks."""
    import paper_1902_09931_b200 as sg
    from paper_1902_09931_b200.ch_dist import DistCHStepper
    n = args.ch_n
    if n % world:
        return {"skipped": f"{n}x{n} does not split into {world} equal y-slabs (CHParams needs a power of two)",
                "n_gpus": world}
    p = sg.CHParams(nx=n, ny=n)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = DistCHStepper(p, world, rank, dist, device=f"cuda:{dev}", mode="p2p")
    for _ in range(3):
        st.step()
    sync_all()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.ch_steps):
        st.step()
    e1.record()
    torch.cuda.synchronize()
    ms = reduce(e0.elapsed_time(e1) / args.ch_steps, dist.ReduceOp.MAX)
    mode = st.mode
    del st
    torch.cuda.empty_cache()
    return {"steps_s": 1e3 / ms, "ms_per_step": ms, "n": n, "n_gpus": world, "timed_steps": args.ch_steps,
            "mode": mode, "graphs": world == 1,
            "path": "DistCHStepper: y-slabs; RHS + x-sweep, y-sweep, combine per step; the all-to-alls and "
                    "halo rows are stored into the peers' buffers by the sweeps / combine (P2P)"
                    if mode == "p2p" else "DistCHStepper NCCL form (halo + 2 all_to_all_single per step)"}


def spawn_ranks(args) -> int:
    """`--gpus N` outside torchrun: re-launch this script under
    torch.distributed.run with N ranks on 127.0.0.1 (rank 0 prints)."""
    import socket
    with socket.socket() as sck:
        sck.bind(("127.0.0.1", 0))
        port = sck.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=500)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--nx", type=int, default=NX, help="grid edge (default: the config's 32768; tests use less)")
    ap.add_argument("--ch-n", type=int, default=8192, help="config 5 grid edge for the multi-GPU CH line")
    ap.add_argument("--ch-steps", type=int, default=40)
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-extra", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--skip-ch", action="store_true")
    ap.add_argument("--slab", action="store_true",
                    help="use the multi-GPU y-slab path even at N=1 (world of one)")
    ap.add_argument("--halo", choices=["p2p", "nccl"], default="p2p",
                    help="multi-GPU halo exchange: p2p = fused into the stencil kernel (the boundary rows are "
                         "stored into the neighbours' buffers over NVLink, CUDA IPC), falling back to nccl "
                         "(torch.distributed P2P overlapped with the interior rows) if peer mapping fails")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    ours_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
