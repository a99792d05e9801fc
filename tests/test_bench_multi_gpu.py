"""bench.py --gpus N on a box with fewer GPUs than N: bench.py re-launches
itself under torch.distributed.run with N ranks (the ranks share the device,
so the process group is gloo and the halos go through CUDA IPC), and rank 0
prints ONE line with n_gpus == N, the weak-scaling headline, the strong
scaling figure, the e2e figure and config 5's distributed CH line. Small
sizes: this checks the wiring, not the numbers."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3])
def test_bench_gpus_n_runs_n_ranks(n):
    cmd = [sys.executable, "bench.py", "--gpus", str(n), "--nx", "2048", "--steps", "20", "--warmup", "3",
           "--ch-n", "256", "--ch-steps", "4", "--e2e-steps", "2", "--skip-cpu"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["ny"] == 2048 * n
    assert d["strong"]["value"] > 0 and "split into" in d["strong"]["workload"]
    assert d["e2e"]["value"] > 0 and d["e2e"]["d2h_bytes_per_step"] == 2048 * 2048 * 8
    assert d["e2e"]["h2d_bytes_per_step"] == (2048 + 2 * n) * 2048 * 8
    ch = d["extra"]["cfg5_ch_8192sq_dist"]
    assert ch["n_gpus"] == n
    if 256 % n == 0:
        assert ch["mode"] == "p2p" and ch["steps_s"] > 0
    else:
        assert "skipped" in ch
    assert d["gpu_launches"] >= n * 20
    assert "p2p" in d["config"]["parallelism"].lower() or "P2P" in d["config"]["parallelism"]


@pytest.mark.gpu
def test_bench_rejects_world_mismatch():
    env = dict(__import__("os").environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--nx", "1024", "--steps", "3"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode != 0 and "WORLD_SIZE" in (r.stderr + r.stdout)
