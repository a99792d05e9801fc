"""The C++ WorkerPool (include/stengrid/worker_pool.hpp) is a real host
thread pool with the reference's semantics: compiled with g++ and run here
(no GPU)."""
import subprocess
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_worker_pool_cxx(tmp_path):
    exe = tmp_path / "test_worker_pool"
    subprocess.run(["g++", "-std=c++20", "-O2", "-pthread", "-I", str(ROOT / "include"),
                    str(ROOT / "tests" / "cxx" / "test_worker_pool.cpp"), "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "worker pool OK" in r.stdout
