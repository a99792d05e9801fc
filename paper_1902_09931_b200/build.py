"""Build libstengrid_b200.so (sm_100a) in-tree.

    python -m paper_1902_09931_b200.build [--force]

Every .cu under csrc/ is compiled with
``nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false``
(no FMA contraction: the device analogue of the reference's
``-ffp-contract=off``, so FP64 results are bitwise identical to the
reference CPU code) into build/, in parallel, then linked into
``paper_1902_09931_b200/libstengrid_b200.so`` with the static CUDA runtime.
The .so is git-ignored but travels to the GPU box with gpurun.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
OBJ = ROOT / "build" / "obj"
LIB = PKG / "libstengrid_b200.so"
CXX_TEST_BIN = ROOT / "build" / "test_stengrid_cxx"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-Wall",
         "-I", str(ROOT / "include"), "-I", str(CSRC)]


def _sources():
    return sorted(CSRC.glob("*.cu"))


def _headers():
    return sorted(list(CSRC.glob("*.hpp")) + list(CSRC.glob("*.cuh")) +
                  list((ROOT / "include" / "stengrid").glob("*")))


def _compile(src: Path, force: bool) -> Path:
    obj = OBJ / (src.stem + ".o")
    newest_dep = max([src.stat().st_mtime] + [h.stat().st_mtime for h in _headers()])
    if not force and obj.exists() and obj.stat().st_mtime >= newest_dep:
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", str(src), "-o", str(obj)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"nvcc failed on {src.name}")
    return obj


def build(force: bool = False, verbose: bool = True) -> Path:
    OBJ.mkdir(parents=True, exist_ok=True)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, force), srcs))
    if force or not LIB.exists() or LIB.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "--cudart", "static",
               "-L/usr/local/cuda/lib64", "-lcufft", "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
        subprocess.run(cmd, check=True)
        if verbose:
            print(f"built {LIB}")
    return LIB


def build_cxx_tests(force: bool = False) -> Path:
    """Compile tests/cxx/test_stengrid_cxx.cpp (the reference-style C++ tests
    of the drop-in API) against libstengrid_b200.so."""
    src = ROOT / "tests" / "cxx" / "test_stengrid_cxx.cpp"
    if not src.exists():
        return CXX_TEST_BIN
    CXX_TEST_BIN.parent.mkdir(parents=True, exist_ok=True)
    deps = [src, LIB] + list((ROOT / "include" / "stengrid").glob("*"))
    if not force and CXX_TEST_BIN.exists() and CXX_TEST_BIN.stat().st_mtime >= max(
            d.stat().st_mtime for d in deps):
        return CXX_TEST_BIN
    cmd = ["g++", "-std=c++20", "-O2", "-ffp-contract=off", "-I", str(ROOT / "include"), str(src),
           "-o", str(CXX_TEST_BIN), "-L", str(PKG), "-lstengrid_b200", f"-Wl,-rpath,{PKG}",
           "-pthread"]
    subprocess.run(cmd, check=True)
    return CXX_TEST_BIN


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    build(force=a.force)
    build_cxx_tests(force=a.force)
