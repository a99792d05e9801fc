"""CPU checks of the C-ABI library: it loads without a GPU and exports every
symbol include/stengrid/sg.h declares; entry points that need no device
behave like the reference (wrap, make_tiles, error classes). No compute call
is made here."""
import ctypes as C
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "stengrid" / "sg.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1902_09931_b200 import _lib
    L = _lib.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    assert set(declared_symbols()) == set(_lib.EXPORTED)
    assert L.sg_abi_version() == 1


def test_wrap_and_make_tiles_kats():
    """test_grid.cpp:13-125 known answers, through the C ABI."""
    import paper_1902_09931_b200 as sg
    assert sg.wrap(-1, 8) == 7
    assert sg.wrap(8, 8) == 0
    assert sg.wrap(-17, 8) == 7
    with pytest.raises(sg.InvalidArgument):
        sg.wrap(3, 0)
    assert sg.make_tiles(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert sg.make_tiles(512, 4) == [(0, 128), (128, 256), (256, 384), (384, 512)]
    for ny in range(1, 65):
        for t in range(1, ny + 1):
            tiles = sg.make_tiles(ny, t)
            assert tiles[0][0] == 0 and tiles[-1][1] == ny
            assert all(a[1] == b[0] for a, b in zip(tiles, tiles[1:]))
            sizes = [e - b for b, e in tiles]
            assert max(sizes) - min(sizes) <= 1 and sizes == sorted(sizes, reverse=True)
    with pytest.raises(sg.InvalidArgument):
        sg.make_tiles(4, 5)
    with pytest.raises(sg.InvalidArgument):
        sg.make_tiles(4, 0)


def test_validation_errors_precede_device_checks():
    """create_plan validation (stencil.cpp:128-161) raises InvalidArgument even
    without a GPU; a valid plan without a GPU raises NoDeviceError (no CPU
    fallback)."""
    import numpy as np
    import paper_1902_09931_b200 as sg
    a, b = sg.Grid2D(16, 8), sg.Grid2D(16, 8)
    with pytest.raises(sg.InvalidArgument):
        sg.create_plan(sg.Direction.X, sg.BoundaryMode.Periodic,
                       sg.WeightStencil(sg.Extents(1, 1, 1, 0), [1.0] * 6), a, b, 1, 1)
    with pytest.raises(sg.InvalidArgument):
        sg.create_plan(sg.Direction.X, sg.BoundaryMode.Periodic,
                       sg.FunctionStencil(sg.Extents(1, 1), "no_such_function", []), a, b, 1, 1)
    import torch
    if not torch.cuda.is_available():
        with pytest.raises(sg.NoDeviceError):
            sg.create_plan(sg.Direction.X, sg.BoundaryMode.Periodic,
                           sg.WeightStencil(sg.Extents(1, 1), [1.0, -2.0, 1.0]), a, b, 1, 1)


def test_plain_c_client_compiles_links_and_fails_loudly_without_gpu(tmp_path):
    """The C ABI is usable from C99 (INTEGRATION.md's example): it compiles
    with gcc against include/stengrid/sg.h, links libstengrid_b200.so, and on
    a machine without a GPU reports SG_ERR_NO_DEVICE instead of computing on
    the CPU."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    import torch
    if torch.cuda.is_available():
        pytest.skip("CPU-only check")
    src = tmp_path / "client.c"
    src.write_text(r'''
#include "stengrid/sg.h"
#include <stdio.h>
int main(void) {
  enum { nx = 64, ny = 32 };
  static double in_host[nx * ny], out_host[nx * ny];
  sg_plan_t plan;
  sg_extents e = {1, 1, 1, 1};
  double coe[9] = {0, 1, 0, 1, -4, 1, 0, 1, 0};
  sg_status st = sg_plan_create(SG_DIR_XY, SG_PERIODIC, e, SG_FN_WEIGHTED_3X3, coe, 9, SG_F64, in_host,
                                out_host, nx, ny, SG_MEM_HOST, 1, 1, &plan);
  printf("%d %s\n", (int)st, st == SG_OK ? "" : sg_last_error());
  return st == SG_ERR_NO_DEVICE ? 0 : 1;
}
''')
    lib = ROOT / "paper_1902_09931_b200"
    exe = tmp_path / "client"
    subprocess.run(["gcc", "-std=c99", "-Wall", "-Werror", f"-I{ROOT / 'include'}", str(src), f"-L{lib}",
                    "-lstengrid_b200", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "no CUDA device" in r.stdout
