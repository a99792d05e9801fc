"""The C++ drop-in headers compile in both storage modes (no GPU needed):
the built-in dense containers, and Eigen types (grid.hpp: `Array2d` is
Eigen::Array<double, Dynamic, Dynamic, RowMajor> when <Eigen/Core> is
available, as in the reference, /root/reference/proj/include/stengrid/
grid.hpp:13). This image has no Eigen, so the Eigen mode is checked against
the storage-subset stand-in under oracle/eigen_shim (test infrastructure)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SRC = ROOT / "tests" / "cxx" / "test_stengrid_cxx.cpp"


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
@pytest.mark.parametrize("mode", ["builtin", "eigen"])
def test_reference_style_suite_compiles(mode):
    extra = ["-DSTENGRID_NO_EIGEN"] if mode == "builtin" else \
        ["-DSTENGRID_USE_EIGEN", f"-I{ROOT / 'oracle' / 'eigen_shim'}"]
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", *extra, f"-I{ROOT / 'include'}", str(SRC)],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]


@pytest.mark.skipif(shutil.which("g++") is None, reason="g++ not available")
def test_eigen_mode_uses_eigen_types(tmp_path):
    src = tmp_path / "t.cpp"
    src.write_text(
        "#include <type_traits>\n#include \"stengrid/grid.hpp\"\n#include \"stengrid/penta.hpp\"\n"
        "static_assert(std::is_same_v<stengrid::Array2d,"
        " Eigen::Array<double, Eigen::Dynamic, Eigen::Dynamic, Eigen::RowMajor>>);\n"
        "static_assert(std::is_same_v<decltype(stengrid::Grid2D{}.values), stengrid::Array2d>);\n"
        "int main() { stengrid::Grid2D g(4, 3, 1.0, 1.0); g(1, 2) = 5.0;"
        " return g.values(2, 1) == 5.0 && g.values.rows() == 3 ? 0 : 1; }\n")
    exe = tmp_path / "t"
    r = subprocess.run(["g++", "-std=c++20", "-DSTENGRID_USE_EIGEN", f"-I{ROOT / 'oracle' / 'eigen_shim'}",
                        f"-I{ROOT / 'include'}", str(src), "-o", str(exe)], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    assert subprocess.run([str(exe)]).returncode == 0
