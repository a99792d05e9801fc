"""Build an A/B variant of the library with extra nvcc defines into
exp_libs/<name>.so (objects under build/obj_<name>); select it at run time
with SG_LIB_PATH=exp_libs/<name>.so. Only the stencil translation units are
rebuilt with the defines; the rest reuse build/obj.

    python scripts/exp/build_variant.py novote -DSG_STORE_VOTE=0
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1902_09931_b200 import build as b  # noqa: E402

name, defs = sys.argv[1], sys.argv[2:]
b.build(verbose=False)  # the default objects are current
root = b.ROOT
b.OBJ = root / "build" / f"obj_{name}"
b.OBJ.mkdir(parents=True, exist_ok=True)
b.FLAGS = b.FLAGS + defs
(root / "exp_libs").mkdir(exist_ok=True)
b.LIB = root / "exp_libs" / f"{name}.so"
base = root / "build" / "obj"
for src in b._sources():
    if not src.stem.startswith("stencil"):
        tgt = b.OBJ / (src.stem + ".o")
        tgt.write_bytes((base / (src.stem + ".o")).read_bytes())
b.build(force=False, verbose=True)
