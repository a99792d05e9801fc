"""The penta sweep's kernel selection knob SG_SWEEP_KERNEL (read once per
process, so each variant runs in a subprocess): "reg" forces the
register-prefetch k_sweep (the path odd batches and unaligned rhs take
anyway) for uniform and per-system tables alike; unset, uniform operators
run the resident-turn k_sweep_res and per-system tables the streaming TMA
k_sweep_tma. Every variant must stay bitwise to the oracle on the uniform
(CH operator) and general per-system batches, periodic and not, including
n not a multiple of the 32-row stage."""
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]

SCRIPT = r"""
import sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1902_09931_b200 as sg
from oracle.oracle import Restatement
orc = Restatement()
bad = []
for periodic in (False, True):
    for B, n, uniform in ((256, 96, True), (64, 40, False), (2048, 33, True), (128, 33, False)):
        if uniform:
            m = sg.build_hyperdiffusion_operator(2.5, n, B, periodic)
        else:
            rng = np.random.default_rng(B + n)
            m = sg.PentaBatch(B, n, periodic)
            for band in m.bands():
                band[:] = rng.uniform(-1, 1, (n, B))
            m.diag += 6.0
        rhs = np.random.default_rng(n).uniform(-1, 1, (n, B))
        f = sg.PeriodicPentaFactor(m) if periodic else sg.PentaFactor(m)
        t = torch.from_numpy(rhs.copy()).cuda()
        f.solve_in_place(t)
        want = orc.penta_solve(periodic, m.bands(), rhs)
        if not np.array_equal(t.cpu().numpy().view(np.uint64), want.view(np.uint64)):
            bad.append((periodic, B, n, uniform))
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("variant", ["reg", "default"])
def test_sweep_variant_bitwise(variant):
    env = dict(os.environ, SG_SWEEP_KERNEL=variant)
    r = subprocess.run([sys.executable, "-c", SCRIPT, str(ROOT)], env=env, cwd=ROOT, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
