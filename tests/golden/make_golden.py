"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs the unmodified reference library (oracle/_ref/libstengrid_ref.so, built
from /root/reference by oracle/Makefile) on seeded inputs and stores inputs
and outputs. Small cases are stored in full (.npz); large ones as a sha256 of
the output bytes plus sampled values. Re-run with:

    make -C oracle && python tests/golden/make_golden.py

The committed fixtures pin both the C restatement (tests/test_oracle.py) and
the GPU path (tests/test_golden_gpu.py) without needing /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle.oracle import FN_IDS, Reference, ch_params  # noqa: E402

TWO_PI = 2.0 * math.pi


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def samples(a, k=64, seed=0):
    rng = np.random.default_rng(seed)
    ny, nx = a.shape
    js = rng.integers(0, ny, k)
    iss = rng.integers(0, nx, k)
    return [[int(j), int(i), float(a[j, i]).hex()] for j, i in zip(js, iss)]


def splitmix_field(nx, ny, seed, amp):
    """initial_condition (cahn_hilliard.cpp:68-76) through the reference."""
    ref = Reference()
    p = ch_params(nx, ny, seed=seed, amp=amp)
    return ref.ch_initial_condition(p)


def stencil_cases(ref):
    rng = np.random.default_rng(2024)
    cases = {}
    k = 0
    fn_list = [("weights", None), ("ch_nonlinear_window", (1, 1, 1, 1, 9)),
               ("fn_weighted_3x3", (1, 1, 1, 1, 9)), ("fn_center", (1, 1, 1, 1, 0)),
               ("fn_lap_cube_diff_first", (1, 1, 1, 1, 2)), ("fn_central_second", (1, 1, 0, 0, 1)),
               ("central_difference_window", (1, 1, 0, 0, 1))]
    for trial in range(48):
        fn, spec = fn_list[trial % len(fn_list)]
        nx, ny = (int(v) for v in rng.integers(1, 70, 2))
        if spec is None:
            d = int(rng.integers(0, 3))
            e = [0, 0, 0, 0]
            if d != 1:
                e[0], e[1] = (int(v) for v in rng.integers(0, min(3, nx - 1) + 1, 2))
            if d != 0:
                e[2], e[3] = (int(v) for v in rng.integers(0, min(3, ny - 1) + 1, 2))
            w = rng.uniform(-2, 2, (e[0] + e[1] + 1) * (e[2] + e[3] + 1))
        else:
            e = list(spec[:4])
            nx, ny = max(nx, 3), max(ny, 3)
            d = 0 if e[2] == 0 else 2
            w = rng.uniform(-2, 2, max(spec[4], 1))[:spec[4]]
        periodic = bool(trial % 3 != 2)
        inp = rng.uniform(-1.5, 1.5, (ny, nx))
        out0 = np.full((ny, nx), -12345.678)
        out = ref.stencil(inp, e, w, direction=d, periodic=periodic, fn=fn, out=out0)
        cases[f"c{k}_in"] = inp
        cases[f"c{k}_w"] = np.asarray(w, dtype=np.float64)
        cases[f"c{k}_meta"] = np.array([d, int(periodic), FN_IDS[fn], *e], dtype=np.int64)
        cases[f"c{k}_out"] = out
        k += 1
    cases["count"] = np.array([k])
    np.savez_compressed(HERE / "stencil_cases.npz", **cases)


def config1(ref):
    """BASELINE config 1: 512^2 XY periodic 5-point Laplacian (the 3x3
    nonlinear_laplacian_coefficients weights), 10 applications (compute +
    swap), input = SplitMix64 seed 1 amplitude 1."""
    n = 512
    inp = splitmix_field(n, n, 1, 1.0)
    dx = TWO_PI / n
    _, nl = ref.ch_weights(dx, dx)
    out = ref.stencil(inp, (1, 1, 1, 1), nl, direction=2, periodic=True, applications=10)
    return {"nx": n, "ny": n, "seed": 1, "amp": 1.0, "weights_hex": [float(x).hex() for x in nl],
            "applications": 10, "sha256": sha(out), "samples": samples(out),
            "input_sha256": sha(inp)}


def config2_small(ref):
    """Config 2 kernel at a small size: batched 1D non-periodic 4th
    x-derivative {1,-4,6,-4,1}/dx^4, 256 points x 64 batches, seed 2."""
    nx, ny = 256, 64
    inp = splitmix_field(nx, ny, 2, 1.0)
    dx = TWO_PI / nx
    s = 1.0 / (dx ** 4)
    w = np.array([s, -4 * s, 6 * s, -4 * s, s])
    out0 = np.full((ny, nx), -12345.678)
    out = ref.stencil(inp, (2, 2, 0, 0), w, direction=0, periodic=False, out=out0)
    np.savez_compressed(HERE / "config2_small.npz", inp=inp, w=w, out=out)


def penta_cases(ref):
    rng = np.random.default_rng(7)
    d = {}
    k = 0
    for periodic in (0, 1):
        for B, n in [(1, 5), (3, 9), (17, 32), (64, 7)]:
            bands = [rng.uniform(-1, 1, (n, B)) for _ in range(5)]
            bands[2] = bands[2] + 6.0
            rhs = rng.uniform(-1, 1, (n, B))
            x = ref.penta_solve(periodic, bands, rhs, workers=2)
            d[f"p{k}_meta"] = np.array([periodic, B, n])
            for name, b in zip(("e", "c", "d", "a", "b"), bands):
                d[f"p{k}_{name}"] = b
            d[f"p{k}_rhs"] = rhs
            d[f"p{k}_x"] = x
            k += 1
    d["count"] = np.array([k])
    np.savez_compressed(HERE / "penta_cases.npz", **d)


def ch_cases(ref):
    out = {}
    # full arrays at 32 x 16, 10 steps
    p = ch_params(32, 16, seed=5)
    c, pr = ref.ch_run(p, 10)
    np.savez_compressed(HERE / "ch_32x16_10steps.npz", curr=c, prev=pr,
                        params=np.array([p["D"], p["gamma"], p["lx"], p["ly"], p["dt"]]))
    # hashes at 64^2 (20 steps) and 128^2 (5 steps, nonlinear off)
    for n, steps, nl in [(64, 20, True), (128, 5, False)]:
        p = ch_params(n, seed=1, nonlinear=nl)
        c, pr = ref.ch_run(p, steps)
        out[f"ch_{n}_{steps}_{'nl' if nl else 'linear'}"] = {
            "nx": n, "ny": n, "steps": steps, "nonlinear": nl, "seed": 1, "dt_hex": float(p["dt"]).hex(),
            "curr_sha256": sha(c), "prev_sha256": sha(pr), "samples": samples(c)}
    return out


def kats(ref):
    out = {}
    for n in (64, 1024, 8192):
        dx = TWO_PI / n
        bw, nl = ref.ch_weights(dx, dx)
        out[f"biharmonic_weights_{n}"] = [float(x).hex() for x in bw]
        out[f"nonlinear_coefficients_{n}"] = [float(x).hex() for x in nl]
    out["wrap"] = [[i, n, ref.wrap(i, n)] for i, n in [(-1, 8), (8, 8), (-17, 8), (5, 3), (-6, 3), (0, 1)]]
    out["make_tiles"] = {f"{ny}_{t}": ref.make_tiles(ny, t) for ny, t in [(10, 3), (512, 4), (7, 7), (13, 5)]}
    return out


def main():
    ref = Reference()
    stencil_cases(ref)
    config2_small(ref)
    penta_cases(ref)
    meta = {"generator": "tests/golden/make_golden.py", "source": "oracle/_ref (unmodified reference)",
            "config1": config1(ref), "ch": ch_cases(ref), "kats": kats(ref)}
    (HERE / "golden.json").write_text(json.dumps(meta, indent=1))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
