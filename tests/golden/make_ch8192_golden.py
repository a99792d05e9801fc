"""Golden digest of BASELINE config 5's CH run at its full geometry
(8192^2, 100 steps) from the UNMODIFIED reference CHStepper (oracle/_ref,
cahn_hilliard.cpp:260-328), generated once in the build container (≈30 min
on 8 cores) because the fields (2 x 512 MiB) cannot be committed.

Writes tests/golden/ch8192_100steps.json:
  * sha256 of both time levels (C^n, C^{n-1}) as little-endian float64 bytes,
  * their L2 norms (so a non-bitwise result can still be graded in rel-L2),
  * rows 0, 4095 and 8191 of C^n and row 4095 of C^{n-1} in hex (so a
    mismatch can be localised and its relative error bounded),
and the same digests after 3 steps (the existing short parity test).

    python tests/golden/make_ch8192_golden.py [--workers 8] [--steps 100]
"""
from __future__ import annotations

import argparse
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle.oracle import Reference, ch_params  # noqa: E402

SAMPLE_ROWS_C = (0, 4095, 8191)
SAMPLE_ROWS_P = (4095,)


def digest(c: np.ndarray, p: np.ndarray) -> dict:
    return {
        "sha256_curr": hashlib.sha256(np.ascontiguousarray(c, dtype="<f8").tobytes()).hexdigest(),
        "sha256_prev": hashlib.sha256(np.ascontiguousarray(p, dtype="<f8").tobytes()).hexdigest(),
        "l2_curr": float(np.sqrt(np.sum(c * c))),
        "l2_prev": float(np.sqrt(np.sum(p * p))),
        "rows_curr": {str(r): c[r].astype("<f8").tobytes().hex() for r in SAMPLE_ROWS_C},
        "rows_prev": {str(r): p[r].astype("<f8").tobytes().hex() for r in SAMPLE_ROWS_P},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=8)
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    n = 8192
    p = ch_params(n)
    ref = Reference()
    out = {"n": n, "params": {k: v for k, v in p.items()}, "workers": a.workers,
           "generator": "oracle/_ref CHStepper (unmodified reference, -O3 -ffp-contract=off)"}
    t0 = time.time()
    c, pr = ref.ch_run(p, 3, tiles=a.workers, workers=a.workers)
    out["steps_3"] = digest(c, pr)
    print(f"3 steps: {time.time() - t0:.1f} s", flush=True)
    c, pr = ref.ch_run(p, a.steps - 3, curr=c, prev=pr, tiles=a.workers, workers=a.workers)
    out[f"steps_{a.steps}"] = digest(c, pr)
    out["seconds"] = time.time() - t0
    print(f"{a.steps} steps: {out['seconds']:.1f} s", flush=True)
    (Path(__file__).parent / "ch8192_100steps.json").write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
