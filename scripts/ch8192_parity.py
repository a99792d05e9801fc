"""Config 5 parity at its full geometry: 8192^2, CHParams defaults, 100
steps — the one-GPU CHStepper and the distributed step (G = 8 simulated
ranks, P2P and NCCL forms) against the UNMODIFIED reference CHStepper's
digest (tests/golden/ch8192_100steps.json, made by
tests/golden/make_ch8192_golden.py from oracle/_ref on 8 cores).

    python scripts/ch8192_parity.py > profiles/r02_ch8192_100steps_parity.json

North-star bar: rel-L2 <= 1e-9 after 100 steps. Reported: sha256 equality
of both time levels, rel-L2 over the golden's sample rows, the relative
difference of the field norms, and the GPU wall time of the 100 steps."""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def compare(c, p, g):
    rows = {r: np.frombuffer(bytes.fromhex(h), dtype="<f8") for r, h in g["rows_curr"].items()}
    num = sum(float(np.sum((c[int(r)] - w) ** 2)) for r, w in rows.items())
    den = sum(float(np.sum(w ** 2)) for w in rows.values())
    return {"sha256_curr_equal": sha(c) == g["sha256_curr"], "sha256_prev_equal": sha(p) == g["sha256_prev"],
            "rel_l2_sample_rows": (num / den) ** 0.5, "sample_rows": sorted(int(r) for r in rows),
            "rel_norm_diff_curr": abs(float(np.linalg.norm(c)) - g["l2_curr"]) / g["l2_curr"],
            "rel_norm_diff_prev": abs(float(np.linalg.norm(p)) - g["l2_prev"]) / g["l2_prev"]}


def main():
    import torch

    import paper_1902_09931_b200 as sg
    from paper_1902_09931_b200.ch_dist import DistCHStepper, LocalTransport
    gold = json.loads((ROOT / "tests" / "golden" / "ch8192_100steps.json").read_text())
    g = gold["steps_100"]
    out = {"config": "BASELINE config 5 grid: CH BDF2-ADI periodic FP64 8192x8192, CHParams defaults, 100 steps",
           "reference": gold["generator"] + f", {gold['workers']} workers, {gold['seconds']:.0f} s",
           "tolerance": "north star: rel-L2 <= 1e-9"}
    p = sg.CHParams(nx=8192, ny=8192)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    st = sg.CHStepper(p)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.step_many(100)
    st.synchronize()
    secs = time.perf_counter() - t0
    c, pr = st.field().values, st.previous_field().values
    out["single_gpu"] = dict(compare(c, pr, g), seconds_100_steps=secs)
    del st
    for mode in ("p2p", "nccl"):
        ranks = []
        tr = LocalTransport(ranks)
        for r in range(8):
            ranks.append(DistCHStepper(p, 8, r, transport=tr, mode=mode))
        for _ in range(100):
            for s in ranks:
                s.phase_x()
            for s in ranks:
                s.phase_y()
            for s in ranks:
                s.phase_combine()
        torch.cuda.synchronize()
        dc = np.concatenate([s.own_rows(0).cpu().numpy() for s in ranks])
        dp = np.concatenate([s.own_rows(1).cpu().numpy() for s in ranks])
        out[f"distributed_g8_{mode}"] = dict(compare(dc, dp, g), mode=ranks[0].mode,
                                             bitwise_vs_single_gpu=bool(np.array_equal(dc.view(np.uint64),
                                                                                       c.view(np.uint64))))
        del ranks, tr
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
