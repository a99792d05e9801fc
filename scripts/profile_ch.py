"""Run CH steps (for ncu launch lists).
python scripts/profile_ch.py [--n 1024] [--steps 20] [--partition P]"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1902_09931_b200 as sg

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--ny", type=int, default=0, help="rows (default: n)")
ap.add_argument("--steps", type=int, default=20)
ap.add_argument("--partition", type=int, default=0)
a = ap.parse_args()
p = sg.CHParams(nx=a.n, ny=a.ny or a.n)
p.dt = 0.1 * p.dx()
p.T = 1.0
st = sg.CHStepper(p)
if a.partition:
    st.set_partition(a.partition)
st.step_many(a.steps)
st.synchronize()
print("done", st.step_index())
