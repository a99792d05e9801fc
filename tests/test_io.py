"""CSG1 snapshots and diagnostics CSV (test_io.cpp restated): byte-identical
to the reference writer (oracle/_ref), round trips, error cases. CPU only;
the device checkpoint/resume test is test_checkpoint_gpu below (gpu)."""
import math

import numpy as np
import pytest

import paper_1902_09931_b200 as sg


def test_snapshot_bytes_match_reference(ref, tmp_path):
    rng = np.random.default_rng(3)
    v = rng.uniform(-1, 1, (7, 13))
    ours, theirs = tmp_path / "a.csg", tmp_path / "b.csg"
    sg.write_snapshot(sg.Grid2D.from_array(v, 0.1, 0.25), ours)
    ref.write_snapshot(v, 0.1, 0.25, theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    g = sg.read_snapshot(theirs)
    assert (g.nx, g.ny, g.dx, g.dy) == (13, 7, 0.1, 0.25)
    assert np.array_equal(g.values.view(np.uint64), v.view(np.uint64))
    back, dx, dy = ref.read_snapshot(ours)
    assert np.array_equal(back.view(np.uint64), v.view(np.uint64)) and (dx, dy) == (0.1, 0.25)


def test_snapshot_errors(tmp_path):
    p = tmp_path / "bad.csg"
    p.write_bytes(b"XXXX" + bytes(24))
    with pytest.raises(RuntimeError):
        sg.read_snapshot(p)
    g = sg.Grid2D(4, 3, 1.0, 1.0)
    sg.write_snapshot(g, p)
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(RuntimeError):
        sg.read_snapshot(p)


def test_diagnostics_csv_matches_reference(ref, tmp_path):
    rows = [sg.Diagnostics(0.0, 1.0, 0.0), sg.Diagnostics(0.1 / 3, 1.0 + 1e-17, math.pi),
            sg.Diagnostics(12.5, 1.2345678901234567, 0.3333333333333333)]
    ours, theirs = tmp_path / "a.csv", tmp_path / "b.csv"
    sg.write_diagnostics_csv(rows, ours)
    ref.write_diagnostics_csv([[d.t, d.s, d.k1Inv] for d in rows], theirs)
    assert ours.read_bytes() == theirs.read_bytes()
    assert ours.read_text().splitlines()[0] == "t,s,k1_inv"


@pytest.mark.gpu
def test_checkpoint_resume_is_bitwise_exact(sg, tmp_path):
    """BDF2 needs both time levels: save C^n, C^{n-1} and the step; a resumed
    run equals an uninterrupted one bitwise."""
    p = sg.CHParams(nx=64, ny=32)
    p.dt = 0.1 * p.dx()
    p.T = 1.0
    a = sg.CHStepper(p)
    a.step_many(10)
    ck = tmp_path / "ck.bin"
    sg.save_checkpoint(a, ck)
    a.step_many(15)
    b = sg.CHStepper(p)
    sg.load_checkpoint(b, ck)
    assert b.step_index() == 10
    b.step_many(15)
    assert b.step_index() == 25 and b.time() == a.time()
    assert np.array_equal(a.field().values.view(np.uint64), b.field().values.view(np.uint64))
