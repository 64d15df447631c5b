"""frames.ptya streamed from disk to the device (PDD_DATA_PTYA_FRAMES_F64,
csrc/ptya.cpp) and the CLI front end (paper_2011_00162_b200/cli.py) on the GPU.

* A solver built from a PTYA path is bit-identical to one built from the same
  intensities in memory (the streamed chunks are converted by the same
  sqrt(f) -> amplitude arithmetic), on stripes, grids and multi-rank handles,
  in float32 and float64.
* Malformed files fail like the reference's read_frames + FrameStack::validate
  (io.cpp:186-202, scan.cpp:46-56): FormatError for the container, invalid
  argument for counts, shapes and negative intensities.
* The CLI reconstructs a dataset directory written by the reference's own I/O
  (oracle/_ref, io.cpp) and writes run outputs the reference's reader accepts,
  equal to the Python API's result; exit codes follow ptychodd_cli.cpp:26-30.
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import ref_lib as R
import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import ptya, sim

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def problem(N=160, s=32, step=8, seed=9):
    probe = sim.make_probe(s, s / 4)
    obj = sim.make_object(N, 4.0, seed, seed + 1)
    g = P.make_raster_scan(N, N, s, step)
    f = sim.poisson_host(P.intensity(P.forward(probe, obj, g, dtype="f64"), dtype="f64"), 1e4, seed + 2)
    return g, probe, f


def states_equal(a, b):
    for x, y in zip(a.u + a.gamma + a.v, b.u + b.gamma + b.v):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("grid,devices", [(None, None), ((2, 2), None), ((2, 2), [0, 0])])
def test_streamed_ptya_equals_in_memory_frames(tmp_path, dtype, grid, devices):
    g, probe, f = problem()
    path = str(tmp_path / "frames.ptya")
    ptya.write_frames(path, f)
    plan = P.plan_grid(g, *grid) if grid else P.plan_stripes(g, 3)
    a = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype=dtype, devices=devices)
    b = P.NonblindSolver(plan, path, probe, P.NonblindConfig(), dtype=dtype, devices=devices)
    sa, sb = a.init_state(), b.init_state()
    aa, ab = [z.copy() for z in sa.z], [z.copy() for z in sb.z]
    for _ in range(2):
        a.step(sa, aa)
        b.step(sb, ab)
        states_equal(sa, sb)
    cfg = P.NonblindConfig(max_iters=5, tol_rf=1e-300)
    ra = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype).run()
    rb = P.NonblindSolver(plan, path, probe, cfg, dtype=dtype).run()
    assert [r.rf for r in ra.records] == [r.rf for r in rb.records]
    assert np.array_equal(ra.merged, rb.merged)


def test_streamed_ptya_large_frames_many_chunks(tmp_path):
    """128^2 frames over more than one 32 MB chunk and a full ring turnover."""
    N, s, step = 2048, 128, 32
    probe = sim.make_probe(s, 32.0)
    obj = sim.make_object(N, 8.0, 4, 5)
    g = P.make_raster_scan(N, N, s, step)
    f = P.intensity(P.forward(probe, obj, g, dtype="f32"), dtype="f64")
    assert f.nbytes > 7 * (32 << 20)
    path = str(tmp_path / "frames.ptya")
    ptya.write_frames(path, f)
    plan = P.plan_stripes(g, 4, "rows")
    cfg = P.NonblindConfig(max_iters=3, tol_rf=1e-300)
    ra = P.NonblindSolver(plan, f, probe, cfg, dtype="f32").run()
    rb = P.NonblindSolver(plan, path, probe, cfg, dtype="f32").run()
    assert [r.rf for r in ra.records] == [r.rf for r in rb.records]
    assert np.array_equal(ra.merged, rb.merged)


def test_blind_from_ptya(tmp_path):
    g, _, f = problem()
    path = str(tmp_path / "frames.ptya")
    ptya.write_frames(path, f)
    plan = P.plan_stripes(g, 2)
    cfg = P.BlindConfig(max_iters=4, tol_rf=1e-300, r=1e3)
    ra = P.BlindSolver(plan, f, cfg, dtype="f32").run()
    rb = P.BlindSolver(plan, path, cfg, dtype="f32").run()
    assert [r.rf for r in ra.records] == [r.rf for r in rb.records]
    assert np.array_equal(ra.probe, rb.probe)


def test_malformed_ptya_inputs(tmp_path):
    g, probe, f = problem(N=96)
    plan = P.plan_stripes(g, 2)
    ok = str(tmp_path / "ok.ptya")
    ptya.write_frames(ok, f)
    b = open(ok, "rb").read()
    (tmp_path / "short.ptya").write_bytes(b[:-8])
    (tmp_path / "long.ptya").write_bytes(b + b"x")
    (tmp_path / "magic.ptya").write_bytes(b"XXXX" + b[4:])
    for name in ("short", "long", "magic"):
        with pytest.raises(P.FormatError):
            P.NonblindSolver(plan, str(tmp_path / f"{name}.ptya"), probe, P.NonblindConfig())
    ptya.write_frames(str(tmp_path / "count.ptya"), f[:-1])
    with pytest.raises(P.InvalidArgument):  # FrameStack: frame count != scan position count
        P.NonblindSolver(plan, str(tmp_path / "count.ptya"), probe, P.NonblindConfig())
    neg = f.copy()
    neg[3, 2, 1] = -1.0
    ptya.write_frames(str(tmp_path / "neg.ptya"), neg)
    with pytest.raises(P.InvalidArgument):  # FrameStack: negative intensity
        P.NonblindSolver(plan, str(tmp_path / "neg.ptya"), probe, P.NonblindConfig())
    with pytest.raises(Exception):
        P.NonblindSolver(plan, str(tmp_path / "missing.ptya"), probe, P.NonblindConfig())


def cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_2011_00162_b200.cli", *args], capture_output=True, text=True,
                          cwd=ROOT, timeout=600)


@pytest.mark.skipif(not R.has_io(), reason="oracle/_ref without the reference's io.cpp")
def test_cli_on_a_reference_written_dataset(tmp_path):
    N, s, step = 64, 16, 4
    sample, probe, pin = R.toy(N, s, step, 7)
    f = R.simulate_frames(probe, sample, step)
    ds = tmp_path / "ds"
    R.write_dataset(ds, N, N, s, step, f, probe, pin=pin, sample=sample)
    out = tmp_path / "run"
    r = cli("reconstruct", "--dataset", str(ds), "--out", str(out), "--subdomains", "2", "--max-iters", "60",
            "--tol-rf", "1e-300", "--backend", "cuda")
    assert r.returncode == 0, r.stdout + r.stderr
    assert "iter 25" in r.stdout and "iter 50" in r.stdout  # progress every 25 iterations
    merged = R.read_array(out / "merged.ptya", "complex")  # the reference's reader accepts our writer
    g = P.make_raster_scan(N, N, s, step)
    api = P.NonblindSolver(P.plan_stripes(g, 2), f, probe, P.NonblindConfig(max_iters=60, tol_rf=1e-300), pin,
                           dtype="f64").run()
    assert np.array_equal(merged, api.merged)
    for d in range(2):
        assert np.array_equal(R.read_array(out / f"sub_{d}.ptya", "complex"), api.sub_solutions[d])
    summ = json.load(open(out / "summary.json"))
    assert summ["iterations"] == 60 and summ["solver"] == "nonblind" and summ["D"] == 2
    rows = open(out / "convergence.csv").read().strip().splitlines()
    assert rows[0] == "iter,rf,re,lagrangian,t_sub_0_ms,t_sub_1_ms,t_virtual_ms,t_actual_ms" and len(rows) == 61
    assert float(rows[-1].split(",")[1]) == api.final_rf
    # blind on the same dataset
    rb = cli("blind", "--dataset", str(ds), "--out", str(tmp_path / "brun"), "--max-iters", "10", "--quiet")
    assert rb.returncode == 0, rb.stderr
    for name in ("probe_recovered", "probe_fourier"):
        assert R.read_array(tmp_path / "brun" / f"{name}.ptya", "complex").shape == (s, s)
    assert R.read_array(tmp_path / "brun" / "support_mask.ptya", "real").shape == (s, s)
    # evaluate: SNR against the dataset's ground truth, PNG rendering
    re_ = cli("evaluate", "--dataset", str(ds), "--run", str(out))
    assert re_.returncode == 0 and "SNR" in re_.stdout
    assert open(out / "magnitude.png", "rb").read(8) == b"\x89PNG\r\n\x1a\n"
    # exit codes: infeasible plan 4, format 3, config 2
    assert cli("reconstruct", "--dataset", str(ds), "--out", str(tmp_path / "x"), "--subdomains", "99").returncode == 4
    (ds / "frames.ptya").write_bytes(open(ds / "frames.ptya", "rb").read()[:-1])
    assert cli("reconstruct", "--dataset", str(ds), "--out", str(tmp_path / "y")).returncode == 3
    assert cli("reconstruct", "--dataset", str(ds), "--out", str(tmp_path / "z"), "--stop", "bogus").returncode == 2
