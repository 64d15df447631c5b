"""Blind OD²BP parity: GPU BlindSolver vs the oracle (oracle/od2p.py), and the
reference's blind tests (proj/tests/test_blind.cpp) restated on the GPU path."""
import numpy as np
import pytest

from tests.helpers import rel_l2
from oracle import od2p as O
import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import sim

pytestmark = pytest.mark.gpu


def fp32_intensity(f):
    a = np.sqrt(f).astype(np.float32).astype(np.float64)
    return a * a


def blind_problem(N=96, s=32, step=8, D=2, grid=None, peak=None, seed=5):
    probe = sim.make_probe(s, s / 4)
    obj = sim.make_object(N, 3.0, seed + 1, seed + 2)
    g = O.make_raster_scan(N, N, s, step)
    f = O.intensity(O.forward(probe, obj, g))
    if peak:
        f = sim.poisson_host(f, peak, seed + 3)
    gp = P.make_raster_scan(N, N, s, step)
    if grid:
        return f, O.plan_grid(g, *grid), P.plan_grid(gp, *grid)
    return f, O.plan_stripes(g, D), P.plan_stripes(gp, D)


def compare(st, ost, tol):
    assert rel_l2(st.w, ost.w) < tol, "w"
    for a, b in zip(st.w_copies, ost.w_copies):
        assert rel_l2(a, b) < tol, "w_copies"
    for a, b in zip(st.delta, ost.delta):
        assert np.linalg.norm(a - b) / np.linalg.norm(ost.w) < tol, "delta"
    for a, b in zip(st.u, ost.u):
        assert rel_l2(a, b) < tol, "u"
    for a, b in zip(st.gamma, ost.gamma):
        assert rel_l2(a, b) < tol, "gamma"
    for a, b in zip(st.v, ost.v):
        assert rel_l2(a, b) < tol, "v"
    for (a0, a1), (b0, b1), v in zip(st.lam, ost.lam, ost.v):
        assert np.linalg.norm(a0 - b0) / np.linalg.norm(v) < tol, "lambda0"
        assert np.linalg.norm(a1 - b1) / np.linalg.norm(v) < tol, "lambda1"


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-5)])
@pytest.mark.parametrize("D,grid", [(2, None), (None, (2, 2))])
def test_blind_setup_and_steps_match_oracle(dtype, tol, D, grid):
    f, oplan, plan = blind_problem(D=D or 1, grid=grid)
    if dtype == "f32":
        f = fp32_intensity(f)
    cfg = dict(r=1e3)
    gs = P.BlindSolver(plan, f, P.BlindConfig(**cfg), dtype=dtype)
    osol = O.BlindSolver(oplan, f, O.BlindConfig(**cfg))
    # amplitude-based initial probe and estimated support (blind.cpp:123-156)
    assert rel_l2(gs.initial_probe(), osol.w0) < tol
    assert np.array_equal(gs.support_mask(), osol.mask)
    st, ost = gs.init_state(), osol.init_state()
    for _ in range(3):
        gs.step(st)
        osol.step(ost)
    compare(st, ost, tol * 10)


@pytest.mark.parametrize("N,step,D,grid", [(256, 16, 2, None), (320, 16, None, (2, 2)), (250, 17, 2, None)])
def test_streamed_blind_frames_match_oracle(N, step, D, grid):
    """float32 s = 64: the BLIND frame pass runs as two streamed launches (the
    R-factor forward with w, then the sweep with W_d and raw q_j output)."""
    f, oplan, plan = blind_problem(N=N, s=64, step=step, D=D or 1, grid=grid, peak=1e4)
    f = fp32_intensity(f)
    cfg = dict(r=5e3)
    gs = P.BlindSolver(plan, f, P.BlindConfig(**cfg), dtype="f32")
    osol = O.BlindSolver(oplan, f, O.BlindConfig(**cfg))
    st, ost = gs.init_state(), osol.init_state()
    for _ in range(2):
        gs.step(st)
        osol.step(ost)
    compare(st, ost, 1e-4)
    res = P.BlindSolver(plan, f, P.BlindConfig(max_iters=5, tol_rf=1e-300, **cfg), dtype="f32").run()
    _, om, oprobe, _, orec = O.BlindSolver(oplan, f, O.BlindConfig(max_iters=5, tol_rf=1e-300, **cfg)).run()
    assert np.max(np.abs(np.array([r.rf for r in res.records]) - [r.rf for r in orec]) /
                  np.array([r.rf for r in orec])) < 1e-3
    assert rel_l2(res.merged, om) < 1e-3
    assert rel_l2(res.probe, oprobe) < 1e-3


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-5)])
def test_blind_custom_initial_probe(dtype, tol):
    # config 3 style: disk initial probe, default support estimate
    f, oplan, plan = blind_problem(D=2)
    if dtype == "f32":
        f = fp32_intensity(f)
    w0 = sim.disk_probe(32, 12.0)
    gs = P.BlindSolver(plan, f, P.BlindConfig(), dtype=dtype)
    osol = O.BlindSolver(oplan, f, O.BlindConfig())
    st, ost = gs.init_state(w0), osol.init_state(w0)
    assert rel_l2(st.w, ost.w) == 0.0
    gs.step(st)
    osol.step(ost)
    compare(st, ost, tol * 10)


def test_blind_run_matches_oracle_short_horizon():
    f, oplan, plan = blind_problem(D=2, peak=1e4)
    cfg = dict(r=1e3, max_iters=8, tol_rf=1e-300)
    res = P.BlindSolver(plan, f, P.BlindConfig(**cfg), dtype="f64").run()
    ou, om, oprobe, ospec, orec = O.BlindSolver(oplan, f, O.BlindConfig(**cfg)).run()
    assert res.iterations == len(orec) == 8
    assert np.max(np.abs(np.array([r.rf for r in res.records]) - [r.rf for r in orec])) < 1e-9
    assert np.max(np.abs(np.array([r.re for r in res.records]) - [r.re for r in orec])) < 1e-9
    assert rel_l2(res.merged, om) < 1e-9
    assert rel_l2(res.probe, oprobe) < 1e-9


def test_blind_exact_support_zeros_and_probe_consistency():
    # test_blind.cpp:60-84 (shortened): masked spectrum has exact zeros and
    # the stored probe is its inverse transform
    f, _, plan = blind_problem(D=2)
    res = P.BlindSolver(plan, f, P.BlindConfig(r=1e3, max_iters=20, tol_rf=1e-4), dtype="f64").run()
    mask = res.support_mask
    assert np.all(res.probe_fourier[mask == 0.0] == 0.0)
    assert np.max(np.abs(P.ifft2_normalized(res.probe_fourier) - res.probe)) < 1e-12
    assert res.final_rf < res.records[0].rf


def test_full_spectrum_support_runs():
    # test_blind.cpp:104-114
    f, _, plan = blind_problem(D=2)
    res = P.BlindSolver(plan, f, P.BlindConfig(support_mask=np.ones((32, 32)), max_iters=5)).run()
    assert res.iterations == 5 and np.isfinite(res.final_rf)


def test_blind_config_validation():
    # test_blind.cpp:116-128
    f, _, plan = blind_problem(D=2)
    with pytest.raises(ValueError):
        P.BlindSolver(plan, f, P.BlindConfig(mu=0.0))
    with pytest.raises(ValueError):
        P.BlindSolver(plan, f, P.BlindConfig(support_mask=np.ones((8, 8))))
    with pytest.raises(ValueError):
        P.BlindSolver(plan, f, P.BlindConfig(support_mask=np.full((32, 32), 0.5)))


def test_disk_support_mask_geometry():
    # test_blind.cpp:35-45
    m = P.disk_support_mask(16, 3.0)
    assert m[0, 0] == 1.0 and m[0, 3] == 1.0 and m[0, 4] == 0.0 and m[13, 0] == 1.0 and m[8, 8] == 0.0
