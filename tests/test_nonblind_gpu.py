"""Nonblind OD²P parity: GPU solver vs the oracle on identical seeded inputs.

North-star bounds (BASELINE.json): one operator sweep <= 1e-5 relative L2 in
float32; reconstruction and R-factor after N iterations <= 1e-3 relative; the
float64 build tightens these (<= 1e-10 after N iterations).  The oracle is fed
the float32-rounded amplitudes (squared, exact in float64) so input rounding is
not an error source.
"""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import od2p as O
import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import sim

pytestmark = pytest.mark.gpu


def fp32_intensity(f):
    a = np.sqrt(f).astype(np.float32).astype(np.float64)
    return a * a


def small_problem(N=128, s=32, step=8, D=2, seed=0, peak=None, grid=None, axis="auto"):
    probe = sim.make_probe(s, s / 4)
    obj = sim.make_object(N, 4.0, seed + 1, seed + 2)
    g = O.make_raster_scan(N, N, s, step)
    f = O.intensity(O.forward(probe, obj, g))
    if peak:
        f = sim.poisson_host(f, peak, seed + 3)
    if grid:
        return probe, f, O.plan_grid(g, *grid), P.plan_grid(P.make_raster_scan(N, N, s, step), *grid)
    return probe, f, O.plan_stripes(g, D, axis), P.plan_stripes(P.make_raster_scan(N, N, s, step), D, axis)


def compare_state(st, ost, tol):
    for a, b in zip(st.u, ost.u):
        assert rel_l2(a, b) < tol, "u"
    for a, b in zip(st.gamma, ost.gamma):
        assert rel_l2(a, b) < tol, "gamma"
    for a, b in zip(st.z, ost.z):
        assert rel_l2(a, b) < tol, "z"
    for a, b in zip(st.v, ost.v):
        assert rel_l2(a, b) < tol, "v"
    for (a0, a1), (b0, b1) in zip(st.lam, ost.lam):
        if np.linalg.norm(b0) > 0:
            assert rel_l2(a0, b0) < tol, "lambda0"
            assert rel_l2(a1, b1) < tol, "lambda1"


@pytest.mark.parametrize("dtype,tol", [("f64", 1e-10), ("f32", 1e-5)])
@pytest.mark.parametrize("D,grid", [(1, None), (2, None), (3, None), (None, (2, 2))])
def test_one_sweep_matches_oracle(dtype, tol, D, grid):
    probe, f, oplan, plan = small_problem(D=D or 1, grid=grid)
    if dtype == "f32":
        f = fp32_intensity(f)
    cfg = P.NonblindConfig()
    gs = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype)
    osol = O.NonblindSolver(oplan, f, probe, O.NonblindConfig())
    st = gs.init_state()
    ost = osol.init_state()
    compare_state(st, ost, tol)
    au = [z.copy() for z in st.z]
    oau = [z.copy() for z in ost.z]
    gs.step(st, au)
    osol.step(ost, oau)
    compare_state(st, ost, tol)
    for a, b in zip(au, oau):
        assert rel_l2(a, b) < tol
    assert abs(gs.r_factor_of(au) - osol.r_factor_of(oau)) <= tol * osol.r_factor_of(oau) * 10


def test_sweeps_f64_track_oracle_over_iterations():
    probe, f, oplan, plan = small_problem(D=2)
    gs = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype="f64")
    osol = O.NonblindSolver(oplan, f, probe, O.NonblindConfig())
    st, ost = gs.init_state(), osol.init_state()
    au, oau = [z.copy() for z in st.z], [z.copy() for z in ost.z]
    for _ in range(5):
        gs.step(st, au)
        osol.step(ost, oau)
    compare_state(st, ost, 1e-10)


@pytest.mark.parametrize("dtype,tol,iters", [("f64", 1e-10, 60), ("f32", 1e-3, 60)])
def test_run_matches_oracle(dtype, tol, iters):
    probe, f, oplan, plan = small_problem(D=2, peak=1e4)
    if dtype == "f32":
        f = fp32_intensity(f)
    cfg = P.NonblindConfig(max_iters=iters, tol_rf=1e-300)
    res = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype).run()
    ou, omerged, orec = O.NonblindSolver(oplan, f, probe, O.NonblindConfig(max_iters=iters, tol_rf=1e-300)).run()
    assert res.iterations == iters == len(orec)
    assert rel_l2(res.merged, omerged) < tol
    rf = np.array([r.rf for r in res.records])
    orf = np.array([r.rf for r in orec])
    assert np.max(np.abs(rf - orf) / orf) < tol
    re = np.array([r.re for r in res.records])
    ore = np.array([r.re for r in orec])
    assert np.max(np.abs(re - ore) / ore) < max(tol, 1e-9) * 10


def test_run_stop_rules_match_oracle():
    # R-factor rule with a reachable tolerance: identical stop iteration and state.
    probe, f, oplan, plan = small_problem(D=2)
    ocfg = O.NonblindConfig(max_iters=200, tol_rf=0.25, r=300.0)
    _, _, orec = O.NonblindSolver(oplan, f, probe, ocfg).run()
    res = P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=200, tol_rf=0.25, r=300.0), dtype="f64").run()
    assert res.iterations == len(orec) < 200
    # relative-error rule
    ocfg = O.NonblindConfig(max_iters=200, stop_rule="relative_error", tol_re=5e-3, r=300.0)
    _, _, orec = O.NonblindSolver(oplan, f, probe, ocfg).run()
    res = P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=200, stop_rule="relative_error", tol_re=5e-3,
                                                            r=300.0), dtype="f64").run()
    assert res.iterations == len(orec)
    assert abs(res.final_re - orec[-1].re) < 1e-9


def test_singular_density_raises_runtime_error():
    # test_solver.cpp:281-285: a probe with one lit pixel leaves interior pixels dark
    g = P.make_raster_scan(40, 40, 8, 4)
    plan = P.plan_stripes(g, 2)
    dark = np.zeros((8, 8), complex)
    dark[0, 0] = 1.0
    f = np.ones((g.frame_count(), 8, 8))
    with pytest.raises(RuntimeError):
        P.NonblindSolver(plan, f, dark, P.NonblindConfig())
    with pytest.raises(ValueError):
        P.NonblindSolver(plan, f, dark, P.NonblindConfig(r=0.0))
    with pytest.raises(ValueError):
        P.NonblindSolver(plan, f, dark, P.NonblindConfig(), np.zeros((8, 8)))
