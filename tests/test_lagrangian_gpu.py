"""Augmented Lagrangian on the device.

augmented_lagrangian (metrics.cpp:73-101) evaluated on the GPU -- frame terms
(stagm value + eta-weighted residual against Gamma) and overlap terms (r-weighted
residual against Lambda) -- both for a given state and as the per-iteration
ConvergenceRecord::lagrangian of run() with record_lagrangian
(solver.cpp:258-260).  Pinned against the compiled reference's records
(tests/golden/reference_goldens.npz, lag_*), and the reference's property
test (test_solver.cpp:234-266): inside the stability set the Lagrangian never
rises by more than 1e-9 relative.
"""
import os

import numpy as np
import pytest

from oracle import od2p as O
import paper_2011_00162_b200 as P
from tests.golden import cases

pytestmark = pytest.mark.gpu

G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_goldens.npz"))


def _problem(name):
    N, s, step, D, f, probe = cases.nonblind_inputs()[name]
    plan = P.plan_stripes(P.make_raster_scan(N, N, s, step), D)
    oplan = O.plan_stripes(O.make_raster_scan(N, N, s, step), D)
    return N, s, step, D, f, probe, plan, oplan


def _lags(plan, f, probe, dtype, **cfg):
    res = P.NonblindSolver(plan, f, probe, P.NonblindConfig(record_lagrangian=True, **cfg), dtype=dtype).run()
    return res, np.array([r.lagrangian for r in res.records])


@pytest.mark.parametrize("name", cases.LAGRANGIAN_CASES)
def test_state_lagrangian_matches_oracle(name):
    N, s, step, D, f, probe, plan, oplan = _problem(name)
    gs = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype="f64")
    osol = O.NonblindSolver(oplan, f, probe, O.NonblindConfig())
    st, ost = gs.init_state(), osol.init_state()
    au, oau = [z.copy() for z in st.z], [z.copy() for z in ost.z]
    ocfg = O.NonblindConfig()
    for k in range(3):
        if k:
            gs.step(st, au)
            osol.step(ost, oau)
        ref = O.augmented_lagrangian(ost, oau, osol.frames, oplan, ocfg.epsilon, ocfg.eta, ocfg.r)
        got = gs.augmented_lagrangian(st)
        assert abs(got - ref) <= 1e-10 * abs(ref), (k, got, ref)


def test_lagrangian_needs_z():
    N, s, step, D, f, probe, plan, oplan = _problem("n64D2")
    gs = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype="f64")
    gs.iterate(2)  # graph path: z is not kept
    import ctypes as C
    from paper_2011_00162_b200 import _lib as L
    out = C.c_double()
    with pytest.raises(P.InvalidArgument):
        L.check(L.lib().pdd_nonblind_lagrangian(gs._h, C.byref(out)))


@pytest.mark.parametrize("name", cases.LAGRANGIAN_CASES)
def test_recorded_lagrangian_matches_reference(name):
    N, s, step, D, f, probe, plan, oplan = _problem(name)
    res, lag = _lags(plan, f, probe, "f64", max_iters=15, tol_rf=1e-300)
    ref = G[f"lag_{name}_default"]
    assert res.iterations == 15 == len(ref)
    assert np.allclose(lag, ref, rtol=1e-9, atol=0)
    # records other than the Lagrangian are those of the graph path
    res2 = P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=15, tol_rf=1e-300), dtype="f64").run()
    assert np.allclose([r.rf for r in res.records], [r.rf for r in res2.records], rtol=1e-12, atol=0)
    assert np.allclose([r.re for r in res.records], [r.re for r in res2.records], rtol=1e-12, atol=0)
    assert np.abs(res.merged - res2.merged).max() <= 1e-12 * np.abs(res2.merged).max()
    assert all(r.lagrangian is None for r in res2.records)


@pytest.mark.parametrize("name", cases.LAGRANGIAN_CASES)
def test_lagrangian_monotone_inside_stability_set(name):
    """test_solver.cpp:234-266 / acceptance.cpp:336-369 on the GPU (float64):
    eta, r from the post-lemma recipe (eta ~ 40: the general three-candidate
    prox path), 60 iterations, each record <= previous + 1e-9 |previous|,
    and the history matches the compiled reference."""
    N, s, step, D, f, probe, plan, oplan = _problem(name)
    eta, r = cases.lagrangian_recipe(N, s, step, D, probe)
    res, lag = _lags(plan, f, probe, "f64", eta=eta, r=r, max_iters=60, tol_rf=1e-14)
    assert len(lag) == 60
    assert np.all(np.diff(lag) <= 1e-9 * np.abs(lag[:-1]))
    assert np.allclose(lag, G[f"lag_{name}_recipe"], rtol=1e-9, atol=0)


def test_lagrangian_float32_tracks_reference():
    """float32 device iterates, fp64 Lagrangian accumulation: the recipe run
    stays within 1e-4 of the reference and is monotone to float32 resolution."""
    N, s, step, D, f, probe, plan, oplan = _problem("n64D2")
    eta, r = cases.lagrangian_recipe(N, s, step, D, probe)
    a = np.sqrt(f).astype(np.float32).astype(np.float64)
    res, lag = _lags(plan, a * a, probe, "f32", eta=eta, r=r, max_iters=30, tol_rf=1e-14)
    ref = G["lag_n64D2_recipe"][:30]
    assert np.max(np.abs(lag - ref) / np.abs(ref)) < 1e-4
    assert np.all(np.diff(lag) <= 1e-5 * np.abs(lag[:-1]))
