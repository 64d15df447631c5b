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


FLOOR_X = 5.0  # as tests/test_configs_gpu.py: blind float32 fields over the bound vs their measured float32 floor


def compare(st, ost, tol, f32ref=None):
    """Fields against their own norm.  f32ref: the numpy restatement evaluated
    in complex64 at the same point (the float32 floor); a float32 field over
    the bound must then stay within FLOOR_X of what float32 arithmetic itself
    makes of the step (z = sign(y) m at near-zero spectral values, Gamma's
    cancellation)."""
    def chk(name, a, b, ref=None, scale=None):
        sc = np.linalg.norm(b) if scale is None else scale
        e = np.linalg.norm(a - b) / sc
        if e < tol:
            return
        assert ref is not None, f"{name} {e:.3e} >= {tol}"
        floor = np.linalg.norm(ref - b) / sc
        assert e <= FLOOR_X * floor, f"{name} {e:.3e} vs float32 floor {floor:.3e}"

    R = f32ref
    chk("w", st.w, ost.w, None if R is None else R.w)
    for k, (a, b) in enumerate(zip(st.w_copies, ost.w_copies)):
        chk("w_copies", a, b, None if R is None else R.w_copies[k])
    for k, (a, b) in enumerate(zip(st.delta, ost.delta)):
        chk("delta", a, b, None if R is None else R.delta[k], scale=np.linalg.norm(ost.w))
    for k, (a, b) in enumerate(zip(st.u, ost.u)):
        chk("u", a, b, None if R is None else R.u[k])
    for k, (a, b) in enumerate(zip(st.gamma, ost.gamma)):
        chk("gamma", a, b, None if R is None else R.gamma[k])
    for k, (a, b) in enumerate(zip(st.v, ost.v)):
        chk("v", a, b, None if R is None else R.v[k])
    for k, ((a0, a1), (b0, b1), v) in enumerate(zip(st.lam, ost.lam, ost.v)):
        chk("lambda0", a0, b0, None if R is None else R.lam[k][0], scale=np.linalg.norm(v))
        chk("lambda1", a1, b1, None if R is None else R.lam[k][1], scale=np.linalg.norm(v))


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
    fsol = O.BlindSolver(oplan, f, O.BlindConfig(**cfg), precision="f32") if dtype == "f32" else None
    fst = fsol.init_state() if fsol else None
    for k in range(3):
        gs.step(st)
        osol.step(ost)
        if fsol:
            fsol.step(fst)
        if k == 0:
            compare(st, ost, tol, fst)  # one sweep: the north-star operator bound
    compare(st, ost, tol * 10, fst)


@pytest.mark.parametrize("N,step,D,grid", [(256, 16, 2, None), (320, 16, None, (2, 2)), (250, 17, 2, None)])
def test_streamed_blind_frames_match_oracle(N, step, D, grid):
    """float32 s = 64: the BLIND frame pass runs as ONE streamed launch -- the
    sweep with W_d (raw q_j output) with the shared-probe R-factor transform
    inside it (frame_stream.cuh RF2)."""
    f, oplan, plan = blind_problem(N=N, s=64, step=step, D=D or 1, grid=grid, peak=1e4)
    f = fp32_intensity(f)
    cfg = dict(r=5e3)
    gs = P.BlindSolver(plan, f, P.BlindConfig(**cfg), dtype="f32")
    osol = O.BlindSolver(oplan, f, O.BlindConfig(**cfg))
    fsol = O.BlindSolver(oplan, f, O.BlindConfig(**cfg), precision="f32")  # the float32 floor
    st, ost, fst = gs.init_state(), osol.init_state(), fsol.init_state()
    for k in range(2):
        gs.step(st)
        osol.step(ost)
        fsol.step(fst)
        if k == 0:
            compare(st, ost, 1e-5, fst)  # one sweep: the north-star operator bound
    compare(st, ost, 1e-4, fst)
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
