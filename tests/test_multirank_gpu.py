"""The multi-rank path of the product, run on one GPU.

One handle over G in-process ranks (pdd_nonblind_create_multi /
pdd_blind_create_multi, csrc/multi.cpp) with a repeated device uses the
host-staged transport (csrc/transport.cpp) instead of NCCL, so the actual C++
solver runs with G ranks -- cut-pair send/recv of s = pi u + Lambda, both
D-vector all-reduces (R-factor and RE partials), the stop-rule agreement and
the state assembly -- on the single GPU of this box.  The reference's
thread-count determinism test (proj/tests/test_solver.cpp:201-216: 1 vs 3
workers agree to 1e-12) becomes: iterates and records are BIT-IDENTICAL for
every rank count at fixed D, on stripes and on a 2-D grid.
"""
import numpy as np
import pytest

import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import sim

pytestmark = pytest.mark.gpu


def problem(N=192, s=32, step=8, D=3, grid=None, peak=1e4, seed=3):
    probe = sim.make_probe(s, s / 4)
    obj = sim.make_object(N, 4.0, seed + 1, seed + 2)
    g = P.make_raster_scan(N, N, s, step)
    f = P.intensity(P.forward(probe, obj, g), dtype="f64")
    if peak:
        f = sim.poisson_host(f, peak, seed + 3)
    plan = P.plan_grid(g, *grid) if grid else P.plan_stripes(g, D)
    return plan, f, probe


def states_equal(a, b):
    for x, y in zip(a.u + a.z + a.gamma + a.v, b.u + b.z + b.gamma + b.v):
        assert np.array_equal(x, y)
    for (x0, x1), (y0, y1) in zip(a.lam, b.lam):
        assert np.array_equal(x0, y0) and np.array_equal(x1, y1)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("D,grid,ranks", [(3, None, 2), (3, None, 3), (None, (2, 2), 2), (None, (2, 2), 4)])
def test_nonblind_rank_count_invariance(dtype, D, grid, ranks):
    plan, f, probe = problem(D=D, grid=grid)
    one = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype=dtype)
    many = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype=dtype, devices=[0] * ranks)
    assert len(many.local_subs) == plan.D  # one handle, global state layout
    a, b = one.init_state(), many.init_state()
    states_equal(a, b)
    au, bu = [z.copy() for z in a.z], [z.copy() for z in b.z]
    for _ in range(3):
        one.step(a, au)
        many.step(b, bu)
        states_equal(a, b)
    cfg = P.NonblindConfig(max_iters=9, tol_rf=1e-300)
    r1 = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype).run()
    rn = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype, devices=[0] * ranks).run()
    assert r1.iterations == rn.iterations == 9
    assert [r.rf for r in r1.records] == [r.rf for r in rn.records]
    assert [r.re for r in r1.records] == [r.re for r in rn.records]
    assert np.array_equal(r1.merged, rn.merged)
    for x, y in zip(r1.sub_solutions, rn.sub_solutions):
        assert np.array_equal(x, y)


def test_nonblind_rank_count_invariance_stop_rule():
    """The R-factor stop rule fires on the same iteration on every rank (the
    all-reduced partials are identical), and rolls back identically."""
    plan, f, probe = problem(D=3, peak=None)
    probe_run = P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=30, tol_rf=1e-300), dtype="f32").run()
    tol = min(r.rf for r in probe_run.records[:20]) * (1 + 1e-9)
    cfg = P.NonblindConfig(max_iters=400, tol_rf=tol)
    r1 = P.NonblindSolver(plan, f, probe, cfg, dtype="f32").run()
    r3 = P.NonblindSolver(plan, f, probe, cfg, dtype="f32", devices=[0, 0, 0]).run()
    assert 1 < r1.iterations <= 20 and r1.iterations == r3.iterations
    assert r1.final_rf == r3.final_rf and np.array_equal(r1.merged, r3.merged)


@pytest.mark.parametrize("grid,ranks", [(None, 2), ((2, 2), 4)])
def test_blind_rank_count_invariance(grid, ranks):
    plan, f, _ = problem(N=160, D=2, grid=grid)
    cfg = P.BlindConfig(r=1e3)
    one = P.BlindSolver(plan, f, cfg, dtype="f32")
    many = P.BlindSolver(plan, f, cfg, dtype="f32", devices=[0] * ranks)
    a, b = one.init_state(), many.init_state()
    for _ in range(3):
        one.step(a)
        many.step(b)
    assert np.array_equal(a.w, b.w)
    for x, y in zip(a.w_copies + a.delta + a.u + a.gamma + a.v, b.w_copies + b.delta + b.u + b.gamma + b.v):
        assert np.array_equal(x, y)
    rc = P.BlindConfig(r=1e3, max_iters=6, tol_rf=1e-300)
    r1 = P.BlindSolver(plan, f, rc, dtype="f32").run()
    rn = P.BlindSolver(plan, f, rc, dtype="f32", devices=[0] * ranks).run()
    assert [r.rf for r in r1.records] == [r.rf for r in rn.records]
    assert np.array_equal(r1.merged, rn.merged) and np.array_equal(r1.probe, rn.probe)


def test_more_ranks_than_subdomains_is_rejected():
    plan, f, probe = problem(D=2)
    with pytest.raises(P.InvalidArgument):
        P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype="f32", devices=[0, 0, 0])


def test_on_iteration_streams_records_during_the_run():
    """solver.hpp:88: on_iteration sees every record, in order, while the device
    loop runs (poll windows of 16 iterations), not after it returns."""
    import time

    plan, f, probe = problem(N=512, s=64, step=16, D=2)
    cfg = P.NonblindConfig(max_iters=1500, tol_rf=1e-300)
    sol = P.NonblindSolver(plan, f, probe, cfg, dtype="f32")
    seen = []
    res = sol.run(on_iteration=lambda r: seen.append((time.perf_counter(), r)))
    t_ret = time.perf_counter()
    assert [r.iteration for _, r in seen] == list(range(1, res.iterations + 1))
    assert [r.rf for _, r in seen] == [r.rf for r in res.records]
    assert [r.re for _, r in seen] == [r.re for r in res.records]
    first, last = seen[0][0], seen[-1][0]
    assert last - first > 0.5 * (t_ret - first)  # spread over the loop, not delivered at the end
    # multi-rank handles stream from rank 0
    seen2 = []
    P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=40, tol_rf=1e-300), dtype="f32",
                     devices=[0, 0]).run(on_iteration=seen2.append)
    assert [r.iteration for r in seen2] == list(range(1, 41))
