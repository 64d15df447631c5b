"""GPU path against the committed golden fixtures of the compiled reference
(tests/golden/reference_goldens.npz).  float64 compute <= 1e-10 (the fp64
build bound), float32 compute <= 1e-5 for single operators/sweeps."""
import os

import numpy as np
import pytest

from tests.helpers import rel_l2
from tests.golden import cases
import paper_2011_00162_b200 as P

pytestmark = pytest.mark.gpu
G = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_goldens.npz"))
TOL = {"f64": 1e-10, "f32": 1e-5}


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_fft_goldens(dtype):
    for name, x in cases.fft_inputs().items():
        assert rel_l2(P.fft2_normalized(x, dtype=dtype), G[f"fft_{name}"]) < TOL[dtype]
        assert rel_l2(P.ifft2_normalized(x, dtype=dtype), G[f"ifft_{name}"]) < TOL[dtype]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_operator_goldens(dtype):
    for name, (probe, img, pos, H, W, z) in cases.operator_inputs().items():
        s = probe.shape[0]
        g = P.ScanGeometry(s, 1, H, W, 1, pos.shape[0], pos)
        assert rel_l2(P.forward(probe, img, g, dtype=dtype), G[f"fwd_{name}"]) < TOL[dtype]
        assert rel_l2(P.adjoint(probe, z, g, dtype=dtype), G[f"adj_{name}"]) < TOL[dtype]
        assert rel_l2(P.illumination_density(probe, g, dtype=dtype), G[f"dens_{name}"]) < TOL[dtype]
        assert rel_l2(P.probe_density(img, g, dtype=dtype), G[f"pdens_{name}"]) < TOL[dtype]
        assert rel_l2(P.adjoint_probe(img, z, g, dtype=dtype), G[f"adjp_{name}"]) < TOL[dtype]


def test_prox_goldens():
    y, b = cases.prox_inputs()
    for lam, eps in cases.PROX_PARAMS:
        ref = G[f"prox_{lam}_{eps}"]
        assert np.max(np.abs(P.stagm.pixel_prox(y, b, lam, eps, dtype="f64") - ref)) <= 1e-14 * np.abs(ref).max()
        assert rel_l2(P.stagm.pixel_prox(y, b, lam, eps, dtype="f32"), ref) < 1e-6


def test_plan_goldens_bit_exact():
    for name, spec in cases.PLAN_SPECS.items():
        g = P.make_raster_scan(spec["H"], spec["W"], spec["s"], spec["step"])
        p = P.plan_grid(g, *spec["grid"]) if "grid" in spec else P.plan_stripes(g, spec["D"], spec.get("axis", "auto"))
        assert np.array_equal(p.frame_assignment, G[f"plan_{name}_assign"])
        subs = np.array([[r.row_start, r.row_end, r.col_start, r.col_end] for r in p.subdomains])
        assert np.array_equal(subs, G[f"plan_{name}_subs"])


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_nonblind_goldens(dtype):
    tol = TOL[dtype]
    for name, (N, s, step, D, f, probe) in cases.nonblind_inputs().items():
        plan = P.plan_stripes(P.make_raster_scan(N, N, s, step), D)
        sol = P.NonblindSolver(plan, f, probe, P.NonblindConfig(), dtype=dtype)
        st = sol.init_state()
        au = [z.copy() for z in st.z]
        rf = []
        for _ in range(3):
            sol.step(st, au)
            rf.append(sol.r_factor_of(au))
        for d, u in enumerate(st.u):
            assert rel_l2(u, G[f"nb_{name}_u{d}"]) < tol
        for p in range(len(plan.overlaps)):
            assert rel_l2(st.v[p], G[f"nb_{name}_v{p}"]) < tol
        gn = np.concatenate([np.linalg.norm(x, axis=(1, 2)) for x in st.gamma])
        assert rel_l2(gn, G[f"nb_{name}_gamma_norms"]) < tol
        assert np.allclose(rf, G[f"nb_{name}_rf3"], rtol=tol * 10, atol=0)
        if dtype == "f64":  # 20 iterations: inside the reference's reproducible horizon
            res = P.NonblindSolver(plan, f, probe, P.NonblindConfig(max_iters=20, tol_rf=1e-300), dtype=dtype).run()
            recs = np.array([[r.rf, r.re] for r in res.records])
            assert np.allclose(recs, G[f"nb_{name}_records"], rtol=1e-9, atol=0)
            assert rel_l2(res.merged, G[f"nb_{name}_merged20"]) < 1e-9


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_blind_goldens(dtype):
    tol = TOL[dtype]
    for name, (N, s, step, D, f, w0) in cases.blind_inputs().items():
        plan = P.plan_stripes(P.make_raster_scan(N, N, s, step), D)
        sol = P.BlindSolver(plan, f, P.BlindConfig(r=1e3), dtype=dtype)
        assert rel_l2(sol.initial_probe(), G[f"bl_{name}_w0"]) < tol
        assert np.array_equal(sol.support_mask(), G[f"bl_{name}_mask"])
        st = sol.init_state()
        for _ in range(2):
            sol.step(st)
        assert rel_l2(st.w, G[f"bl_{name}_w"]) < tol * 10
        for d, u in enumerate(st.u):
            assert rel_l2(u, G[f"bl_{name}_u{d}"]) < tol * 10
        if dtype == "f64":
            res = P.BlindSolver(plan, f, P.BlindConfig(r=1e3, max_iters=6, tol_rf=1e-300), dtype=dtype).run()
            assert np.allclose([[r.rf, r.re] for r in res.records], G[f"bl_{name}_records"], rtol=1e-9, atol=0)
            assert rel_l2(res.probe, G[f"bl_{name}_probe"]) < 1e-9
            res = P.BlindSolver(plan, f, P.BlindConfig(max_iters=6, tol_rf=1e-300), dtype=dtype).run(w0=w0)
            assert np.allclose([[r.rf, r.re] for r in res.records], G[f"bl_{name}_disk_records"], rtol=1e-9, atol=0)
            assert rel_l2(res.probe, G[f"bl_{name}_disk_probe"]) < 1e-9
