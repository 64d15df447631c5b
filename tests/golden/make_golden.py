"""Generate golden fixtures from the compiled, unmodified reference.

Run here (where /root/reference exists and oracle/build_ref.sh has built
oracle/_ref/libptychodd_ref.so):  python tests/golden/make_golden.py
Writes tests/golden/reference_goldens.npz.  Inputs are seeded and regenerated
identically by the tests from paper_2011_00162_b200.sim object/probe helpers
and numpy forward models, so only reference OUTPUTS are stored.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import od2p as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402
from tests.golden import cases  # noqa: E402


def main():
    out = {}
    # FFT (fft.cpp) on non-square and square grids
    for name, x in cases.fft_inputs().items():
        out[f"fft_{name}"] = R.fft2(x)
        out[f"ifft_{name}"] = R.fft2(x, inverse=True)
    # forward model operators (forward.cpp)
    for name, (probe, img, pos, H, W, z) in cases.operator_inputs().items():
        out[f"fwd_{name}"] = R.forward(probe, img, pos)
        out[f"adj_{name}"] = R.adjoint(probe, z, pos, H, W)
        out[f"dens_{name}"] = R.illumination_density(probe, pos, H, W)
        out[f"pdens_{name}"] = R.probe_density(img, pos, probe.shape[0])
        out[f"adjp_{name}"] = R.adjoint_probe(img, z, pos)
    # ST-AGM prox (stagm.cpp:45-73)
    y, b = cases.prox_inputs()
    for lam, eps in cases.PROX_PARAMS:
        out[f"prox_{lam}_{eps}"] = R.pixel_prox(y, b, lam, eps)
    val, grad = R.pixel_value_gradient(y, b, 0.3)
    out["value_0.3"], out["gradient_0.3"] = val, grad
    # plans (ddplan.cpp)
    for name, spec in cases.PLAN_SPECS.items():
        rp = R.plan(R.plan_spec(**spec))
        out[f"plan_{name}_assign"] = rp.assignment
        out[f"plan_{name}_subs"] = rp.subdomains
        out[f"plan_{name}_pairs"] = rp.pairs
        out[f"plan_{name}_regions"] = rp.regions
        out[f"plan_{name}_lgrid"] = rp.local_grid
    # nonblind solver: 3 steps (state) and a 20-iteration run (records, image)
    for name, (N, s, step, D, f, probe) in cases.nonblind_inputs().items():
        ps = R.plan_spec(N, N, s, step, D)
        st = R.nonblind_steps(ps, f, probe, R.nonblind_cfg(), 3)
        for d, u in enumerate(st["u"]):
            out[f"nb_{name}_u{d}"] = u
        for p, (v, lam) in enumerate(zip(st["v"], st["lam"])):
            out[f"nb_{name}_v{p}"] = v
            out[f"nb_{name}_lam{p}"] = np.stack(lam)
        out[f"nb_{name}_gamma_norms"] = np.concatenate([np.linalg.norm(g, axis=(1, 2)) for g in st["gamma"]])
        out[f"nb_{name}_rf3"] = st["rf"]
        run = R.nonblind_run(ps, f, probe, R.nonblind_cfg(max_iters=20, tol_rf=1e-300))
        out[f"nb_{name}_records"] = run["records"][:, :2]
        out[f"nb_{name}_merged20"] = run["merged"]
    # augmented Lagrangian records (metrics.cpp:73-101 via solver.cpp:258-260):
    # default parameters, and the stability-set recipe of test_solver.cpp:234-266
    for name, (N, s, step, D, f, probe) in cases.nonblind_inputs().items():
        if name not in cases.LAGRANGIAN_CASES:
            continue
        ps = R.plan_spec(N, N, s, step, D)
        run = R.nonblind_run(ps, f, probe, R.nonblind_cfg(max_iters=15, tol_rf=1e-300, record_lagrangian=True))
        out[f"lag_{name}_default"] = run["records"][:, 2]
        eta, r = cases.lagrangian_recipe(N, s, step, D, probe)
        run = R.nonblind_run(ps, f, probe, R.nonblind_cfg(eta=eta, r=r, max_iters=60, tol_rf=1e-14,
                                                          record_lagrangian=True))
        out[f"lag_{name}_recipe"] = run["records"][:, 2]
    # blind solver: stock w0 + estimated mask, 2 steps; custom disk w0 run
    for name, (N, s, step, D, f, w0) in cases.blind_inputs().items():
        ps = R.plan_spec(N, N, s, step, D)
        bc = R.blind_cfg(r=1e3)
        st = R.blind_steps(ps, f, bc, 2)
        out[f"bl_{name}_w"] = st["w"]
        for d, u in enumerate(st["u"]):
            out[f"bl_{name}_u{d}"] = u
        run = R.blind_run(ps, f, R.blind_cfg(r=1e3, max_iters=6, tol_rf=1e-300))
        out[f"bl_{name}_w0"] = run["w0"]
        out[f"bl_{name}_mask"] = run["mask"]
        out[f"bl_{name}_records"] = run["records"][:, :2]
        out[f"bl_{name}_probe"] = run["probe"]
        run = R.blind_run(ps, f, R.blind_cfg(max_iters=6, tol_rf=1e-300), w0=w0)
        out[f"bl_{name}_disk_records"] = run["records"][:, :2]
        out[f"bl_{name}_disk_probe"] = run["probe"]
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_goldens.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
