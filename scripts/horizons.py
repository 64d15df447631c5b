"""Reproducible horizons of the five BASELINE configs (test infrastructure).

For each config, two float64 runs of the compiled reference (oracle/_ref) on
inputs that differ by a float32-level perturbation (every amplitude scaled by
1 + d, |d| <= 2^-24, seeded) -- the size of the rounding a float32 GPU run
commits per operation.  Config 0 (complex128 on the GPU) compares the compiled
reference with the numpy restatement instead (float64 FFT rounding only).
The per-iteration relative R-factor gap and the merged-image gap at a few
iterations show where any two implementations stop agreeing to the north-star
bounds; tests/config_cases.py HORIZON takes the horizons from here.

  python scripts/horizons.py [config ...]   -> profiles/r2_horizons.json
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import od2p as O  # noqa: E402
from oracle import ref_lib as R  # noqa: E402
from tests.config_cases import case  # noqa: E402
from tests.helpers import rel_l2  # noqa: E402

ITERS = {0: 100, 1: 60, 2: 25, 3: 40, "c4_band": 6}


def perturbed(f, seed=7):
    a = np.sqrt(f)
    d = np.random.default_rng(seed).uniform(-1.0, 1.0, a.shape) * 2.0 ** -24
    a = a * (1.0 + d)
    return a * a


def run(c, f, n):
    ps = c.ref_plan()
    if c.cfg.blind:
        cfg = R.blind_cfg(max_iters=n, tol_rf=1e-300, **c.cfg.solver)
        return R.blind_run(ps, f, cfg, w0=c.w0)
    return R.nonblind_run(ps, f, c.probe, R.nonblind_cfg(max_iters=n, tol_rf=1e-300))


def main(keys):
    out_path = os.path.join(ROOT, "profiles", "r2_horizons.json")
    res = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for k in keys:
        t0 = time.time()
        c = case(k)
        n = ITERS[k]
        a = run(c, c.f, n)
        if k == 0:
            g = O.make_raster_scan(c.N_rows, c.N_cols, c.cfg.s, c.cfg.step)
            _, m, rec = O.NonblindSolver(O.plan_stripes(g, 2), c.f, c.probe,
                                         O.NonblindConfig(max_iters=n, tol_rf=1e-300)).run()
            rf_b = np.array([r.rf for r in rec])
            merged_b = m
            what = "compiled reference vs numpy restatement (float64 FFT rounding)"
        else:
            b = run(c, perturbed(c.f), n)
            rf_b = b["records"][:, 0]
            merged_b = b["merged"]
            what = "amplitudes x (1 + d), |d| <= 2^-24"
        rf_a = a["records"][:, 0]
        gap = np.abs(rf_a - rf_b) / np.abs(rf_a)
        res[str(k)] = {
            "perturbation": what,
            "iterations": n,
            "rf_rel_gap": [float(x) for x in gap],
            "merged_rel_gap_final": rel_l2(merged_b, a["merged"]),
            "seconds": time.time() - t0,
        }
        print(k, "final merged gap %.3e" % res[str(k)]["merged_rel_gap_final"],
              "rf gap at", [(i + 1, "%.1e" % gap[i]) for i in range(0, n, max(1, n // 12))], flush=True)
        json.dump(res, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    ks = [a if a == "c4_band" else int(a) for a in sys.argv[1:]] or [0, 1, 3, 2]
    main(ks)
