"""Graph-timed vs eager-profiled iteration (developer tool)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402,F401

import paper_2011_00162_b200 as P  # noqa: E402
from paper_2011_00162_b200 import _lib as L, sim  # noqa: E402

cfg = sim.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
inp = sim.make_inputs(cfg, device=True)
s = P.NonblindSolver(inp["plan"], None, inp["probe"], P.NonblindConfig(max_iters=200, tol_rf=1e-300),
                     amplitudes=inp["amplitudes_dev"], dtype=cfg.dtype)
for n in (2, 20, 40, 20):
    ms = C.c_double()
    L.check(L.lib().pdd_nonblind_iterate_timed(s._h, C.c_int32(n), C.byref(ms)))
    print(f"iterate_timed({n}): {ms.value:.2f} ms = {ms.value / n:.3f} ms/it", flush=True)
prof = (C.c_double * 3)()
L.check(L.lib().pdd_nonblind_profile(s._h, C.c_int32(4), prof))
print(f"profile: frame {prof[0]:.3f} gather {prof[1]:.3f} iteration {prof[2]:.3f}")
import time
s2 = P.NonblindSolver(inp["plan"], None, inp["probe"], P.NonblindConfig(max_iters=6, tol_rf=1e-300),
                      amplitudes=inp["amplitudes_dev"], dtype=cfg.dtype)
t0 = time.perf_counter(); r = s2.run(); t1 = time.perf_counter()
print(f"run(6 its) {t1 - t0:.3f} s, rf {[round(x.rf, 6) for x in r.records]}")
