"""Download-path timing of NonblindSolver.run (developer tool): python scripts/e2e_dl.py [config]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2011_00162_b200 as P  # noqa: E402
from paper_2011_00162_b200 import _lib as L, sim  # noqa: E402
from paper_2011_00162_b200._lib import ptr  # noqa: E402
from paper_2011_00162_b200.ptychodd import _Prefault, _prefaulted  # noqa: E402

cfg = sim.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
inp = sim.make_inputs(cfg, device=True)
s = P.NonblindSolver(inp["plan"], None, inp["probe"], P.NonblindConfig(max_iters=50, tol_rf=1e-300),
                     amplitudes=inp["amplitudes_dev"], dtype=cfg.dtype)
g = inp["plan"].geometry
t0 = time.perf_counter()
a = _prefaulted((g.image_height, g.image_width)); b = _prefaulted((s._lay.image_elems,))
t1 = time.perf_counter()
print(f"prefault alone {t1-t0:.3f}", flush=True)
del a, b
n = C.c_int64(); div = C.c_int64(); rec = np.zeros((50, 3))
t0 = time.perf_counter()
pf = _Prefault((g.image_height, g.image_width), (s._lay.image_elems,)); pf.start()
rc = L.lib().pdd_nonblind_run(s._h, C.byref(n), ptr(rec), C.byref(div))
t1 = time.perf_counter()
merged, u = pf.result()
t2 = time.perf_counter()
L.check(L.lib().pdd_nonblind_merged(s._h, ptr(merged)))
t3 = time.perf_counter()
L.check(L.lib().pdd_nonblind_get_state(s._h, ptr(u), None, None, None, None, None))
t4 = time.perf_counter()
sp = s._split_images(u)
t5 = time.perf_counter()
print(f"run {t1-t0:.3f} join {t2-t1:.3f} merged {t3-t2:.3f} get_u {t4-t3:.3f} split {t5-t4:.3f}", flush=True)
