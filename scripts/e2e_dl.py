"""Phase timing of the e2e solve as bench.py runs it (developer tool):
python scripts/e2e_dl.py [config] [repeats]   (PDD_STAGED_D2H=0: plain pageable downloads)"""
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
from paper_2011_00162_b200.ptychodd import _Prefault  # noqa: E402

cfg = sim.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
inp = sim.make_inputs(cfg, device=True)
host = torch.empty(inp["amplitudes_dev"].shape, dtype=torch.float32, pin_memory=True)
host.copy_(inp["amplitudes_dev"])
del inp["amplitudes_dev"]
torch.cuda.empty_cache()
g = inp["plan"].geometry
J = host.shape[0]
for r in range(reps):
    t0 = time.perf_counter()
    s = P.NonblindSolver(inp["plan"], None, inp["probe"], P.NonblindConfig(max_iters=cfg.iterations, tol_rf=1e-300),
                         amplitudes=host.numpy(), dtype=cfg.dtype)
    t1 = time.perf_counter()
    n = C.c_int64()
    div = C.c_int64()
    rec = np.zeros((cfg.iterations, 3))
    pf = _Prefault((g.image_height, g.image_width), (s._lay.image_elems,))
    pf.start()
    rc = L.lib().pdd_nonblind_run(s._h, C.byref(n), ptr(rec), C.byref(div))
    t2 = time.perf_counter()
    merged, u = pf.result()
    t3 = time.perf_counter()
    L.check(L.lib().pdd_nonblind_merged(s._h, ptr(merged)))
    t4 = time.perf_counter()
    L.check(L.lib().pdd_nonblind_get_state(s._h, ptr(u), None, None, None, None, None))
    t5 = time.perf_counter()
    del s
    tot = t5 - t0
    print(f"staged={os.environ.get('PDD_STAGED_D2H', '1')} rep {r}: create {t1-t0:.3f} run {t2-t1:.3f} "
          f"join {t3-t2:.3f} merged {t4-t3:.3f} get_u {t5-t4:.3f} total {tot:.3f} "
          f"-> {J * cfg.iterations / tot / 1e6:.2f} M frames*it/s", flush=True)
