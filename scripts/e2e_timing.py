"""Breakdown of the end-to-end solve (developer tool): PDD_TIMING=1 python scripts/e2e_timing.py [config]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_00162_b200 as P  # noqa: E402
from paper_2011_00162_b200 import sim  # noqa: E402

cfg = sim.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
inp = sim.make_inputs(cfg, device=True)
host = torch.empty(inp["amplitudes_dev"].shape, dtype=torch.float32, pin_memory=True)
host.copy_(inp["amplitudes_dev"])
del inp["amplitudes_dev"]
torch.cuda.empty_cache()
t0 = time.perf_counter()
s = P.NonblindSolver(inp["plan"], None, inp["probe"], P.NonblindConfig(max_iters=cfg.iterations, tol_rf=1e-300),
                     amplitudes=host.numpy(), dtype=cfg.dtype)
t1 = time.perf_counter()
res = s.run()
t2 = time.perf_counter()
print(f"create {t1 - t0:.3f} s, run+download+merge {t2 - t1:.3f} s, iterations {res.iterations}", flush=True)
