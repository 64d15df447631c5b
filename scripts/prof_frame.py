"""Small driver for ncu: one solver on a BASELINE geometry with synthetic
amplitudes generated on the device (no host data path), N eager profiled
iterations.  Usage: python scripts/prof_frame.py <config> [iters]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2011_00162_b200 as P  # noqa: E402
from paper_2011_00162_b200 import _lib as L, sim  # noqa: E402

arg = sys.argv[1] if len(sys.argv) > 1 else "4"
if "/" in arg:  # ad-hoc geometry N/s/step (stripes over 8 row blocks, f32)
    N, s_, st = (int(x) for x in arg.split("/"))
    cfg = sim.Config(f"adhoc{N}_{s_}_{st}", N, s_, st, 4.0, s_ / 4, ("stripes", 8, "rows"), "f32", 1e4, 10)
else:
    cfg = sim.CONFIGS[int(arg)]
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
plan = sim.make_plan(cfg)
J, s = plan.geometry.frame_count(), cfg.s
g = torch.Generator(device="cuda").manual_seed(0)
amp = torch.rand((J, s, s), generator=g, device="cuda", dtype=torch.float32) * 30.0
probe = sim.make_probe(s, cfg.sigma_probe)
solver = P.NonblindSolver(plan, None, probe, P.NonblindConfig(max_iters=50), amplitudes=amp, dtype=cfg.dtype)
ms = (C.c_double * 3)()
L.check(L.lib().pdd_nonblind_profile(solver._h, C.c_int32(iters), ms))
print(f"{cfg.name}: frame {ms[0]:.3f} ms, gather {ms[1]:.3f} ms, iteration {ms[2]:.3f} ms")
