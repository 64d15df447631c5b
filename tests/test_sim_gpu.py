"""Device-side input synthesis against the
reference: pdd_simulate_intensity_device is simulate_frames
(simulate.cpp:157-160 = intensity(forward(...)), forward.cpp:28-41, 95-106)
computed on the GPU; the device Poisson path follows add_poisson_noise
(simulate.cpp:162-178: Poisson(scale f) / scale, one global scale).  The
reference draws from libstdc++'s mt19937_64 + poisson_distribution, a stream
no GPU generator reproduces, so the noise is checked in distribution; the
parity tests therefore keep reference-generated data as ground truth
(tests/config_cases.py)."""
import ctypes as C

import numpy as np
import pytest

from oracle import ref_lib as R
import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import _lib as L
from paper_2011_00162_b200 import sim
from tests.helpers import rel_l2

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not R.available(), reason="oracle/_ref not built")]


@pytest.mark.parametrize("key", [0, 1, 3])
@pytest.mark.parametrize("dtype,tol", [("f64", 1e-12), ("f32", 1e-5)])
def test_device_simulation_matches_reference_simulate_frames(key, dtype, tol):
    import torch

    cfg = sim.CONFIGS[key]
    probe = sim.make_probe(cfg.s, cfg.sigma_probe)
    obj = sim.make_object(cfg.N, cfg.sigma_obj, *cfg.seeds[:2])
    ref = R.simulate_frames(probe, obj, cfg.step)
    g = P.make_raster_scan(cfg.N, cfg.N, cfg.s, cfg.step)
    J = g.frame_count()
    out = torch.empty((J, cfg.s, cfg.s), dtype=torch.float64, device="cuda")
    L.check(L.lib().pdd_simulate_intensity_device(L.ptr(L.c128(probe)), C.c_int64(cfg.s), L.ptr(L.c128(obj)),
                                                  C.c_int64(cfg.N), C.c_int64(cfg.N), L.ptr(L.i64(g.positions)),
                                                  C.c_int64(J), C.c_void_p(out.data_ptr()), L.dtype_code(dtype)))
    torch.cuda.synchronize()
    assert rel_l2(out.cpu().numpy(), ref) < tol


def test_device_simulation_large_frames_fp64():
    """128^2 frames through the complex128 streamed forward (config-2 geometry, a band)."""
    cfg = sim.CONFIGS[2]
    probe = sim.make_probe(cfg.s, cfg.sigma_probe)
    obj = np.ascontiguousarray(sim.make_object(cfg.N, cfg.sigma_obj, *cfg.seeds[:2])[:384])
    ref = R.simulate_frames(probe, obj, cfg.step)
    g = P.make_raster_scan(384, cfg.N, cfg.s, cfg.step)
    dev = P.intensity(P.forward(probe, obj, g, dtype="f64"), dtype="f64")
    assert rel_l2(dev, ref) < 1e-12


def test_device_poisson_noise_distribution():
    """The benchmark's device noise (sim.make_inputs) against the model of
    add_poisson_noise: counts ~ Poisson(scale f) with scale = peak / max f."""
    import torch

    cfg = sim.CONFIGS[1]
    inp = sim.make_inputs(cfg, device=True)
    amp = inp["amplitudes_dev"].double()
    probe, obj, g = inp["probe"], inp["object"], inp["plan"].geometry
    f = torch.as_tensor(P.intensity(P.forward(probe, obj, g, dtype="f64"), dtype="f64"), device="cuda")
    scale = cfg.peak / float(f.max())
    lam = f * scale
    counts = (amp ** 2) * scale
    assert bool(((counts - torch.round(counts)).abs() <= 1e-3 * counts.clamp(min=1)).all())  # integral counts
    m = lam > 10  # (k - lam) / sqrt(lam) has mean 0 and variance 1 exactly for Poisson counts
    z = ((counts - lam) / lam.sqrt())[m]
    assert z.numel() > 5000
    assert abs(float(z.mean())) < 0.05 and abs(float(z.var()) - 1.0) < 0.05
