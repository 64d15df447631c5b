"""Seeded inputs shared by make_golden.py (reference outputs) and the tests
(numpy only: no GPU library, no reference library needed to rebuild them)."""
import math

import numpy as np

from oracle import od2p as O

PROX_PARAMS = [(0.1, 0.5), (2.0, 0.5), (40.0, 0.3), (0.02, 0.95)]

PLAN_SPECS = {
    "s256_D2": dict(H=256, W=256, s=64, step=8, D=2),
    "s512_D6": dict(H=512, W=512, s=64, step=16, D=6),
    "rows3": dict(H=128, W=256, s=64, step=8, D=3, axis="rows"),
    "c2grid": dict(H=2048, W=2048, s=128, step=32, grid=(2, 4)),
    "c3grid": dict(H=1024, W=1024, s=64, step=16, grid=(4, 2)),
    "c4rows": dict(H=8192, W=8192, s=128, step=32, D=8, axis="rows"),
}


def rfield(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


def gaussian_probe(s, sigma):
    yy, xx = np.mgrid[0:s, 0:s].astype(float)
    r2 = (yy - s / 2) ** 2 + (xx - s / 2) ** 2
    return np.exp(-r2 / (2 * sigma * sigma)) * np.exp(1j * math.pi * r2 / (s * s))


def smooth_object(N, seed):
    r = np.random.default_rng(seed)
    k = np.fft.fftfreq(N)
    filt = np.exp(-(k[:, None] ** 2 + k[None, :] ** 2) * (2 * math.pi * 3.0) ** 2 / 2)
    a = np.real(np.fft.ifft2(np.fft.fft2(r.random((N, N))) * filt))
    p = np.real(np.fft.ifft2(np.fft.fft2(r.random((N, N))) * filt))
    a = 0.5 + 0.5 * (a - a.min()) / (a.max() - a.min())
    p = -math.pi / 4 + math.pi / 2 * (p - p.min()) / (p.max() - p.min())
    return a * np.exp(1j * p)


def fft_inputs():
    return {"16x12": rfield((16, 12), 4), "4x5": rfield((4, 5), 6), "32x32": rfield((32, 32), 7)}


def operator_inputs():
    out = {}
    for name, (H, s, step, seed) in {"toy12": (12, 4, 2, 1), "s16": (64, 16, 8, 2), "s32": (64, 32, 16, 3)}.items():
        g = O.make_raster_scan(H, H, s, step)
        out[name] = (rfield((s, s), seed), rfield((H, H), seed + 10), g.positions, H, H,
                     rfield((g.frame_count(), s, s), seed + 20))
    return out


def prox_inputs(n=4000):
    r = np.random.default_rng(11)
    y = r.uniform(0, 4, n) * np.exp(1j * r.uniform(-3.14, 3.14, n))
    y[:8] = 0.0  # sign(0) := 1 branch
    return y, r.uniform(0, 4, n)


def _poisson(f, peak, seed):
    scale = peak / f.max()
    return np.random.default_rng(seed).poisson(f * scale) / scale


def nonblind_inputs():
    out = {}
    for name, (N, s, step, D, peak, seed) in {"n64D2": (64, 16, 8, 2, None, 31), "n64D3": (64, 16, 4, 3, 1e4, 32),
                                                "n96D2": (96, 32, 8, 2, 1e4, 33)}.items():
        probe = gaussian_probe(s, s / 4)
        g = O.make_raster_scan(N, N, s, step)
        f = O.intensity(O.forward(probe, smooth_object(N, seed), g))
        if peak:
            f = _poisson(f, peak, seed + 1)
        out[name] = (N, s, step, D, f, probe)
    return out


def blind_inputs():
    out = {}
    for name, (N, s, step, D, seed) in {"b64": (64, 16, 4, 2, 41), "b96": (96, 32, 8, 2, 42)}.items():
        probe = gaussian_probe(s, s / 4)
        g = O.make_raster_scan(N, N, s, step)
        f = O.intensity(O.forward(probe, smooth_object(N, seed), g))
        yy, xx = np.mgrid[0:s, 0:s].astype(float)
        w0 = (((yy - s / 2) ** 2 + (xx - s / 2) ** 2) <= (0.375 * s) ** 2).astype(complex)
        out[name] = (N, s, step, D, f, w0)
    return out


# nonblind cases with augmented-Lagrangian goldens
LAGRANGIAN_CASES = ("n64D2", "n64D3")


def lagrangian_recipe(N, s, step, D, probe):
    """(eta, r) inside the stability set, the recipe of test_solver.cpp:234-266:
    c0 = max(2 max rho, sqrt(max rho)), c1 = 2 max rho over the subdomains'
    illumination densities, L = lipschitz_constant(0.5)."""
    plan = O.plan_stripes(O.make_raster_scan(N, N, s, step), D)
    mx = max(float(np.max(O.illumination_density(probe, lg))) for lg in plan.local_geometries)
    c0 = max(2.0 * mx, np.sqrt(mx))
    c1 = 2.0 * mx
    L = O.lipschitz_constant(0.5)
    eta = 1.05 * (6.0 * L + 2.0 * L * L + 2.0 * c1 * (L + 1.0) ** 2 / (c0 * c0))
    return eta, 1.1 * c0 * eta
