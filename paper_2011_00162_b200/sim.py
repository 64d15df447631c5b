"""Synthetic inputs for the five BASELINE.json configurations.

Input synthesis only -- outside every timed region.  No public dataset is
involved; seeded synthetic objects, probes and Poisson data with the configs'
shapes and value ranges stand in:
  object  N x N: amplitude = uniform noise (seed A), periodic Gaussian blur
          (kernel truncated at 4 sigma), rescaled to [0.5, 1.0]; phase the same
          from seed B, rescaled to [-pi/4, pi/4]
  probe   s x s: exp(-r^2 / (2 sigma_p^2)) * exp(i pi r^2 / s^2), r from (s/2, s/2)
  data    f = |FFT2(P o O_patch)|^2 (unitary), then for noisy configs
          Poisson(scale * f) / scale with scale = peak / max f (one global scale,
          as add_poisson_noise, simulate.cpp:162-178)
Small problems are simulated through the C-ABI forward operator in float64 and
noised with numpy; large ones run the forward model on the device
(pdd_simulate_intensity_device) and draw the Poisson counts with torch.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import Optional, Tuple

import numpy as np

from . import _lib as L
from .ptychodd import make_raster_scan, plan_grid, plan_stripes


@dataclass
class Config:
    name: str
    N: int
    s: int
    step: int
    sigma_obj: float
    sigma_probe: float
    plan: Tuple  # ("stripes", D, axis) | ("grid", Dr, Dc)
    dtype: str
    peak: Optional[float]  # Poisson peak photons; None = noiseless
    iterations: int
    blind: bool = False
    init_disk_radius: Optional[float] = None
    seeds: Tuple[int, int, int] = (11, 12, 13)
    solver: dict = field(default_factory=dict)

    @property
    def frames(self) -> int:
        n = (self.N - self.s) // self.step + 1
        return n * n


# BASELINE.json "configs" (Appendix A of SURVEY.md for the plan resolutions).
CONFIGS = {
    0: Config("c0", 128, 32, 8, 4.0, 8.0, ("stripes", 2, "auto"), "f64", None, 100, seeds=(1001, 1002, 1003)),
    1: Config("c1", 512, 64, 16, 4.0, 16.0, ("stripes", 2, "auto"), "f32", 1e4, 200, seeds=(1101, 1102, 1103)),
    2: Config("c2", 2048, 128, 32, 8.0, 32.0, ("grid", 2, 4), "f32", 1e5, 100, seeds=(1201, 1202, 1203)),
    3: Config("c3", 1024, 64, 16, 8.0, 16.0, ("grid", 4, 2), "f32", 1e4, 300, blind=True, init_disk_radius=24.0,
              seeds=(1301, 1302, 1303), solver={"r": 5e3, "mu": 2e2, "gamma": 1e-4}),
    4: Config("c4", 8192, 128, 32, 16.0, 32.0, ("stripes", 8, "rows"), "f32", 1e5, 50, seeds=(1401, 1402, 1403)),
}


def gaussian_blur_periodic(img: np.ndarray, sigma: float) -> np.ndarray:
    """Periodic convolution with a unit-sum Gaussian truncated at 4 sigma."""
    H, W = img.shape
    rad = int(math.ceil(4.0 * sigma))
    k = np.zeros((H, W))
    ax = np.arange(-rad, rad + 1)
    g1 = np.exp(-(ax.astype(float) ** 2) / (2.0 * sigma * sigma))
    g2 = np.outer(g1, g1)
    g2 /= g2.sum()
    for i, dy in enumerate(ax):
        k[dy % H, ax % W] += g2[i]
    return np.fft.irfft2(np.fft.rfft2(img) * np.fft.rfft2(k), s=(H, W))


def _rescale(a: np.ndarray, lo: float, hi: float) -> np.ndarray:
    mn, mx = float(a.min()), float(a.max())
    return lo + (hi - lo) * (a - mn) / (mx - mn if mx > mn else 1.0)


def make_object(N: int, sigma: float, seed_amp: int, seed_phase: int) -> np.ndarray:
    amp = _rescale(gaussian_blur_periodic(np.random.default_rng(seed_amp).random((N, N)), sigma), 0.5, 1.0)
    ph = _rescale(gaussian_blur_periodic(np.random.default_rng(seed_phase).random((N, N)), sigma),
                  -math.pi / 4, math.pi / 4)
    return amp * np.exp(1j * ph)


def make_probe(s: int, sigma: float) -> np.ndarray:
    yy, xx = np.mgrid[0:s, 0:s].astype(float)
    r2 = (yy - s / 2) ** 2 + (xx - s / 2) ** 2
    return np.exp(-r2 / (2.0 * sigma * sigma)) * np.exp(1j * math.pi * r2 / (s * s))


def disk_probe(s: int, radius: float) -> np.ndarray:
    """Uniform-amplitude disk of the given radius, zero phase (config 3 initial probe)."""
    yy, xx = np.mgrid[0:s, 0:s].astype(float)
    return ((yy - s / 2) ** 2 + (xx - s / 2) ** 2 <= radius * radius).astype(np.complex128)


def make_plan(cfg: Config):
    g = make_raster_scan(cfg.N, cfg.N, cfg.s, cfg.step)
    if cfg.plan[0] == "grid":
        return plan_grid(g, cfg.plan[1], cfg.plan[2])
    return plan_stripes(g, cfg.plan[1], cfg.plan[2])


def simulate_intensity(probe: np.ndarray, obj: np.ndarray, positions: np.ndarray) -> np.ndarray:
    """Host float64 intensities via the C-ABI forward (float64 compute)."""
    s = probe.shape[0]
    J = positions.shape[0]
    out = np.zeros((J, s, s))
    L.check(L.lib().pdd_forward(L.ptr(L.c128(probe)), C.c_int64(s), L.ptr(L.c128(obj)), C.c_int64(obj.shape[0]),
                                C.c_int64(obj.shape[1]), L.ptr(L.i64(positions)), C.c_int64(J), None, L.ptr(out),
                                L.PDD_F64))
    return out


def poisson_host(f: np.ndarray, peak: float, seed: int) -> np.ndarray:
    scale = peak / float(f.max())
    return np.random.default_rng(seed).poisson(f * scale).astype(np.float64) / scale


def make_inputs(cfg: Config, device: bool = False):
    """Returns dict(plan, probe, object, intensities | amplitudes_dev, w0?).

    device=False: float64 host intensities (parity tests, reference runs).
    device=True : float32 amplitudes as a torch CUDA tensor (benchmark path).
    """
    plan = make_plan(cfg)
    probe = make_probe(cfg.s, cfg.sigma_probe)
    obj = make_object(cfg.N, cfg.sigma_obj, cfg.seeds[0], cfg.seeds[1])
    pos = plan.geometry.positions
    out = {"plan": plan, "probe": probe, "object": obj, "config": cfg}
    if cfg.blind and cfg.init_disk_radius:
        out["w0"] = disk_probe(cfg.s, cfg.init_disk_radius)
    if not device:
        f = simulate_intensity(probe, obj, pos)
        if cfg.peak is not None:
            f = poisson_host(f, cfg.peak, cfg.seeds[2])
        out["intensities"] = f
        return out
    import torch

    J, s = pos.shape[0], cfg.s
    inten = torch.empty((J, s, s), dtype=torch.float64, device="cuda")
    sim_dtype = L.PDD_F64  # float64 forward model (complex128 frame engine, every side)
    L.check(L.lib().pdd_simulate_intensity_device(L.ptr(L.c128(probe)), C.c_int64(s), L.ptr(L.c128(obj)),
                                                  C.c_int64(cfg.N), C.c_int64(cfg.N), L.ptr(L.i64(pos)),
                                                  C.c_int64(J), C.c_void_p(inten.data_ptr()), sim_dtype))
    if cfg.peak is not None:
        scale = cfg.peak / float(inten.max().item())
        gen = torch.Generator(device="cuda")
        gen.manual_seed(cfg.seeds[2])
        amp = torch.empty((J, s, s), dtype=torch.float32, device="cuda")
        chunk = max(1, (1 << 27) // (s * s))
        for a in range(0, J, chunk):  # bounded temporaries
            x = inten[a : a + chunk]
            amp[a : a + chunk] = torch.sqrt(torch.poisson(x * scale, generator=gen) / scale).float()
    else:
        amp = torch.sqrt(inten).float()
    del inten
    out["amplitudes_dev"] = amp
    return out
