"""ORACLE TEST INFRASTRUCTURE — ctypes access to the compiled, unmodified
reference (``oracle/_ref/libptychodd_ref.so``, built by ``oracle/build_ref.sh``
from ``/root/reference/proj/src`` + our FFTW-API shim).  Used by tests to pin the
numpy restatement, by ``tests/golden/make_golden.py``, and by ``bench.py``'s
reference / cpu_baseline legs.  Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libptychodd_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_r_factor_subs.restype = C.c_double
    return _lib


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(rc: int) -> None:
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


class PlanSpec(C.Structure):
    _fields_ = [("H", C.c_int64), ("W", C.c_int64), ("s", C.c_int64), ("step", C.c_int64),
                ("kind", C.c_int32), ("D", C.c_int32), ("Dr", C.c_int32), ("Dc", C.c_int32),
                ("axis", C.c_int32)]


class NonblindCfg(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("eta", C.c_double), ("r", C.c_double),
                ("tol_rf", C.c_double), ("tol_re", C.c_double), ("max_iters", C.c_int32),
                ("stop_rule", C.c_int32), ("record_lagrangian", C.c_int32), ("threads", C.c_int32)]


class BlindCfg(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("eta", C.c_double), ("r", C.c_double), ("mu", C.c_double),
                ("gamma", C.c_double), ("support_energy", C.c_double), ("tol_rf", C.c_double),
                ("tol_re", C.c_double), ("max_iters", C.c_int32), ("stop_rule", C.c_int32),
                ("threads", C.c_int32), ("has_mask", C.c_int32)]


def _p(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.c_void_p)


def _c(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _d(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def plan_spec(H, W, s, step, D=1, axis="auto", grid=None) -> PlanSpec:
    """kind 0: plan_stripes(D, axis); kind 1: plan_grid(*grid)."""
    ax = {"auto": 0, "columns": 1, "rows": 2}[axis]
    if grid is not None:
        return PlanSpec(H, W, s, step, 1, grid[0] * grid[1], grid[0], grid[1], 0)
    return PlanSpec(H, W, s, step, 0, D, 0, 0, ax)


@dataclass
class RefPlan:
    D: int
    positions: np.ndarray
    assignment: np.ndarray
    subdomains: np.ndarray
    pairs: np.ndarray
    regions: np.ndarray
    local_grid: np.ndarray


def plan(ps: PlanSpec) -> RefPlan:
    counts = np.zeros(3, np.int64)
    _check(lib().ref_plan(C.byref(ps), _p(counts), None, None, None, None, None, None))
    D, J, P = (int(x) for x in counts)
    pos = np.zeros((J, 2), np.int64)
    asg = np.zeros(J, np.int32)
    subs = np.zeros((D, 4), np.int64)
    pairs = np.zeros((max(P, 1), 2), np.int32)
    regs = np.zeros((max(P, 1), 4), np.int64)
    lgrid = np.zeros((D, 2), np.int64)
    _check(lib().ref_plan(C.byref(ps), _p(counts), _p(pos), _p(asg), _p(subs), _p(pairs), _p(regs), _p(lgrid)))
    return RefPlan(D, pos, asg, subs, pairs[:P], regs[:P], lgrid)


def fft2(x: np.ndarray, inverse=False) -> np.ndarray:
    a = _c(x).copy()
    _check(lib().ref_fft2(_p(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), C.c_int(int(inverse))))
    return a


def forward(probe, image, positions) -> np.ndarray:
    probe, image, pos = _c(probe), _c(image), np.ascontiguousarray(positions, np.int64)
    s = probe.shape[0]
    out = np.zeros((pos.shape[0], s, s), np.complex128)
    _check(lib().ref_forward(_p(probe), C.c_int64(s), _p(image), C.c_int64(image.shape[0]),
                             C.c_int64(image.shape[1]), _p(pos), C.c_int64(pos.shape[0]), _p(out)))
    return out


def adjoint(probe, frames, positions, H, W) -> np.ndarray:
    probe, frames, pos = _c(probe), _c(frames), np.ascontiguousarray(positions, np.int64)
    out = np.zeros((H, W), np.complex128)
    _check(lib().ref_adjoint(_p(probe), C.c_int64(probe.shape[0]), _p(frames), _p(pos),
                             C.c_int64(pos.shape[0]), C.c_int64(H), C.c_int64(W), _p(out)))
    return out


def illumination_density(probe, positions, H, W) -> np.ndarray:
    probe, pos = _c(probe), np.ascontiguousarray(positions, np.int64)
    out = np.zeros((H, W))
    _check(lib().ref_illumination_density(_p(probe), C.c_int64(probe.shape[0]), _p(pos),
                                          C.c_int64(pos.shape[0]), C.c_int64(H), C.c_int64(W), _p(out)))
    return out


def probe_density(image, positions, s) -> np.ndarray:
    image, pos = _c(image), np.ascontiguousarray(positions, np.int64)
    out = np.zeros((s, s))
    _check(lib().ref_probe_density(_p(image), C.c_int64(image.shape[0]), C.c_int64(image.shape[1]),
                                   _p(pos), C.c_int64(pos.shape[0]), C.c_int64(s), _p(out)))
    return out


def adjoint_probe(image, frames, positions) -> np.ndarray:
    image, frames, pos = _c(image), _c(frames), np.ascontiguousarray(positions, np.int64)
    s = frames.shape[1]
    out = np.zeros((s, s), np.complex128)
    _check(lib().ref_adjoint_probe(_p(image), C.c_int64(image.shape[0]), C.c_int64(image.shape[1]),
                                   _p(frames), _p(pos), C.c_int64(pos.shape[0]), C.c_int64(s), _p(out)))
    return out


def pixel_prox(y, b, lam, eps) -> np.ndarray:
    y, b = _c(y), _d(b)
    out = np.zeros_like(y)
    _check(lib().ref_pixel_prox(_p(y), _p(b), C.c_int64(y.size), C.c_double(lam), C.c_double(eps), _p(out)))
    return out


def pixel_value_gradient(x, b, eps):
    x, b = _c(x), _d(b)
    val = np.zeros(x.shape)
    grad = np.zeros_like(x)
    _check(lib().ref_pixel_value_gradient(_p(x), _p(b), C.c_int64(x.size), C.c_double(eps), _p(val), _p(grad)))
    return val, grad


def nonblind_cfg(epsilon=0.5, eta=0.1, r=4e3, max_iters=1000, tol_rf=1e-5, tol_re=1e-3,
                 stop_rule="rfactor", record_lagrangian=False, threads=0) -> NonblindCfg:
    return NonblindCfg(epsilon, eta, r, tol_rf, tol_re, max_iters, int(stop_rule != "rfactor"),
                       int(record_lagrangian), threads)


def blind_cfg(epsilon=0.5, eta=0.1, r=5e3, mu=2e2, gamma=1e-4, support_energy=0.995, max_iters=1000,
              tol_rf=1e-5, tol_re=1e-3, stop_rule="rfactor", threads=0, has_mask=False) -> BlindCfg:
    return BlindCfg(epsilon, eta, r, mu, gamma, support_energy, tol_rf, tol_re, max_iters,
                    int(stop_rule != "rfactor"), threads, int(has_mask))


def _sizes(rp: RefPlan, s: int):
    nsub = [int((r[1] - r[0]) * (r[3] - r[2])) for r in rp.subdomains]
    nreg = [int((r[1] - r[0]) * (r[3] - r[2])) for r in rp.regions]
    return nsub, nreg


def _split_images(flat, rp: RefPlan):
    out, o = [], 0
    for r in rp.subdomains:
        h, w = int(r[1] - r[0]), int(r[3] - r[2])
        out.append(flat[o : o + h * w].reshape(h, w))
        o += h * w
    return out


def _split_regions(flat, rp: RefPlan, per=1):
    out, o = [], 0
    for r in rp.regions:
        h, w = int(r[1] - r[0]), int(r[3] - r[2])
        grp = []
        for _ in range(per):
            grp.append(flat[o : o + h * w].reshape(h, w))
            o += h * w
        out.append(grp if per > 1 else grp[0])
    return out


def _split_frames(flat, rp: RefPlan, s):
    out, o = [], 0
    for d in range(rp.D):
        n = int(np.sum(rp.assignment == d))
        out.append(flat[o : o + n * s * s].reshape(n, s, s))
        o += n * s * s
    return out


def nonblind_run(ps: PlanSpec, intensities, probe, cfg: NonblindCfg, pin=None):
    rp = plan(ps)
    nsub, _ = _sizes(rp, ps.s)
    merged = np.zeros((ps.H, ps.W), np.complex128)
    subs = np.zeros(sum(nsub), np.complex128)
    rec = np.zeros((cfg.max_iters, 4))
    n = C.c_int64(0)
    f, pr = _d(intensities), _c(probe)
    pin = None if pin is None else _d(pin)
    _check(lib().ref_nonblind_run(C.byref(ps), _p(f), _p(pr), _p(pin), C.byref(cfg), _p(merged), _p(subs),
                                  _p(rec), C.byref(n)))
    return {"merged": merged, "subs": _split_images(subs, rp), "records": rec[: n.value], "iterations": n.value}


def nonblind_steps(ps: PlanSpec, intensities, probe, cfg: NonblindCfg, nsteps: int, pin=None):
    rp = plan(ps)
    s = ps.s
    nsub, nreg = _sizes(rp, s)
    J = rp.positions.shape[0]
    u = np.zeros(sum(nsub), np.complex128)
    z = np.zeros(J * s * s, np.complex128)
    g = np.zeros_like(z)
    au = np.zeros_like(z)
    v = np.zeros(max(sum(nreg), 1), np.complex128)
    lam = np.zeros(max(2 * sum(nreg), 1), np.complex128)
    rf = np.zeros(max(nsteps, 1))
    pin = None if pin is None else _d(pin)
    _check(lib().ref_nonblind_steps(C.byref(ps), _p(_d(intensities)), _p(_c(probe)), _p(pin), C.byref(cfg),
                                    C.c_int64(nsteps), _p(u), _p(z), _p(g), _p(au), _p(v), _p(lam), _p(rf)))
    return {"u": _split_images(u, rp), "z": _split_frames(z, rp, s), "gamma": _split_frames(g, rp, s),
            "au": _split_frames(au, rp, s), "v": _split_regions(v, rp), "lam": _split_regions(lam, rp, 2),
            "rf": rf[:nsteps]}


def blind_run(ps: PlanSpec, intensities, cfg: BlindCfg, pin=None, mask=None, w0=None):
    rp = plan(ps)
    s = ps.s
    nsub, _ = _sizes(rp, s)
    merged = np.zeros((ps.H, ps.W), np.complex128)
    subs = np.zeros(sum(nsub), np.complex128)
    probe = np.zeros((s, s), np.complex128)
    spec = np.zeros((s, s), np.complex128)
    mask_out = np.zeros((s, s))
    w0_out = np.zeros((s, s), np.complex128)
    rec = np.zeros((cfg.max_iters, 4))
    n = C.c_int64(0)
    pin = None if pin is None else _d(pin)
    mask = None if mask is None else _d(mask)
    w0 = None if w0 is None else _c(w0)
    _check(lib().ref_blind_run(C.byref(ps), _p(_d(intensities)), _p(pin), C.byref(cfg), _p(mask), _p(w0),
                               _p(merged), _p(subs), _p(probe), _p(spec), _p(mask_out), _p(w0_out), _p(rec),
                               C.byref(n)))
    return {"merged": merged, "subs": _split_images(subs, rp), "probe": probe, "probe_fourier": spec,
            "mask": mask_out, "w0": w0_out, "records": rec[: n.value], "iterations": n.value}


def blind_steps(ps: PlanSpec, intensities, cfg: BlindCfg, nsteps: int, pin=None, mask=None, w0=None):
    rp = plan(ps)
    s = ps.s
    nsub, nreg = _sizes(rp, s)
    J = rp.positions.shape[0]
    w = np.zeros((s, s), np.complex128)
    wc = np.zeros((rp.D, s, s), np.complex128)
    dl = np.zeros((rp.D, s, s), np.complex128)
    u = np.zeros(sum(nsub), np.complex128)
    z = np.zeros(J * s * s, np.complex128)
    g = np.zeros_like(z)
    v = np.zeros(max(sum(nreg), 1), np.complex128)
    lam = np.zeros(max(2 * sum(nreg), 1), np.complex128)
    pin = None if pin is None else _d(pin)
    mask = None if mask is None else _d(mask)
    w0 = None if w0 is None else _c(w0)
    _check(lib().ref_blind_steps(C.byref(ps), _p(_d(intensities)), _p(pin), C.byref(cfg), _p(mask), _p(w0),
                                 C.c_int64(nsteps), _p(w), _p(wc), _p(dl), _p(u), _p(z), _p(g), _p(v), _p(lam)))
    return {"w": w, "w_copies": list(wc), "delta": list(dl), "u": _split_images(u, rp),
            "z": _split_frames(z, rp, s), "gamma": _split_frames(g, rp, s), "v": _split_regions(v, rp),
            "lam": _split_regions(lam, rp, 2)}


def simulate_frames(probe, sample, step) -> np.ndarray:
    probe, sample = _c(probe), _c(sample)
    s = probe.shape[0]
    H, W = sample.shape
    gr, gc = (H - s) // step + 1, (W - s) // step + 1
    out = np.zeros((gr * gc, s, s))
    _check(lib().ref_simulate_frames(_p(probe), C.c_int64(s), _p(sample), C.c_int64(H), C.c_int64(W),
                                     C.c_int64(step), _p(out)))
    return out


def add_poisson_noise(frames, scale, seed) -> np.ndarray:
    f = _d(frames)
    out = np.zeros_like(f)
    _check(lib().ref_add_poisson_noise(_p(f), C.c_int64(f.shape[0]), C.c_int64(f.shape[1]), C.c_double(scale),
                                       C.c_uint64(seed), _p(out)))
    return out


def toy(size, probe_side, step, seed):
    """make_toy of the reference tests (proj/tests/test_solver.cpp:22-32)."""
    sample = np.zeros((size, size), np.complex128)
    probe = np.zeros((probe_side, probe_side), np.complex128)
    pin = np.zeros((size, size))
    _check(lib().ref_toy(C.c_int64(size), C.c_int64(probe_side), C.c_int64(step), C.c_uint64(seed),
                         _p(sample), _p(probe), _p(pin)))
    return sample, probe, pin


# ---- the reference's own I/O (io.cpp), when compiled in (build_ref.sh) ----
def has_io() -> bool:
    return available() and hasattr(lib(), "ref_write_dataset")


def write_dataset(path, H, W, s, step, frames, probe, pin=None, sample=None, noisy=False) -> None:
    """A dataset directory exactly as the reference CLI's `simulate` writes it
    (ptychodd_cli.cpp:155-169): frames.ptya, probe.ptya, [pin.ptya],
    [sample.ptya], meta.json."""
    pin = None if pin is None else _d(pin)
    sample = None if sample is None else _c(sample)
    _check(lib().ref_write_dataset(os.fsencode(str(path)), C.c_int64(H), C.c_int64(W), C.c_int64(s),
                                   C.c_int64(step), _p(_d(frames)), _p(_c(probe)), _p(pin), _p(sample),
                                   C.c_int(int(noisy))))


def write_frames(path, frames) -> None:
    f = _d(frames)
    _check(lib().ref_write_frames(os.fsencode(str(path)), _p(f), C.c_int64(f.shape[0]), C.c_int64(f.shape[1]),
                                  C.c_int64(f.shape[2])))


def read_array(path, kind: str):
    """kind 'complex' | 'real' | 'frames' -> numpy array via read_complex_array /
    read_real_array / read_frames.  FormatError surfaces as RefError code 6."""
    code = {"frames": 0, "real": 1, "complex": 2}[kind]
    dims = np.zeros(3, np.int64)
    _check(lib().ref_read_array(os.fsencode(str(path)), C.c_int(code), _p(dims), None))
    if code == 2:
        out = np.zeros((int(dims[0]), int(dims[1])), np.complex128)
    elif code == 1:
        out = np.zeros((int(dims[0]), int(dims[1])))
    else:
        out = np.zeros((int(dims[0]), int(dims[1]), int(dims[2])))
    _check(lib().ref_read_array(os.fsencode(str(path)), C.c_int(code), _p(dims), _p(out)))
    return out
