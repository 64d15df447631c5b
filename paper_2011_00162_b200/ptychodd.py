"""Python mirror of the reference's public C++ API (proj/include/ptychodd/*.hpp),
backed by the CUDA library through the C-ABI.

Same names, argument meaning and error types as the reference:
  scan.hpp     make_raster_scan, ScanGeometry, scan_coverage
  ddplan.hpp   plan_stripes (+ plan_grid), DecompositionPlan, restrict_overlap,
               merge, partition_frames
  fft.hpp      fft2_normalized, ifft2_normalized
  forward.hpp  forward, adjoint, illumination_density, probe_density,
               adjoint_probe, intensity
  stagm.hpp    stagm.pixel_prox / prox / pixel_value / pixel_gradient / value /
               gradient / lipschitz_constant / check_epsilon
  solver.hpp   NonblindConfig, SolverState, NonblindSolver (init_state, step,
               run, r_factor_of), ConvergenceRecord, NonblindResult
  blind.hpp    BlindConfig, BlindSolver, disk_support_mask
  metrics.hpp  r_factor, relative_error, snr_db
Fields are numpy arrays (complex128 for complex fields, float64 intensities);
frame stacks are [J, s, s] arrays.  Compute precision is chosen per call with
``dtype='f32'`` (complex64 on the GPU, the BASELINE configs 1-4) or ``'f64'``.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
import time
from dataclasses import dataclass, field
from types import SimpleNamespace
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _lib as L
from ._lib import (CudaError, DivergenceError, FormatError, InvalidArgument, OutOfRange, PtychoRuntimeError, c128,
                   check, f64, i64, ptr)

DEFAULT_DTYPE = "f64"


# --------------------------------------------------------------------------- scan / plans
@dataclass
class Region:
    """field.hpp:14-45 (half-open)."""

    row_start: int
    row_end: int
    col_start: int
    col_end: int

    def height(self) -> int:
        return self.row_end - self.row_start

    def width(self) -> int:
        return self.col_end - self.col_start

    def area(self) -> int:
        return self.height() * self.width()

    def contains(self, o: "Region") -> bool:
        return (o.row_start >= self.row_start and o.row_end <= self.row_end and o.col_start >= self.col_start
                and o.col_end <= self.col_end)

    def intersection(self, o: "Region") -> "Region":
        return Region(max(self.row_start, o.row_start), min(self.row_end, o.row_end),
                      max(self.col_start, o.col_start), min(self.col_end, o.col_end))

    def slices(self):
        return slice(self.row_start, self.row_end), slice(self.col_start, self.col_end)


@dataclass
class ScanGeometry:
    """scan.hpp:11-28."""

    frame_side: int
    step: int
    image_height: int
    image_width: int
    grid_rows: int
    grid_cols: int
    positions: np.ndarray  # [J, 2] int64

    def frame_count(self) -> int:
        return int(self.positions.shape[0])

    def window(self, j: int) -> Region:
        r, c = (int(x) for x in self.positions[j])
        return Region(r, r + self.frame_side, c, c + self.frame_side)


def _plan_handle(h: C.c_void_p) -> "DecompositionPlan":
    info = L.PlanInfo()
    check(L.lib().pdd_plan_info_get(h, C.byref(info)))
    J, D, P = info.n_frames, info.n_sub, info.n_pairs
    pos = np.zeros((J, 2), np.int64)
    asg = np.zeros(J, np.int32)
    subs = np.zeros((D, 4), np.int64)
    pairs = np.zeros((max(P, 1), 2), np.int32)
    regs = np.zeros((max(P, 1), 4), np.int64)
    lgrid = np.zeros((D, 2), np.int64)
    check(L.lib().pdd_plan_arrays(h, ptr(pos), ptr(asg), ptr(subs), ptr(pairs), ptr(regs), ptr(lgrid)))
    g = ScanGeometry(int(info.frame_side), int(info.step), int(info.image_height), int(info.image_width),
                     int(info.grid_rows), int(info.grid_cols), pos)
    return DecompositionPlan(h, g, D, subs, asg, pairs[:P], regs[:P], lgrid)


class DecompositionPlan:
    """ddplan.hpp:12-35, owning a C++ plan (pdd_plan*)."""

    def __init__(self, handle, geometry, D, subs, assign, pairs, regions, local_grid):
        self._h = handle
        self.geometry = geometry
        self.D = int(D)
        self.subdomains = [Region(*(int(x) for x in r)) for r in subs]
        self.frame_assignment = assign
        self.frames_of = [np.nonzero(assign == d)[0].astype(np.int64) for d in range(self.D)]
        self.overlaps = [SimpleNamespace(d1=int(p[0]), d2=int(p[1]), region=Region(*(int(x) for x in r)))
                         for p, r in zip(pairs, regions)]
        self.local_geometries = []
        for d, sub in enumerate(self.subdomains):
            lp = geometry.positions[self.frames_of[d]] - np.array([sub.row_start, sub.col_start], np.int64)
            self.local_geometries.append(ScanGeometry(geometry.frame_side, geometry.step, sub.height(), sub.width(),
                                                      int(local_grid[d][0]), int(local_grid[d][1]), lp))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            L.lib().pdd_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def pair_index(self, a: int, b: int) -> int:
        """ddplan.cpp:7-12."""
        a, b = min(a, b), max(a, b)
        for p, ov in enumerate(self.overlaps):
            if ov.d1 == a and ov.d2 == b:
                return p
        raise InvalidArgument("DecompositionPlan: subdomains are not neighbors")

    def local_overlap(self, d: int, p: int) -> Region:
        """ddplan.cpp:14-19."""
        ov, sub = self.overlaps[p].region, self.subdomains[d]
        return Region(ov.row_start - sub.row_start, ov.row_end - sub.row_start, ov.col_start - sub.col_start,
                      ov.col_end - sub.col_start)

    def pairs_of(self, d: int) -> List[int]:
        """ddplan.cpp:21-26."""
        return [p for p, ov in enumerate(self.overlaps) if ov.d1 == d or ov.d2 == d]


def make_raster_scan(image_height: int, image_width: int, frame_side: int, step: int) -> ScanGeometry:
    """scan.cpp:18-34 (built by the C++ plan layer)."""
    return plan_stripes_raw(image_height, image_width, frame_side, step, 1, "auto").geometry


_AXES = {"auto": 0, "columns": 1, "rows": 2}


def plan_stripes_raw(H, W, s, step, D, axis="auto") -> DecompositionPlan:
    h = C.c_void_p()
    check(L.lib().pdd_plan_stripes(C.c_int64(H), C.c_int64(W), C.c_int64(s), C.c_int64(step), C.c_int32(D),
                                   C.c_int32(_AXES[axis]), C.byref(h)))
    return _plan_handle(h)


def plan_stripes(geometry: ScanGeometry, D: int, axis: str = "auto") -> DecompositionPlan:
    """ddplan.cpp:28-94 (raster geometries, as the reference produces them)."""
    g = geometry
    return plan_stripes_raw(g.image_height, g.image_width, g.frame_side, g.step, D, axis)


def plan_grid(geometry: ScanGeometry, Dr: int, Dc: int) -> DecompositionPlan:
    """2-D block plan (configs 2 and 3)."""
    g = geometry
    h = C.c_void_p()
    check(L.lib().pdd_plan_grid(C.c_int64(g.image_height), C.c_int64(g.image_width), C.c_int64(g.frame_side),
                                C.c_int64(g.step), C.c_int32(Dr), C.c_int32(Dc), C.byref(h)))
    return _plan_handle(h)


def plan_from_arrays(geometry: ScanGeometry, D: int, assignment, subdomains, pairs, regions) -> DecompositionPlan:
    """Any DecompositionPlan (ddplan.hpp:12-35) from its arrays: frame
    assignment [J], subdomain rectangles [D][4] (r0, r1, c0, c1), overlap
    pairs [P][2] (d1 < d2) and regions [P][4]; validated as the reference's
    plan invariants require (windows inside their subdomain, overlaps inside
    both sides)."""
    g = geometry
    pos = np.ascontiguousarray(g.positions, np.int64)
    asg = np.ascontiguousarray(assignment, np.int32)
    subs = np.ascontiguousarray(subdomains, np.int64).reshape(-1, 4)
    prs = np.ascontiguousarray(pairs, np.int32).reshape(-1, 2)
    regs = np.ascontiguousarray(regions, np.int64).reshape(-1, 4)
    h = C.c_void_p()
    check(L.lib().pdd_plan_from_arrays(C.c_int64(g.frame_side), C.c_int64(g.step), C.c_int64(g.image_height),
                                       C.c_int64(g.image_width), C.c_int64(pos.shape[0]), ptr(pos), C.c_int32(D),
                                       ptr(asg), ptr(subs), C.c_int32(prs.shape[0]), ptr(prs), ptr(regs),
                                       C.byref(h)))
    return _plan_handle(h)


def scan_coverage(geometry: ScanGeometry) -> np.ndarray:
    """scan.cpp:36-44 (as float64, like RealField2D)."""
    plan = plan_stripes(geometry, 1) if geometry.frame_count() == geometry.grid_rows * geometry.grid_cols else None
    out = np.zeros((geometry.image_height, geometry.image_width), np.int32)
    check(L.lib().pdd_scan_coverage(plan.handle, ptr(out)))
    return out.astype(np.float64)


def restrict_overlap(u_d: np.ndarray, plan: DecompositionPlan, d: int, neighbor: int) -> np.ndarray:
    """ddplan.cpp:96-102."""
    p = plan.pair_index(d, neighbor)
    sub = plan.subdomains[d]
    if u_d.shape != (sub.height(), sub.width()):
        raise InvalidArgument("restrict_overlap: sub-solution shape mismatch")
    return u_d[plan.local_overlap(d, p).slices()].copy()


def merge(sub_solutions: Sequence[np.ndarray], plan: DecompositionPlan) -> np.ndarray:
    """ddplan.cpp:104-121."""
    if len(sub_solutions) != plan.D:
        raise InvalidArgument("merge: one sub-solution per subdomain required")
    for u, sub in zip(sub_solutions, plan.subdomains):
        if u.shape != (sub.height(), sub.width()):
            raise InvalidArgument("merge: sub-solution shape mismatch")
    flat = c128(np.concatenate([c128(u).ravel() for u in sub_solutions]))
    g = plan.geometry
    out = np.zeros((g.image_height, g.image_width), np.complex128)
    check(L.lib().pdd_merge(plan.handle, ptr(flat), ptr(out)))
    return out


def partition_frames(frames: np.ndarray, plan: DecompositionPlan) -> List[np.ndarray]:
    """ddplan.cpp:123-133."""
    if frames.shape[0] != plan.geometry.frame_count():
        raise InvalidArgument("partition_frames: frame count mismatch")
    return [frames[plan.frames_of[d]] for d in range(plan.D)]


# --------------------------------------------------------------------------- fft / forward
def _dt(dtype) -> int:
    return L.dtype_code(dtype or DEFAULT_DTYPE)


def fft2_normalized(x: np.ndarray, dtype=None) -> np.ndarray:
    """fft.cpp:49-55."""
    a = c128(x).copy()
    check(L.lib().pdd_fft2(ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), C.c_int32(0), _dt(dtype)))
    return a


def ifft2_normalized(x: np.ndarray, dtype=None) -> np.ndarray:
    """fft.cpp:57-62."""
    a = c128(x).copy()
    check(L.lib().pdd_fft2(ptr(a), C.c_int64(a.shape[0]), C.c_int64(a.shape[1]), C.c_int32(1), _dt(dtype)))
    return a


def _check_probe_image(probe, image, g: ScanGeometry):
    if probe.shape != (g.frame_side, g.frame_side):
        raise InvalidArgument("forward model: probe shape != frame_side^2")
    if image is not None and image.shape != (g.image_height, g.image_width):
        raise InvalidArgument("forward model: image shape != geometry image_shape")


def forward(probe: np.ndarray, image: np.ndarray, geometry: ScanGeometry, dtype=None) -> np.ndarray:
    """forward.cpp:28-41."""
    _check_probe_image(probe, image, geometry)
    s, J = geometry.frame_side, geometry.frame_count()
    out = np.zeros((J, s, s), np.complex128)
    pr, im, pos = c128(probe), c128(image), i64(geometry.positions)
    check(L.lib().pdd_forward(ptr(pr), C.c_int64(s), ptr(im), C.c_int64(image.shape[0]), C.c_int64(image.shape[1]),
                              ptr(pos), C.c_int64(J), ptr(out), None, _dt(dtype)))
    return out


def adjoint(probe: np.ndarray, frames: np.ndarray, geometry: ScanGeometry, dtype=None) -> np.ndarray:
    """forward.cpp:43-54."""
    _check_probe_image(probe, None, geometry)
    s, J = geometry.frame_side, geometry.frame_count()
    if frames.shape != (J, s, s):
        raise InvalidArgument("forward model: frame count mismatch")
    H, W = geometry.image_height, geometry.image_width
    out = np.zeros((H, W), np.complex128)
    pr, fr, pos = c128(probe), c128(frames), i64(geometry.positions)
    check(L.lib().pdd_adjoint(ptr(pr), C.c_int64(s), ptr(fr), ptr(pos), C.c_int64(J), C.c_int64(H), C.c_int64(W),
                              ptr(out), _dt(dtype)))
    return out


def illumination_density(probe: np.ndarray, geometry: ScanGeometry, dtype=None) -> np.ndarray:
    """forward.cpp:56-66."""
    _check_probe_image(probe, None, geometry)
    g = geometry
    out = np.zeros((g.image_height, g.image_width))
    pr, pos = c128(probe), i64(g.positions)
    check(L.lib().pdd_illumination_density(ptr(pr), C.c_int64(g.frame_side), ptr(pos), C.c_int64(g.frame_count()),
                                           C.c_int64(g.image_height), C.c_int64(g.image_width), ptr(out), _dt(dtype)))
    return out


def _probe_sums(image, frames, g: ScanGeometry, dtype):
    s = g.frame_side
    num = np.zeros((s, s), np.complex128)
    den = np.zeros((s, s))
    im, pos = c128(image), i64(g.positions)
    fr = None if frames is None else c128(frames)
    check(L.lib().pdd_probe_sums(ptr(im), C.c_int64(g.image_height), C.c_int64(g.image_width), ptr(fr), ptr(pos),
                                 C.c_int64(g.frame_count()), C.c_int64(s), ptr(num), ptr(den), _dt(dtype)))
    return num, den


def probe_density(image: np.ndarray, geometry: ScanGeometry, dtype=None) -> np.ndarray:
    """forward.cpp:68-78."""
    if image.shape != (geometry.image_height, geometry.image_width):
        raise InvalidArgument("forward model: image shape != geometry image_shape")
    return _probe_sums(image, None, geometry, dtype)[1]


def adjoint_probe(image: np.ndarray, frames: np.ndarray, geometry: ScanGeometry, dtype=None) -> np.ndarray:
    """forward.cpp:80-93."""
    if image.shape != (geometry.image_height, geometry.image_width):
        raise InvalidArgument("forward model: image shape != geometry image_shape")
    if frames.shape[0] != geometry.frame_count():
        raise InvalidArgument("forward model: frame count mismatch")
    return _probe_sums(image, frames, geometry, dtype)[0]


def intensity(frames: np.ndarray, dtype=None) -> np.ndarray:
    """forward.cpp:95-106."""
    z = c128(frames)
    out = np.zeros(z.shape)
    check(L.lib().pdd_intensity(ptr(z), C.c_int64(z.size), ptr(out), _dt(dtype)))
    return out


# --------------------------------------------------------------------------- stagm
class stagm:  # noqa: N801 - mirrors the reference namespace
    """stagm.hpp:13-37."""

    @staticmethod
    def check_epsilon(epsilon: float) -> None:
        if not (0.0 < epsilon < 1.0):
            raise InvalidArgument("stagm: epsilon must lie in (0,1)")

    @staticmethod
    def pixel_prox(y, b, lam: float, epsilon: float, dtype=None):
        ya, ba = c128(np.atleast_1d(y)), f64(np.broadcast_to(b, np.shape(np.atleast_1d(y))))
        out = np.zeros_like(ya)
        check(L.lib().pdd_stagm_prox(ptr(ya), ptr(ba), C.c_int64(ya.size), C.c_double(lam), C.c_double(epsilon),
                                     ptr(out), _dt(dtype)))
        return out if np.ndim(y) else out[0]

    prox_pixels = pixel_prox

    @staticmethod
    def prox(y, f, lam: float, epsilon: float, dtype=None):
        """stagm.cpp:101-116 (stack level)."""
        stagm.check_epsilon(epsilon)
        if lam <= 0.0:
            raise InvalidArgument("stagm::prox: lambda must be positive")
        if np.shape(y) != np.shape(f):
            raise InvalidArgument("stagm::prox: frame count mismatch")
        return stagm.pixel_prox(y, f, lam, epsilon, dtype)

    @staticmethod
    def _vg(x, b, epsilon, dtype):
        xa, ba = c128(np.atleast_1d(x)), f64(np.broadcast_to(b, np.shape(np.atleast_1d(x))))
        val = np.zeros(xa.shape)
        grad = np.zeros_like(xa)
        check(L.lib().pdd_stagm_value_gradient(ptr(xa), ptr(ba), C.c_int64(xa.size), C.c_double(epsilon), ptr(val),
                                               ptr(grad), _dt(dtype)))
        return val, grad

    @staticmethod
    def pixel_value(x, b, epsilon: float, dtype=None):
        v = stagm._vg(x, b, epsilon, dtype)[0]
        return v if np.ndim(x) else float(v[0])

    @staticmethod
    def pixel_gradient(x, b, epsilon: float, dtype=None):
        g = stagm._vg(x, b, epsilon, dtype)[1]
        return g if np.ndim(x) else g[0]

    @staticmethod
    def value(z, f, epsilon: float, dtype=None) -> float:
        stagm.check_epsilon(epsilon)
        return float(np.sum(stagm._vg(z, f, epsilon, dtype)[0]))

    @staticmethod
    def gradient(z, f, epsilon: float, dtype=None):
        stagm.check_epsilon(epsilon)
        return stagm._vg(z, f, epsilon, dtype)[1]

    @staticmethod
    def lipschitz_constant(epsilon: float) -> float:
        stagm.check_epsilon(epsilon)
        return 2.0 / epsilon - 1.0


# --------------------------------------------------------------------------- metrics
def r_factor(sub_iterates: Sequence[np.ndarray], frames: np.ndarray, probe: np.ndarray, plan: DecompositionPlan,
             dtype=None) -> float:
    """metrics.cpp:11-27; frames: the global intensity stack [J, s, s]."""
    if len(sub_iterates) != plan.D:
        raise InvalidArgument("r_factor: subdomain count mismatch")
    flat = c128(np.concatenate([c128(u).ravel() for u in sub_iterates]))
    out = C.c_double()
    check(L.lib().pdd_r_factor(plan.handle, ptr(flat), ptr(f64(frames)), ptr(c128(probe)), C.byref(out), _dt(dtype)))
    return out.value


def relative_error(current: Sequence[np.ndarray], previous: Sequence[np.ndarray], dtype=None) -> float:
    """metrics.cpp:29-46."""
    if len(current) != len(previous):
        raise InvalidArgument("relative_error: subdomain count mismatch")
    for a, b in zip(current, previous):
        if np.shape(a) != np.shape(b):
            raise InvalidArgument("relative_error: shape mismatch")
    cur = c128(np.concatenate([c128(a).ravel() for a in current]))
    prev = c128(np.concatenate([c128(a).ravel() for a in previous]))
    sizes = i64([np.size(a) for a in current])
    out = C.c_double()
    check(L.lib().pdd_relative_error(ptr(cur), ptr(prev), C.c_int32(len(current)), ptr(sizes), C.byref(out),
                                     _dt(dtype)))
    return out.value


def snr_db(recovered: np.ndarray, truth: np.ndarray) -> float:
    """metrics.cpp:48-57 (reporting helper; not on the iteration path)."""
    if recovered.shape != truth.shape:
        raise InvalidArgument("snr_db: shape mismatch")
    d = recovered - truth
    diff = float(np.sum(np.abs(d) ** 2))
    ref = float(np.sum(np.abs(recovered) ** 2))
    return math.inf if diff == 0.0 else -10.0 * math.log10(diff / ref)


# --------------------------------------------------------------------------- solvers
@dataclass
class NonblindConfig:
    """solver.hpp:16-28."""

    epsilon: float = 0.5
    eta: float = 0.1
    r: float = 4.0e3
    max_iters: int = 1000
    tol_rf: float = 1.0e-5
    tol_re: float = 1.0e-3
    stop_rule: str = "rfactor"  # "rfactor" | "relative_error"
    record_lagrangian: bool = False
    threads: int = 0

    def c(self) -> L.NonblindConfigC:
        return L.NonblindConfigC(self.epsilon, self.eta, self.r, self.tol_rf, self.tol_re, self.max_iters,
                                 0 if self.stop_rule == "rfactor" else 1, int(self.record_lagrangian), self.threads)


@dataclass
class ConvergenceRecord:
    """solver.hpp:31-39."""

    iteration: int
    rf: float
    re: float
    lagrangian: Optional[float] = None
    t_sub_ms: List[float] = field(default_factory=list)
    t_virtual_ms: float = 0.0
    t_actual_ms: float = 0.0


@dataclass
class SolverState:
    """solver.hpp:44-51; lam[p] = [side d1, side d2]."""

    u: list
    z: list
    gamma: list
    v: list
    lam: list
    iteration: int = 0


def _prefaulted(shape) -> np.ndarray:
    """complex128 array whose pages are already mapped (written once):
    device->host copies into it then run at copy speed instead of at
    page-fault speed."""
    a = np.empty(shape, np.complex128)
    a.fill(0)
    return a


class _Prefault(threading.Thread):
    """Allocates and maps the host result buffers on a helper thread while the
    device loop runs (the C-ABI call releases the GIL).  (Page-locking them
    instead costs more than it saves: cudaMallocHost of 2 GB takes ~0.9 s and
    stalls the device loop.)  It also reserves the library's small page-locked
    staging buffer through which the results are downloaded."""

    def __init__(self, *shapes):
        super().__init__(daemon=True)
        self.shapes, self.out, self.rc = shapes, None, 0

    def run(self):
        # the library's page-locked download staging (a no-op after the first call)
        self.rc = L.lib().pdd_host_stage_reserve()
        self.out = [_prefaulted(sh) for sh in self.shapes]

    def result(self):
        self.join()
        check(self.rc)
        return self.out


class _LazyList(list):
    """A list filled on first access (device -> host download on demand)."""

    def __init__(self, fetch):
        super().__init__()
        self._fetch = fetch
        self._done = False

    def _load(self):
        if not self._done:
            self._done = True
            super().extend(self._fetch())

    def __getitem__(self, i):
        self._load()
        return super().__getitem__(i)

    def __iter__(self):
        self._load()
        return super().__iter__()

    def __len__(self):
        self._load()
        return super().__len__()


@dataclass
class NonblindResult:
    """solver.hpp:53-60."""

    sub_solutions: list
    merged: np.ndarray
    records: List[ConvergenceRecord]
    iterations: int
    final_rf: float
    final_re: float


class _DataArg:
    """Measured data for a solver: intensities (reference semantics) or amplitudes;
    numpy (host) or torch CUDA tensors (device)."""

    def __init__(self, frames=None, amplitudes=None):
        if (frames is None) == (amplitudes is None):
            raise InvalidArgument("give exactly one of frames (intensities) or amplitudes")
        a = frames if frames is not None else amplitudes
        self.path = None
        if frames is not None and isinstance(frames, (str, os.PathLike)):
            # a frames.ptya file: streamed from disk to the device by the library
            from . import ptya

            self.path = os.fsencode(frames)
            self.arr, self.kind, self.on_device = C.c_char_p(self.path), L.DATA_PTYA_FRAMES_F64, False
            self.shape = ptya.header(frames, ptya.F64)[0]
            self._file = frames
            return
        self.on_device = bool(hasattr(a, "is_cuda") and a.is_cuda)
        if self.on_device:
            import torch

            if frames is not None:
                self.arr, self.kind = a.to(torch.float64).contiguous(), L.DATA_INTENSITY_F64
            elif a.dtype == torch.float32:
                self.arr, self.kind = a.contiguous(), L.DATA_AMPLITUDE_F32
            else:
                self.arr, self.kind = a.to(torch.float64).contiguous(), L.DATA_AMPLITUDE_F64
            self.shape = tuple(a.shape)
            # the solver copies on its own stream, which is not ordered after
            # torch's: the producer (and the conversions above) must be done
            # (ptychodd_cuda.h ordering contract for data_on_device)
            torch.cuda.current_stream(a.device).synchronize()
        else:
            if frames is not None:
                self.arr, self.kind = f64(frames), L.DATA_INTENSITY_F64
            elif np.asarray(a).dtype == np.float32:
                self.arr, self.kind = np.ascontiguousarray(a), L.DATA_AMPLITUDE_F32
            else:
                self.arr, self.kind = f64(a), L.DATA_AMPLITUDE_F64
            self.shape = self.arr.shape

    def validate(self, g: ScanGeometry):
        if self.shape != (g.frame_count(), g.frame_side, g.frame_side):
            raise InvalidArgument("FrameStack: frame count != scan position count or frame shape mismatch")

    def host_sqrt(self):
        if self.path is not None:
            from . import ptya

            return np.sqrt(ptya.read_frames(self._file))
        if self.on_device:
            a = self.arr.double().cpu().numpy()
        else:
            a = np.asarray(self.arr, np.float64)
        return np.sqrt(a) if self.kind == L.DATA_INTENSITY_F64 else a


class _SolverBase:
    def _layout(self, get_fn, arrays_fn=None):
        lay = L.LayoutC()
        check(get_fn(self._h, C.byref(lay)))
        self._lay = lay
        n = lay.n_local_sub
        subs = np.zeros(max(n, 1), np.int32)
        hw = np.zeros((max(n, 1), 2), np.int64)
        nfr = np.zeros(max(n, 1), np.int64)
        pairs = np.zeros(max(lay.n_local_pairs, 1), np.int32)
        phw = np.zeros((max(lay.n_local_pairs, 1), 2), np.int64)
        if arrays_fn is not None:
            check(arrays_fn(self._h, ptr(subs), ptr(hw), ptr(nfr), ptr(pairs), ptr(phw)))
        else:  # single rank: derive from the plan
            subs = np.arange(self.plan.D, dtype=np.int32)
            hw = np.array([[s.height(), s.width()] for s in self.plan.subdomains], np.int64)
            nfr = np.array([len(f) for f in self.plan.frames_of], np.int64)
            pairs = np.arange(len(self.plan.overlaps), dtype=np.int32)
            phw = np.array([[o.region.height(), o.region.width()] for o in self.plan.overlaps], np.int64).reshape(-1, 2)
        self.local_subs = [int(x) for x in subs[:n]]
        self.sub_hw = [tuple(int(v) for v in x) for x in hw[:n]]
        self.sub_frames = [int(x) for x in nfr[:n]]
        self.local_pairs = [int(x) for x in pairs[: lay.n_local_pairs]]
        self.pair_hw = [tuple(int(v) for v in x) for x in phw[: lay.n_local_pairs]]

    def _split_images(self, flat):
        out, o = [], 0
        for h, w in self.sub_hw:  # views into the freshly downloaded buffer
            out.append(flat[o : o + h * w].reshape(h, w))
            o += h * w
        return out

    def _split_frames(self, flat):
        s = self.plan.geometry.frame_side
        out, o = [], 0
        for n in self.sub_frames:
            out.append(flat[o : o + n * s * s].reshape(n, s, s).copy())
            o += n * s * s
        return out

    def _split_pairs(self, flat, per=1):
        out, o = [], 0
        for h, w in self.pair_hw:
            grp = []
            for _ in range(per):
                grp.append(flat[o : o + h * w].reshape(h, w).copy())
                o += h * w
            out.append(grp if per > 1 else grp[0])
        return out

    @staticmethod
    def _cat(arrs):
        if not arrs:
            return np.zeros(1, np.complex128)
        return c128(np.concatenate([c128(a).ravel() for a in arrs]))


_RECORD_CB = C.CFUNCTYPE(None, C.c_int64, C.c_double, C.c_double, C.c_double, C.c_double, C.c_void_p)


def _record_callback(on_iteration, n_sub):
    """ctypes trampoline for pdd_*_run_cb: on_iteration(ConvergenceRecord) per
    iteration while the device loop runs (solver.hpp:88).  Exceptions raised by
    the callback are collected and re-raised after the run."""
    errors = []
    if on_iteration is None:
        return _RECORD_CB(0), errors

    def tramp(it, rf, re, t_ms, lag, _user):
        if errors:
            return
        try:
            on_iteration(ConvergenceRecord(int(it), float(rf), float(re), None if math.isnan(lag) else float(lag),
                                           [float(t_ms)] * n_sub, float(t_ms), float(t_ms)))
        except BaseException as e:  # noqa: BLE001 - re-raised by the caller
            errors.append(e)

    return _RECORD_CB(tramp), errors


class NonblindSolver(_SolverBase):
    """solver.hpp:72-107 on the GPU.

    ``dtype``: 'f32' (complex64 compute, float amplitudes) or 'f64'.
    ``rank/world/nccl_id``: rank-sharded multi-GPU mode (subdomain d on rank
    floor(d*world/D)); use paper_2011_00162_b200.dist to bootstrap.
    """

    def __init__(self, plan: DecompositionPlan, frames=None, probe=None, config: Optional[NonblindConfig] = None,
                 pin_ones: Optional[np.ndarray] = None, *, amplitudes=None, dtype=None, device: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 devices: Optional[Sequence[int]] = None):
        self.plan, self.config = plan, config or NonblindConfig()
        g = plan.geometry
        self._data = _DataArg(frames, amplitudes)
        self._data.validate(g)
        self.probe = c128(probe)
        if self.probe.shape != (g.frame_side, g.frame_side):
            raise InvalidArgument("forward model: probe shape != frame_side^2")
        if pin_ones is not None and pin_ones.shape != (g.image_height, g.image_width):
            raise InvalidArgument("NonblindSolver: pin mask shape mismatch")
        self._pin = None if pin_ones is None else f64(pin_ones)
        self.dtype = L.dtype_code(dtype or DEFAULT_DTYPE)
        self.device, self.rank, self.world = device, rank, world
        self._cfg = self.config.c()
        h = C.c_void_p()
        if devices is not None:  # one handle over len(devices) in-process ranks
            devs = (C.c_int32 * len(devices))(*devices)
            check(L.lib().pdd_nonblind_create_multi(plan.handle, ptr(self._data.arr), self._data.kind,
                                                    int(self._data.on_device), ptr(self.probe), C.byref(self._cfg),
                                                    ptr(self._pin), self.dtype, devs, len(devices), C.byref(h)))
        elif world > 1 or nccl_id is not None:
            idb = C.create_string_buffer(bytes(nccl_id), 128)
            check(L.lib().pdd_nonblind_create_rank(plan.handle, ptr(self._data.arr), self._data.kind,
                                                   int(self._data.on_device), ptr(self.probe), C.byref(self._cfg),
                                                   ptr(self._pin), self.dtype, device, rank, world, idb, C.byref(h)))
        else:
            check(L.lib().pdd_nonblind_create(plan.handle, ptr(self._data.arr), self._data.kind,
                                              int(self._data.on_device), ptr(self.probe), C.byref(self._cfg),
                                              ptr(self._pin), self.dtype, device, C.byref(h)))
        self._h = h
        self._layout(L.lib().pdd_nonblind_layout_get, L.lib().pdd_nonblind_layout_arrays)
        self._sqrt_f = None
        self._dev_iter = None  # iteration of the state last produced on the device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            L.lib().pdd_nonblind_destroy(h)
            self._h = None

    # -- state transfer -------------------------------------------------------
    def _get_state(self) -> SolverState:
        lay = self._lay
        u = np.zeros(lay.image_elems, np.complex128)
        z = np.zeros(lay.frame_elems, np.complex128)
        g = np.zeros(lay.frame_elems, np.complex128)
        v = np.zeros(max(lay.v_elems, 1), np.complex128)
        lam = np.zeros(max(lay.lambda_elems, 1), np.complex128)
        it = C.c_int64()
        check(L.lib().pdd_nonblind_get_state(self._h, ptr(u), ptr(z), ptr(g), ptr(v), ptr(lam), C.byref(it)))
        return SolverState(self._split_images(u), self._split_frames(z), self._split_frames(g), self._split_pairs(v),
                           self._split_pairs(lam, 2), int(it.value))

    def _set_state(self, st: SolverState) -> None:
        lam = [x for pair in st.lam for x in pair]
        check(L.lib().pdd_nonblind_set_state(self._h, ptr(self._cat(st.u)), ptr(self._cat(st.z)),
                                             ptr(self._cat(st.gamma)), ptr(self._cat(st.v)), ptr(self._cat(lam)),
                                             C.c_int64(st.iteration)))

    def init_state(self) -> SolverState:
        """solver.cpp:96-116 (z^0 = A u^0 included)."""
        check(L.lib().pdd_nonblind_init_state(self._h))
        st = self._get_state()
        st.z = self._forward_local()
        return st

    def _forward_local(self):
        au = np.zeros(self._lay.frame_elems, np.complex128)
        check(L.lib().pdd_nonblind_forward(self._h, ptr(au)))
        return self._split_frames(au)

    def step(self, state: SolverState, au: list) -> List[float]:
        """solver.cpp:118-205: one iteration in place; au replaced by A u^{n+1}.
        (Correctness path: the state round-trips through host memory.)"""
        t0 = time.perf_counter()
        self._set_state(state)
        check(L.lib().pdd_nonblind_step(self._h, 1))
        new = self._get_state()
        state.u, state.z, state.gamma, state.v, state.lam = new.u, new.z, new.gamma, new.v, new.lam
        state.iteration = new.iteration
        au[:] = self._forward_local()
        dt = (time.perf_counter() - t0) * 1e3
        return [dt for _ in self.local_subs]

    def augmented_lagrangian(self, state: SolverState) -> float:
        """metrics.cpp:73-101 for `state` with au = A u (the solver invariant
        after init_state/step), evaluated on the device in fp64 accumulation."""
        self._set_state(state)
        out = C.c_double()
        check(L.lib().pdd_nonblind_lagrangian(self._h, C.byref(out)))
        return out.value

    def r_factor_of(self, au: list) -> float:
        """solver.cpp:207-214 over host arrays au (as the reference's signature)."""
        if self._sqrt_f is None:
            sf = self._data.host_sqrt()
            self._sqrt_f = [sf[self.plan.frames_of[d]] for d in self.local_subs]
            self._sqrt_f_l1 = float(sum(np.sum(x) for x in self._sqrt_f))
        num = sum(float(np.sum(np.abs(np.abs(a) - s))) for a, s in zip(au, self._sqrt_f))
        return num / self._sqrt_f_l1

    def run(self, on_iteration: Optional[Callable[[ConvergenceRecord], None]] = None) -> NonblindResult:
        """solver.cpp:216-267 (performance path: no per-iteration host round
        trip; on_iteration receives each record while the device loop runs, at
        most one poll window behind it)."""
        cfg = self.config
        n = C.c_int64()
        div = C.c_int64()
        rec = np.zeros((cfg.max_iters, 3))
        g = self.plan.geometry
        pf = _Prefault((g.image_height, g.image_width) if self.world == 1 else (0,), (self._lay.image_elems,))
        pf.start()
        cb, errors = _record_callback(on_iteration, len(self.local_subs))
        rc = L.lib().pdd_nonblind_run_cb(self._h, cb, None, C.byref(n), ptr(rec), C.byref(div))
        merged, u = pf.result()
        check(rc, iteration=int(div.value))
        if errors:
            raise errors[0]
        lag = [None] * int(n.value)
        if cfg.record_lagrangian:  # solver.cpp:258-260, evaluated on the device
            nl = C.c_int64()
            hist = np.zeros(max(int(n.value), 1))
            check(L.lib().pdd_nonblind_lagrangian_history(self._h, ptr(hist), C.c_int64(hist.size), C.byref(nl)))
            lag = [float(x) for x in hist[:int(nl.value)]] + [None] * (int(n.value) - int(nl.value))
        records = []
        for k in range(int(n.value)):
            r = ConvergenceRecord(k + 1, float(rec[k, 0]), float(rec[k, 1]), lag[k],
                                  [float(rec[k, 2])] * len(self.local_subs), float(rec[k, 2]), float(rec[k, 2]))
            records.append(r)
        if self.world == 1:  # merged on the device (ddplan.cpp:104-121)
            check(L.lib().pdd_nonblind_merged(self._h, ptr(merged)))
        else:
            merged = None
        u = self._get_u(u)
        last = records[-1] if records else ConvergenceRecord(0, math.nan, math.nan)
        return NonblindResult(u, merged, records, int(n.value), last.rf, last.re)

    def _get_u(self, out: Optional[np.ndarray] = None) -> list:
        u = np.empty(self._lay.image_elems, np.complex128) if out is None else out
        check(L.lib().pdd_nonblind_get_state(self._h, ptr(u), None, None, None, None, None))
        return self._split_images(u)

    def iterate(self, n: int) -> None:
        """Exactly n device iterations from the current state (benchmark path)."""
        check(L.lib().pdd_nonblind_iterate(self._h, C.c_int32(n)))

    def last_rf(self) -> float:
        out = C.c_double()
        check(L.lib().pdd_nonblind_last_rf(self._h, C.byref(out)))
        return out.value

    def sync(self) -> None:
        check(L.lib().pdd_nonblind_sync(self._h))

    def launches_per_iteration(self) -> int:
        out = C.c_int64()
        check(L.lib().pdd_nonblind_launches_per_iteration(self._h, C.byref(out)))
        return int(out.value)

    def partitioned_frames(self):
        return partition_frames(self._data.arr if not self._data.on_device else self._data.arr.cpu().numpy(),
                                self.plan)


# --------------------------------------------------------------------------- blind (blind.hpp)
@dataclass
class BlindConfig:
    """blind.hpp:7-22."""

    epsilon: float = 0.5
    eta: float = 0.1
    r: float = 5.0e3
    mu: float = 2.0e2
    gamma: float = 1.0e-4
    support_mask: Optional[np.ndarray] = None
    support_energy: float = 0.995
    max_iters: int = 1000
    tol_rf: float = 1.0e-5
    tol_re: float = 1.0e-3
    stop_rule: str = "rfactor"
    threads: int = 0

    def c(self) -> L.BlindConfigC:
        return L.BlindConfigC(self.epsilon, self.eta, self.r, self.mu, self.gamma, self.support_energy, self.tol_rf,
                              self.tol_re, self.max_iters, 0 if self.stop_rule == "rfactor" else 1, self.threads)


@dataclass
class BlindState:
    """blind.hpp:24-34."""

    w: np.ndarray
    w_copies: list
    delta: list
    u: list
    z: list
    gamma: list
    v: list
    lam: list
    iteration: int = 0


@dataclass
class BlindResult:
    """blind.hpp:36-46."""

    probe: np.ndarray
    probe_fourier: np.ndarray
    support_mask: np.ndarray
    sub_solutions: list
    merged: np.ndarray
    records: List[ConvergenceRecord]
    iterations: int
    final_rf: float
    final_re: float


def _freq_radius(side: int) -> np.ndarray:
    k = np.arange(side)
    kk = np.minimum(k, side - k).astype(float)
    return np.sqrt(kk[:, None] ** 2 + kk[None, :] ** 2)


def disk_support_mask(side: int, radius: float) -> np.ndarray:
    """blind.cpp:46-52."""
    return (_freq_radius(side) <= radius).astype(np.float64)


def estimate_support_mask(probe_guess: np.ndarray, energy_fraction: float) -> np.ndarray:
    """blind.cpp:54-75 (spectrum by the GPU FFT)."""
    side = probe_guess.shape[0]
    spec = fft2_normalized(probe_guess)
    e = (np.abs(spec) ** 2).ravel()
    rad = _freq_radius(side).ravel()
    order = np.lexsort((e, rad))
    acc = np.cumsum(e[order])
    hit = np.nonzero(acc >= energy_fraction * float(np.cumsum(e)[-1]))[0]
    return disk_support_mask(side, float(rad[order][hit[0]] if hit.size else rad[order][-1]))


class BlindSolver(_SolverBase):
    """blind.hpp:58-85 on the GPU.  ``init_state(w0)`` optionally replaces the
    amplitude-based initial probe."""

    def __init__(self, plan: DecompositionPlan, frames=None, config: Optional[BlindConfig] = None,
                 pin_ones: Optional[np.ndarray] = None, *, amplitudes=None, dtype=None, device: int = 0,
                 rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 devices: Optional[Sequence[int]] = None):
        self.plan, self.config = plan, config or BlindConfig()
        g = plan.geometry
        s = g.frame_side
        self._data = _DataArg(frames, amplitudes)
        self._data.validate(g)
        m = self.config.support_mask
        if m is not None and np.size(m) > 0 and np.shape(m) != (s, s):
            raise InvalidArgument("BlindConfig: support mask must be frame-sized")
        self._mask = None if (m is None or np.size(m) == 0) else f64(m)
        if pin_ones is not None and pin_ones.shape != (g.image_height, g.image_width):
            raise InvalidArgument("BlindSolver: pin mask shape mismatch")
        self._pin = None if pin_ones is None else f64(pin_ones)
        self.dtype = L.dtype_code(dtype or DEFAULT_DTYPE)
        self.device, self.rank, self.world = device, rank, world
        self._cfg = self.config.c()
        h = C.c_void_p()
        if devices is not None:
            devs = (C.c_int32 * len(devices))(*devices)
            check(L.lib().pdd_blind_create_multi(plan.handle, ptr(self._data.arr), self._data.kind,
                                                 int(self._data.on_device), C.byref(self._cfg), ptr(self._mask),
                                                 ptr(self._pin), self.dtype, devs, len(devices), C.byref(h)))
        elif world > 1 or nccl_id is not None:
            idb = C.create_string_buffer(bytes(nccl_id), 128)
            check(L.lib().pdd_blind_create_rank(plan.handle, ptr(self._data.arr), self._data.kind,
                                                int(self._data.on_device), C.byref(self._cfg), ptr(self._mask),
                                                ptr(self._pin), self.dtype, device, rank, world, idb, C.byref(h)))
        else:
            check(L.lib().pdd_blind_create(plan.handle, ptr(self._data.arr), self._data.kind, int(self._data.on_device),
                                           C.byref(self._cfg), ptr(self._mask), ptr(self._pin), self.dtype, device,
                                           C.byref(h)))
        self._h = h
        self._layout(L.lib().pdd_blind_layout_get, None)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            L.lib().pdd_blind_destroy(h)
            self._h = None

    def _probe_info(self):
        s = self.plan.geometry.frame_side
        probe = np.zeros((s, s), np.complex128)
        spec = np.zeros((s, s), np.complex128)
        mask = np.zeros((s, s))
        w0 = np.zeros((s, s), np.complex128)
        check(L.lib().pdd_blind_get_probe(self._h, ptr(probe), ptr(spec), ptr(mask), ptr(w0)))
        return probe, spec, mask, w0

    def support_mask(self) -> np.ndarray:
        return self._probe_info()[2]

    def initial_probe(self) -> np.ndarray:
        """The solver's amplitude-based w^0 (blind.cpp:123-153)."""
        return self._probe_info()[3]

    def _get_state(self) -> BlindState:
        lay = self._lay
        s = self.plan.geometry.frame_side
        n = lay.n_local_sub
        w = np.zeros((s, s), np.complex128)
        wc = np.zeros((max(n, 1), s, s), np.complex128)
        dl = np.zeros((max(n, 1), s, s), np.complex128)
        u = np.zeros(lay.image_elems, np.complex128)
        z = np.zeros(lay.frame_elems, np.complex128)
        g = np.zeros(lay.frame_elems, np.complex128)
        v = np.zeros(max(lay.v_elems, 1), np.complex128)
        lam = np.zeros(max(lay.lambda_elems, 1), np.complex128)
        it = C.c_int64()
        check(L.lib().pdd_blind_get_state(self._h, ptr(w), ptr(wc), ptr(dl), ptr(u), ptr(z), ptr(g), ptr(v),
                                          ptr(lam), C.byref(it)))
        return BlindState(w, list(wc[:n]), list(dl[:n]), self._split_images(u), self._split_frames(z),
                          self._split_frames(g), self._split_pairs(v), self._split_pairs(lam, 2), int(it.value))

    def _set_state(self, st: BlindState) -> None:
        lam = [x for pair in st.lam for x in pair]
        check(L.lib().pdd_blind_set_state(self._h, ptr(c128(st.w)), ptr(self._cat(st.w_copies)),
                                          ptr(self._cat(st.delta)), ptr(self._cat(st.u)), ptr(self._cat(st.z)),
                                          ptr(self._cat(st.gamma)), ptr(self._cat(st.v)), ptr(self._cat(lam)),
                                          C.c_int64(st.iteration)))

    def init_state(self, w0: Optional[np.ndarray] = None) -> BlindState:
        """blind.cpp:169-192."""
        check(L.lib().pdd_blind_init_state(self._h, ptr(None if w0 is None else c128(w0))))
        st = self._get_state()
        return st

    def step(self, state: BlindState) -> List[float]:
        """blind.cpp:194-296 (state round-trips through host memory)."""
        t0 = time.perf_counter()
        self._set_state(state)
        check(L.lib().pdd_blind_step(self._h, 1))
        new = self._get_state()
        for k in ("w", "w_copies", "delta", "u", "z", "gamma", "v", "lam", "iteration"):
            setattr(state, k, getattr(new, k))
        return [(time.perf_counter() - t0) * 1e3 for _ in self.local_subs]

    def run(self, on_iteration=None, w0: Optional[np.ndarray] = None) -> BlindResult:
        """blind.cpp:298-358 from a fresh init_state (optionally with w0)."""
        check(L.lib().pdd_blind_init_state(self._h, ptr(None if w0 is None else c128(w0))))
        cfg = self.config
        n = C.c_int64()
        div = C.c_int64()
        rec = np.zeros((cfg.max_iters, 3))
        g = self.plan.geometry
        pf = _Prefault((g.image_height, g.image_width) if self.world == 1 else (0,), (self._lay.image_elems,))
        pf.start()
        cb, errors = _record_callback(on_iteration, len(self.local_subs))
        rc = L.lib().pdd_blind_run_cb(self._h, cb, None, C.byref(n), ptr(rec), C.byref(div))
        merged, u = pf.result()
        check(rc, iteration=int(div.value))
        if errors:
            raise errors[0]
        records = []
        for k in range(int(n.value)):
            r = ConvergenceRecord(k + 1, float(rec[k, 0]), float(rec[k, 1]), None,
                                  [float(rec[k, 2])] * len(self.local_subs), float(rec[k, 2]), float(rec[k, 2]))
            records.append(r)
        check(L.lib().pdd_blind_get_state(self._h, None, None, None, ptr(u), None, None, None, None, None))
        u = self._split_images(u)
        probe, spec, mask, _ = self._probe_info()
        if self.world == 1:  # merged on the device (ddplan.cpp:104-121)
            check(L.lib().pdd_blind_merged(self._h, ptr(merged)))
        else:
            merged = None
        last = records[-1] if records else ConvergenceRecord(0, math.nan, math.nan)
        return BlindResult(probe, spec, mask, u, merged, records, int(n.value), last.rf, last.re)

    def iterate(self, n: int) -> None:
        check(L.lib().pdd_blind_iterate(self._h, C.c_int32(n)))

    def launches_per_iteration(self) -> int:
        out = C.c_int64()
        check(L.lib().pdd_blind_launches_per_iteration(self._h, C.byref(out)))
        return int(out.value)
