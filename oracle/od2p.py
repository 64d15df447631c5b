"""ORACLE TEST INFRASTRUCTURE — CPU restatement of the reference OD²P path.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` leg may import it.
It restates, in float64 numpy, the reference C++ implementation under
``/root/reference/proj`` (arXiv 2011.00162 "ptychodd"); every function cites the
reference ``file:line`` it follows.  The restatement is pinned against the
compiled, unmodified reference (``oracle/_ref/libptychodd_ref.so``, built by
``oracle/build_ref.sh``) through golden fixtures in ``tests/golden/`` (generated
by ``tests/golden/make_golden.py``) and the reference's own known-answer tests.

Conventions: complex fields are ``complex128`` arrays, row-major like
``ComplexField2D`` (field.hpp:48-91); frame stacks are ``[J, s, s]`` arrays in the
reference frame order; per-pixel accumulation orders follow the reference (ascending
frame index for every overlap-add, ascending pair index for the consensus terms).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class OutOfRange(IndexError):
    """std::out_of_range."""


class DivergenceError(RuntimeError):
    """ptychodd::DivergenceError (solver.hpp:62-68)."""

    def __init__(self, iteration: int):
        super().__init__(f"solver diverged: non-finite iterate at iteration {iteration}")
        self.iteration = iteration


# ----------------------------------------------------------------------------- scan.cpp
@dataclass
class ScanGeometry:
    """scan.hpp:11-28; positions are (row, col) window corners, [J, 2] int64."""

    frame_side: int
    step: int
    image_height: int
    image_width: int
    grid_rows: int
    grid_cols: int
    positions: np.ndarray

    def frame_count(self) -> int:
        return int(self.positions.shape[0])

    def window(self, j: int):
        r, c = (int(v) for v in self.positions[j])
        return (r, r + self.frame_side, c, c + self.frame_side)

    def validate(self) -> None:
        """scan.cpp:5-16."""
        if self.frame_side < 1 or self.step < 1:
            raise InvalidArgument("ScanGeometry: frame_side, step >= 1")
        if self.step >= self.frame_side:
            raise InvalidArgument("ScanGeometry: step must be < frame_side for sufficient overlap")
        if self.frame_count() == 0:
            raise InvalidArgument("ScanGeometry: no scan positions")
        if self.frame_count() != self.grid_rows * self.grid_cols:
            raise InvalidArgument("ScanGeometry: positions do not form the declared raster grid")
        p = self.positions
        if (p < 0).any() or (p[:, 0] + self.frame_side > self.image_height).any() or (
            p[:, 1] + self.frame_side > self.image_width
        ).any():
            raise InvalidArgument("ScanGeometry: window outside image bounds")


def make_raster_scan(image_height: int, image_width: int, frame_side: int, step: int) -> ScanGeometry:
    """scan.cpp:18-34: row-major corners (i*step, j*step), grid (N-s)//step + 1."""
    if frame_side > image_height or frame_side > image_width:
        raise InvalidArgument("make_raster_scan: frame larger than image")
    gr = (image_height - frame_side) // step + 1
    gc = (image_width - frame_side) // step + 1
    ii, jj = np.meshgrid(np.arange(gr, dtype=np.int64), np.arange(gc, dtype=np.int64), indexing="ij")
    pos = np.stack([ii.ravel() * step, jj.ravel() * step], axis=1)
    g = ScanGeometry(frame_side, step, image_height, image_width, gr, gc, pos)
    g.validate()
    return g


def scan_coverage(g: ScanGeometry) -> np.ndarray:
    """scan.cpp:36-44."""
    cov = np.zeros((g.image_height, g.image_width))
    s = g.frame_side
    for r, c in g.positions:
        cov[r : r + s, c : c + s] += 1.0
    return cov


# ----------------------------------------------------------------------------- ddplan.cpp
@dataclass
class OverlapPair:
    d1: int
    d2: int
    region: tuple  # (r0, r1, c0, c1) image coordinates


@dataclass
class DecompositionPlan:
    """ddplan.hpp:12-35."""

    D: int
    geometry: ScanGeometry
    subdomains: List[tuple]
    frame_assignment: np.ndarray
    frames_of: List[np.ndarray]
    overlaps: List[OverlapPair]
    local_geometries: List[ScanGeometry]

    def pair_index(self, a: int, b: int) -> int:
        """ddplan.cpp:7-12."""
        if a > b:
            a, b = b, a
        for p, ov in enumerate(self.overlaps):
            if ov.d1 == a and ov.d2 == b:
                return p
        raise InvalidArgument("DecompositionPlan: subdomains are not neighbors")

    def local_overlap(self, d: int, p: int) -> tuple:
        """ddplan.cpp:14-19."""
        r0, r1, c0, c1 = self.overlaps[p].region
        s = self.subdomains[d]
        return (r0 - s[0], r1 - s[0], c0 - s[2], c1 - s[2])

    def pairs_of(self, d: int) -> List[int]:
        """ddplan.cpp:21-26."""
        return [p for p, ov in enumerate(self.overlaps) if ov.d1 == d or ov.d2 == d]


def _blocks(lines: int, n: int) -> List[int]:
    """ddplan.cpp:38-42: contiguous blocks, earlier blocks take the remainder."""
    base, extra = divmod(lines, n)
    b = [0]
    for i in range(n):
        b.append(b[-1] + base + (1 if i < extra else 0))
    return b


def _intersects(a, b) -> bool:
    return a[0] < b[1] and b[0] < a[1] and a[2] < b[3] and b[2] < a[3]


def _intersection(a, b) -> tuple:
    return (max(a[0], b[0]), min(a[1], b[1]), max(a[2], b[2]), min(a[3], b[3]))


def _finish_plan(g: ScanGeometry, D: int, assign: np.ndarray, local_grid) -> DecompositionPlan:
    """Subdomains, overlaps and local geometries: ddplan.cpp:59-92."""
    frames_of = [np.nonzero(assign == d)[0].astype(np.int64) for d in range(D)]
    s = g.frame_side
    subs = []
    for d in range(D):
        if frames_of[d].size == 0:
            raise InvalidArgument("plan_stripes: empty subdomain")
        p = g.positions[frames_of[d]]
        subs.append((int(p[:, 0].min()), int(p[:, 0].max()) + s, int(p[:, 1].min()), int(p[:, 1].max()) + s))
    overlaps = []
    for d1 in range(D):
        for d2 in range(d1 + 1, D):
            if _intersects(subs[d1], subs[d2]):
                overlaps.append(OverlapPair(d1, d2, _intersection(subs[d1], subs[d2])))
    locals_ = []
    for d in range(D):
        sub = subs[d]
        lp = g.positions[frames_of[d]] - np.array([sub[0], sub[2]], dtype=np.int64)
        lg = ScanGeometry(s, g.step, sub[1] - sub[0], sub[3] - sub[2], local_grid[d][0], local_grid[d][1], lp)
        lg.validate()
        locals_.append(lg)
    return DecompositionPlan(D, g, subs, assign.astype(np.int32), frames_of, overlaps, locals_)


def plan_stripes(g: ScanGeometry, D: int, axis: str = "auto") -> DecompositionPlan:
    """ddplan.cpp:28-94 (axis: 'auto' | 'columns' | 'rows')."""
    g.validate()
    if D < 1:
        raise InvalidArgument("plan_stripes: D must be >= 1")
    if axis == "auto":
        axis = "columns" if g.grid_cols >= g.grid_rows else "rows"
    by_cols = axis == "columns"
    lines = g.grid_cols if by_cols else g.grid_rows
    if D > lines:
        raise InvalidArgument("plan_stripes: D exceeds the scan frame-line count")
    b = _blocks(lines, D)
    j = np.arange(g.frame_count(), dtype=np.int64)
    line = j % g.grid_cols if by_cols else j // g.grid_cols
    assign = np.searchsorted(np.array(b[1:]), line, side="right")
    grid = [((g.grid_rows, b[d + 1] - b[d]) if by_cols else (b[d + 1] - b[d], g.grid_cols)) for d in range(D)]
    return _finish_plan(g, D, assign, grid)


def plan_grid(g: ScanGeometry, Dr: int, Dc: int) -> DecompositionPlan:
    """2-D block plan (extension): the plan_stripes rules
    (ddplan.cpp:28-94) applied to both scan axes; d = block_row*Dc + block_col."""
    g.validate()
    if Dr < 1 or Dc < 1:
        raise InvalidArgument("plan_grid: Dr, Dc must be >= 1")
    if Dr > g.grid_rows or Dc > g.grid_cols:
        raise InvalidArgument("plan_grid: block count exceeds the scan frame-line count")
    rb, cb = _blocks(g.grid_rows, Dr), _blocks(g.grid_cols, Dc)
    j = np.arange(g.frame_count(), dtype=np.int64)
    bi = np.searchsorted(np.array(rb[1:]), j // g.grid_cols, side="right")
    bj = np.searchsorted(np.array(cb[1:]), j % g.grid_cols, side="right")
    grid = [(rb[d // Dc + 1] - rb[d // Dc], cb[d % Dc + 1] - cb[d % Dc]) for d in range(Dr * Dc)]
    return _finish_plan(g, Dr * Dc, bi * Dc + bj, grid)


def restrict_overlap(u_d: np.ndarray, plan: DecompositionPlan, d: int, neighbor: int) -> np.ndarray:
    """ddplan.cpp:96-102."""
    p = plan.pair_index(d, neighbor)
    r0, r1, c0, c1 = plan.local_overlap(d, p)
    return u_d[r0:r1, c0:c1].copy()


def merge(subs: Sequence[np.ndarray], plan: DecompositionPlan) -> np.ndarray:
    """ddplan.cpp:104-121: mean over covering subdomains, vacuum 1 elsewhere."""
    g = plan.geometry
    out = np.zeros((g.image_height, g.image_width), complex)
    cnt = np.zeros((g.image_height, g.image_width))
    for d in range(plan.D):
        r0, r1, c0, c1 = plan.subdomains[d]
        out[r0:r1, c0:c1] += subs[d]
        cnt[r0:r1, c0:c1] += 1.0
    return np.where(cnt > 0, out / np.where(cnt > 0, cnt, 1.0), 1.0 + 0j)


def partition_frames(frames: np.ndarray, plan: DecompositionPlan) -> List[np.ndarray]:
    """ddplan.cpp:123-133."""
    return [frames[plan.frames_of[d]] for d in range(plan.D)]


# ----------------------------------------------------------------------------- fft.cpp
def fft2n(x: np.ndarray) -> np.ndarray:
    """Unitary 2-D DFT, sign -1, scale 1/sqrt(hw): fft.cpp:39-50."""
    return np.fft.fft2(x, axes=(-2, -1), norm="ortho")


def ifft2n(x: np.ndarray) -> np.ndarray:
    """Unitary inverse: fft.cpp:49-62."""
    return np.fft.ifft2(x, axes=(-2, -1), norm="ortho")


# ----------------------------------------------------------------------------- forward.cpp
def _patches(image: np.ndarray, pos: np.ndarray, s: int) -> np.ndarray:
    """extract (field.cpp:5-16) for every window, stacked [J, s, s]."""
    a = np.arange(s)
    return image[pos[:, 0, None, None] + a[None, :, None], pos[:, 1, None, None] + a[None, None, :]]


def forward(probe: np.ndarray, image: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """forward.cpp:28-41: frame j = F(probe o image|window_j)."""
    if probe.shape != (g.frame_side, g.frame_side):
        raise InvalidArgument("forward model: probe shape != frame_side^2")
    if image.shape != (g.image_height, g.image_width):
        raise InvalidArgument("forward model: image shape != geometry image_shape")
    return fft2n(_patches(image, g.positions, g.frame_side) * probe)


def _overlap_add(tiles: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """embed_add (field.cpp:34-45) of each tile, ascending j."""
    out = np.zeros((g.image_height, g.image_width), tiles.dtype)
    s = g.frame_side
    for j, (r, c) in enumerate(g.positions):
        out[r : r + s, c : c + s] += tiles[j]
    return out


def adjoint(probe: np.ndarray, frames: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """forward.cpp:43-54: sum_j S_j^T(conj P o F*(frame_j)), ascending j."""
    if probe.shape != (g.frame_side, g.frame_side):
        raise InvalidArgument("forward model: probe shape != frame_side^2")
    if frames.shape[0] != g.frame_count():
        raise InvalidArgument("forward model: frame count mismatch")
    return _overlap_add(ifft2n(frames) * np.conj(probe), g)


def illumination_density(probe: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """forward.cpp:56-66."""
    n = (probe.real**2 + probe.imag**2)
    return _overlap_add(np.broadcast_to(n, (g.frame_count(),) + n.shape), g)


def probe_density(image: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """forward.cpp:68-78: sum_j |image|window_j|^2, ascending j."""
    p = _patches(image, g.positions, g.frame_side)
    out = np.zeros((g.frame_side, g.frame_side), p.real.dtype)
    for j in range(p.shape[0]):
        out += p[j].real ** 2 + p[j].imag ** 2
    return out


def adjoint_probe(image: np.ndarray, frames: np.ndarray, g: ScanGeometry) -> np.ndarray:
    """forward.cpp:80-93: sum_j conj(image|window_j) o F*(frame_j), ascending j."""
    back = ifft2n(frames)
    p = _patches(image, g.positions, g.frame_side)
    out = np.zeros((g.frame_side, g.frame_side), back.dtype)
    for j in range(p.shape[0]):
        out += np.conj(p[j]) * back[j]
    return out


def intensity(frames: np.ndarray) -> np.ndarray:
    """forward.cpp:95-106."""
    return frames.real**2 + frames.imag**2


# ----------------------------------------------------------------------------- stagm.cpp
def check_epsilon(eps: float) -> None:
    """stagm.cpp:22-25."""
    if not (0.0 < eps < 1.0):
        raise InvalidArgument("stagm: epsilon must lie in (0,1)")


def _mag_obj(m, absy, b, lam, eps):
    """magnitude_objective, stagm.cpp:9-20 (same operation order)."""
    root_b = np.sqrt(b)
    d = m - root_b
    g = np.where(m < eps * root_b, 0.5 * (1.0 - eps) * (b - m * m / eps), 0.5 * d * d)
    e = m - absy
    return g + 0.5 * lam * e * e


def pixel_prox(y, b, lam: float, eps: float):
    """stagm.cpp:45-73, vectorised: outer candidate clamped to eps*sqrt(b), then
    the origin, then the inner stationary point; strict < so ties keep the
    earlier candidate; phase of y with sign(0) := 1."""
    y = np.asarray(y)
    y = y if y.dtype in (np.complex64, np.complex128) else y.astype(complex)
    b = np.asarray(b, np.float32 if y.dtype == np.complex64 else float)
    absy = np.abs(y)
    root_b = np.sqrt(b)
    inner_edge = eps * root_b
    best_m = (root_b + lam * absy) / (1.0 + lam)
    best_m = np.where(best_m < inner_edge, inner_edge, best_m)
    best_obj = _mag_obj(best_m, absy, b, lam, eps)
    o0 = _mag_obj(np.zeros_like(best_m), absy, b, lam, eps)
    take = o0 < best_obj
    best_m = np.where(take, 0.0, best_m)
    best_obj = np.where(take, o0, best_obj)
    inner_coeff = lam - (1.0 - eps) / eps
    if inner_coeff > 0.0:
        mi = lam * absy / inner_coeff
        oi = _mag_obj(mi, absy, b, lam, eps)
        take = (mi < inner_edge) & (oi < best_obj)
        best_m = np.where(take, mi, best_m)
    safe = np.where(absy > 0.0, absy, 1.0)
    phase = np.where(absy > 0.0, y / safe, 1.0 + 0j)
    return phase * best_m


def pixel_value(x, b, eps: float):
    """stagm.cpp:29-35."""
    ax = np.abs(np.asarray(x, complex))
    b = np.asarray(b, float)
    rb = np.sqrt(b)
    d = ax - rb
    return np.where(ax < eps * rb, 0.5 * (1.0 - eps) * (b - ax * ax / eps), 0.5 * d * d)


def pixel_gradient(x, b, eps: float):
    """stagm.cpp:37-43."""
    x = np.asarray(x, complex)
    ax = np.abs(x)
    rb = np.sqrt(np.asarray(b, float))
    inner = (1.0 - 1.0 / eps) * x
    outer = np.where(ax == 0.0, 0.0, (1.0 - rb / np.where(ax == 0.0, 1.0, ax))) * x
    return np.where(ax < eps * rb, inner, outer)


def stagm_value(z: np.ndarray, f: np.ndarray, eps: float) -> float:
    """stagm.cpp:75-85."""
    check_epsilon(eps)
    return float(np.sum(pixel_value(z, f, eps)))


def prox(y: np.ndarray, f: np.ndarray, lam: float, eps: float) -> np.ndarray:
    """stagm.cpp:101-116."""
    check_epsilon(eps)
    if lam <= 0.0:
        raise InvalidArgument("stagm::prox: lambda must be positive")
    return pixel_prox(y, f, lam, eps)


def lipschitz_constant(eps: float) -> float:
    """stagm.cpp:118-121."""
    check_epsilon(eps)
    return 2.0 / eps - 1.0


# ----------------------------------------------------------------------------- solver.cpp
@dataclass
class NonblindConfig:
    """solver.hpp:16-28."""

    epsilon: float = 0.5
    eta: float = 0.1
    r: float = 4.0e3
    max_iters: int = 1000
    tol_rf: float = 1.0e-5
    tol_re: float = 1.0e-3
    stop_rule: str = "rfactor"  # or "relative_error"
    record_lagrangian: bool = False
    threads: int = 0

    def validate(self) -> None:
        """solver.cpp:24-31."""
        check_epsilon(self.epsilon)
        if self.eta <= 0.0 or self.r <= 0.0:
            raise InvalidArgument("NonblindConfig: eta, r must be > 0")
        if self.max_iters < 1:
            raise InvalidArgument("NonblindConfig: max_iters >= 1")
        if self.tol_rf <= 0.0 or self.tol_re <= 0.0:
            raise InvalidArgument("NonblindConfig: tolerances must be > 0")
        if self.threads < 0:
            raise InvalidArgument("NonblindConfig: threads >= 0")


@dataclass
class SolverState:
    """solver.hpp:44-51 (lam[p] = [side d1, side d2])."""

    u: list
    z: list
    gamma: list
    v: list
    lam: list
    iteration: int = 0

    def copy(self) -> "SolverState":
        return SolverState([a.copy() for a in self.u], [a.copy() for a in self.z],
                           [a.copy() for a in self.gamma], [a.copy() for a in self.v],
                           [[a.copy(), b.copy()] for a, b in self.lam], self.iteration)


@dataclass
class ConvergenceRecord:
    iteration: int
    rf: float
    re: float
    lagrangian: Optional[float] = None


def _dtypes(precision: str):
    if precision not in ("f64", "f32"):
        raise InvalidArgument("precision must be 'f64' or 'f32'")
    return (np.float32, np.complex64) if precision == "f32" else (np.float64, np.complex128)


def _local_pins(plan: DecompositionPlan, pin_ones: Optional[np.ndarray]) -> List[np.ndarray]:
    """Uncovered pixels plus the caller's vacuum mask (solver.cpp:43-48,64-69)."""
    g = plan.geometry
    cov = scan_coverage(g)
    if pin_ones is not None and pin_ones.shape != cov.shape:
        raise InvalidArgument("NonblindSolver: pin mask shape mismatch")
    gpin = (cov == 0.0) | ((pin_ones > 0.5) if pin_ones is not None else False)
    return [gpin[r0:r1, c0:c1].copy() for (r0, r1, c0, c1) in plan.subdomains]


def _overlap_penalty(plan: DecompositionPlan, d: int, base: np.ndarray, r: float) -> np.ndarray:
    """denom_ += r per covering pair, ascending p (solver.cpp:57-61, blind.cpp:100-107)."""
    out = base.copy()
    for p in plan.pairs_of(d):
        r0, r1, c0, c1 = plan.local_overlap(d, p)
        out[r0:r1, c0:c1] += r
    return out


def _v_update(state: SolverState, plan: DecompositionPlan) -> None:
    """solver.cpp:141-151."""
    for p, ov in enumerate(plan.overlaps):
        r1 = restrict_overlap(state.u[ov.d1], plan, ov.d1, ov.d2)
        r2 = restrict_overlap(state.u[ov.d2], plan, ov.d2, ov.d1)
        state.v[p] = 0.5 * (r1 + r2 + state.lam[p][0] + state.lam[p][1])


def _lambda_update(state: SolverState, plan: DecompositionPlan) -> None:
    """solver.cpp:182-193."""
    for p, ov in enumerate(plan.overlaps):
        r1 = restrict_overlap(state.u[ov.d1], plan, ov.d1, ov.d2)
        r2 = restrict_overlap(state.u[ov.d2], plan, ov.d2, ov.d1)
        state.lam[p][0] = state.lam[p][0] + (r1 - state.v[p])
        state.lam[p][1] = state.lam[p][1] + (r2 - state.v[p])


def _consensus_terms(plan, d, num, state, r):
    """num += r (v_p - Lambda_{p,side}) over pairs_of(d) ascending (solver.cpp:166-175)."""
    for p in plan.pairs_of(d):
        side = 0 if plan.overlaps[p].d1 == d else 1
        r0, r1, c0, c1 = plan.local_overlap(d, p)
        num[r0:r1, c0:c1] += r * (state.v[p] - state.lam[p][side])
    return num


def _relative_error_solver(u, u_prev) -> float:
    """run(): max_d sqrt(diff)/sqrt(norm) (solver.cpp:229-238)."""
    re = 0.0
    for a, b in zip(u, u_prev):
        dd = a - b
        diff = float(np.sum(dd.real**2 + dd.imag**2))
        norm = float(np.sum(a.real**2 + a.imag**2))
        re = max(re, math.sqrt(diff) / math.sqrt(norm) if norm > 0 else math.inf)
    return re


class NonblindSolver:
    """solver.hpp:72-107 / solver.cpp."""

    def __init__(self, plan: DecompositionPlan, intensities: np.ndarray, probe: np.ndarray,
                 config: NonblindConfig, pin_ones: Optional[np.ndarray] = None, precision: str = "f64"):
        """precision "f32": the same restatement evaluated in numpy float32 /
        complex64 -- not the reference (which is double throughout) but the
        float32 floor: what float32 arithmetic itself makes of these formulas,
        against which a float32 GPU result is judged where cancellation makes
        the 1e-5 bound unattainable (tests/test_configs_gpu.py)."""
        config.validate()
        self.rdt, self.cdt = _dtypes(precision)
        g = plan.geometry
        if intensities.shape != (g.frame_count(), g.frame_side, g.frame_side):
            raise InvalidArgument("FrameStack: frame count or shape mismatch")
        if (intensities < 0).any():
            raise InvalidArgument("FrameStack: negative intensity")
        self.plan, self.probe, self.config = plan, np.asarray(probe, self.cdt), config
        self.frames = partition_frames(np.asarray(intensities, self.rdt), plan)
        self.pin = _local_pins(plan, pin_ones)
        self.denom = []
        for d in range(plan.D):
            dens = illumination_density(self.probe, plan.local_geometries[d])
            self.denom.append(_overlap_penalty(plan, d, config.eta * dens, config.r))
            if ((~self.pin[d]) & (dens <= 0.0)).any():
                raise RuntimeError(f"NonblindSolver: illumination density vanishes inside subdomain {d}")
        self.sqrt_f = [np.sqrt(f) for f in self.frames]
        self.sqrt_f_l1 = float(sum(np.sum(s) for s in self.sqrt_f))
        if self.sqrt_f_l1 <= 0.0:
            raise InvalidArgument("NonblindSolver: all-zero measurements, R-factor undefined")

    def init_state(self) -> SolverState:
        """solver.cpp:96-116."""
        u, z, gamma = [], [], []
        for d in range(self.plan.D):
            lg = self.plan.local_geometries[d]
            u.append(np.ones((lg.image_height, lg.image_width), self.cdt))
            z.append(forward(self.probe, u[-1], lg))
            gamma.append(np.zeros_like(z[-1]))
        v, lam = [], []
        for ov in self.plan.overlaps:
            r1 = restrict_overlap(u[ov.d1], self.plan, ov.d1, ov.d2)
            r2 = restrict_overlap(u[ov.d2], self.plan, ov.d2, ov.d1)
            v.append(0.5 * (r1 + r2))
            lam.append([np.zeros_like(r1), np.zeros_like(r1)])
        return SolverState(u, z, gamma, v, lam, 0)

    def step(self, state: SolverState, au: list) -> None:
        """solver.cpp:118-205: z/Gamma -> v -> u -> Lambda -> A u^{n+1} (au replaced)."""
        cfg, plan = self.config, self.plan
        for d in range(plan.D):
            y = state.gamma[d] + au[d]
            state.z[d] = pixel_prox(y, self.frames[d], cfg.eta, cfg.epsilon)
            state.gamma[d] = y - state.z[d]
        _v_update(state, plan)
        for d in range(plan.D):
            lg = plan.local_geometries[d]
            num = adjoint(self.probe, state.z[d] - state.gamma[d], lg) * cfg.eta
            num = _consensus_terms(plan, d, num, state, cfg.r)
            state.u[d] = np.where(self.pin[d], 1.0 + 0j, num / self.denom[d])
        _lambda_update(state, plan)
        for d in range(plan.D):
            au[d] = forward(self.probe, state.u[d], plan.local_geometries[d])
        state.iteration += 1

    def r_factor_of(self, au: list) -> float:
        """solver.cpp:207-214."""
        num = 0.0
        for d in range(self.plan.D):
            num += float(np.sum(np.abs(np.abs(au[d]) - self.sqrt_f[d])))
        return num / self.sqrt_f_l1

    def run(self, on_iteration=None):
        """solver.cpp:216-267.  Returns (sub_solutions, merged, records)."""
        cfg = self.config
        state = self.init_state()
        au = [z.copy() for z in state.z]
        u_prev = [u.copy() for u in state.u]
        records = []
        for n in range(1, cfg.max_iters + 1):
            self.step(state, au)
            re = _relative_error_solver(state.u, u_prev)
            u_prev = [u.copy() for u in state.u]
            rf = self.r_factor_of(au)
            if not (math.isfinite(rf) and math.isfinite(re)):
                raise DivergenceError(n)
            rec = ConvergenceRecord(n, rf, re)
            if cfg.record_lagrangian:
                rec.lagrangian = augmented_lagrangian(state, au, self.frames, self.plan, cfg.epsilon, cfg.eta, cfg.r)
            if on_iteration:
                on_iteration(rec)
            records.append(rec)
            if (rf <= cfg.tol_rf) if cfg.stop_rule == "rfactor" else (re <= cfg.tol_re):
                break
        return state.u, merge(state.u, self.plan), records


# ----------------------------------------------------------------------------- blind.cpp
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

    def validate(self, s: int) -> None:
        """blind.cpp:30-44."""
        check_epsilon(self.epsilon)
        if self.eta <= 0 or self.r <= 0 or self.mu <= 0 or self.gamma <= 0:
            raise InvalidArgument("BlindConfig: eta, r, mu, gamma must be > 0")
        if self.max_iters < 1:
            raise InvalidArgument("BlindConfig: max_iters >= 1")
        if self.tol_rf <= 0 or self.tol_re <= 0:
            raise InvalidArgument("BlindConfig: tolerances must be > 0")
        if self.support_mask is not None and self.support_mask.size > 0:
            if self.support_mask.shape != (s, s):
                raise InvalidArgument("BlindConfig: support mask must be frame-sized")
            if not np.isin(self.support_mask, (0.0, 1.0)).all():
                raise InvalidArgument("BlindConfig: support mask entries must be 0 or 1")


def _freq_radius(side: int) -> np.ndarray:
    """blind.cpp:22-27."""
    k = np.arange(side)
    kk = np.minimum(k, side - k).astype(float)
    return np.sqrt(kk[:, None] ** 2 + kk[None, :] ** 2)


def disk_support_mask(side: int, radius: float) -> np.ndarray:
    """blind.cpp:46-52."""
    return (_freq_radius(side) <= radius).astype(float)


def estimate_support_mask(probe_guess: np.ndarray, energy_fraction: float) -> np.ndarray:
    """blind.cpp:54-75: sort (radius, energy) pairs, smallest radius reaching the fraction."""
    side = probe_guess.shape[0]
    spec = fft2n(probe_guess)
    e = (spec.real**2 + spec.imag**2).ravel()
    rad = _freq_radius(side).ravel()
    total = float(np.cumsum(e)[-1])
    order = np.lexsort((e, rad))
    acc = np.cumsum(e[order])
    hit = np.nonzero(acc >= energy_fraction * total)[0]
    radius = float(rad[order][hit[0]] if hit.size else rad[order][-1])
    return disk_support_mask(side, radius)


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


class BlindSolver:
    """blind.hpp:58-85 / blind.cpp."""

    def __init__(self, plan: DecompositionPlan, intensities: np.ndarray, config: BlindConfig,
                 pin_ones: Optional[np.ndarray] = None, precision: str = "f64"):
        """precision: see NonblindSolver (w0 and the mask are always built in float64)."""
        self.rdt, self.cdt = _dtypes(precision)
        s = plan.geometry.frame_side
        config.validate(s)
        self.plan, self.config = plan, config
        self.frames = partition_frames(np.asarray(intensities, float), plan)
        self.pin = _local_pins(plan, pin_ones)
        self.rpen = [_overlap_penalty(plan, d, np.zeros((lg.image_height, lg.image_width), self.rdt), config.r)
                     for d, lg in enumerate(plan.local_geometries)]
        self.sqrt_f = [np.sqrt(f) for f in self.frames]
        self.sqrt_f_l1 = float(sum(np.sum(x) for x in self.sqrt_f))
        if self.sqrt_f_l1 <= 0.0:
            raise InvalidArgument("BlindSolver: all-zero measurements")
        # w0: checkerboard-recentred mean back-transform of the amplitudes,
        # rescaled to the largest per-frame flux (blind.cpp:123-153).
        k = np.arange(s)
        cb = np.where((k[:, None] + k[None, :]) % 2 == 0, 1.0, -1.0)
        w0 = np.zeros((s, s), complex)
        count = 0
        flux = 0.0
        for f in self.frames:
            back = ifft2n(np.sqrt(f) * cb)
            for j in range(back.shape[0]):
                w0 += back[j]
                count += 1
            for j in range(f.shape[0]):
                flux = max(flux, float(np.cumsum(f[j].ravel())[-1]))
        w0 /= float(count)
        w0 *= math.sqrt(flux / float(np.sum(w0.real**2 + w0.imag**2)))
        self.w0 = w0
        m = config.support_mask
        self.mask = m.astype(float) if (m is not None and m.size > 0) else estimate_support_mask(w0, config.support_energy)
        self.frames = [f.astype(self.rdt) for f in self.frames]
        self.mask = self.mask.astype(self.rdt)

    def project_support(self, probe: np.ndarray):
        """blind.cpp:159-167 -> (spatial, masked spectrum)."""
        spec = fft2n(probe)
        spec = np.where(self.mask == 0.0, 0.0, spec)
        return ifft2n(spec), spec

    def init_state(self, w_init: Optional[np.ndarray] = None) -> BlindState:
        """blind.cpp:169-192 (w_init: SURVEY.md Appendix A custom initial probe)."""
        w = (self.w0 if w_init is None else np.asarray(w_init)).astype(self.cdt)
        st = BlindState(w, [], [], [], [], [], [], [], 0)
        s = self.plan.geometry.frame_side
        for lg in self.plan.local_geometries:
            st.w_copies.append(w.copy())
            st.delta.append(np.zeros((s, s), self.cdt))
            st.u.append(np.ones((lg.image_height, lg.image_width), self.cdt))
            st.z.append(forward(w, st.u[-1], lg))
            st.gamma.append(np.zeros_like(st.z[-1]))
        for ov in self.plan.overlaps:
            r1 = restrict_overlap(st.u[ov.d1], self.plan, ov.d1, ov.d2)
            r2 = restrict_overlap(st.u[ov.d2], self.plan, ov.d2, ov.d1)
            st.v.append(0.5 * (r1 + r2))
            st.lam.append([np.zeros_like(r1), np.zeros_like(r1)])
        return st

    def step(self, st: BlindState) -> None:
        """blind.cpp:194-296."""
        cfg, plan = self.config, self.plan
        D = plan.D
        avg = np.zeros_like(st.w)
        for d in range(D):
            avg += st.delta[d] + st.w_copies[d]
        avg /= float(D)
        st.w, _ = self.project_support(avg)
        _v_update(st, plan)
        for d in range(D):
            lg = plan.local_geometries[d]
            bn = forward(st.w_copies[d], st.u[d], lg)
            y = st.gamma[d] + bn
            st.z[d] = pixel_prox(y, self.frames[d], cfg.eta, cfg.epsilon)
            st.gamma[d] = y - st.z[d]
            resid = st.z[d] - st.gamma[d]
            num = adjoint_probe(st.u[d], resid, lg)
            den = probe_density(st.u[d], lg)
            st.w_copies[d] = (cfg.eta * num + cfg.mu * (st.w - st.delta[d])) / (cfg.eta * den + cfg.mu)
            num = adjoint(st.w_copies[d], resid, lg) * cfg.eta
            den = illumination_density(st.w_copies[d], lg)
            num = _consensus_terms(plan, d, num, st, cfg.r)
            dd = cfg.eta * den + self.rpen[d] + cfg.gamma
            st.u[d] = np.where(self.pin[d], 1.0 + 0j, (num + cfg.gamma * st.u[d]) / dd)
            st.delta[d] = st.delta[d] + (st.w_copies[d] - st.w)
        _lambda_update(st, plan)
        st.iteration += 1

    def rf_shared(self, st: BlindState) -> float:
        """RF with the shared probe (blind.cpp:320-332)."""
        num = 0.0
        for d in range(self.plan.D):
            bw = forward(st.w, st.u[d], self.plan.local_geometries[d])
            num += float(np.sum(np.abs(np.abs(bw) - self.sqrt_f[d])))
        return num / self.sqrt_f_l1

    def run(self, on_iteration=None, w_init: Optional[np.ndarray] = None):
        """blind.cpp:298-358 -> (u, merged, probe, probe_fourier, records)."""
        cfg = self.config
        st = self.init_state(w_init)
        u_prev = [u.copy() for u in st.u]
        records = []
        for n in range(1, cfg.max_iters + 1):
            self.step(st)
            re = _relative_error_solver(st.u, u_prev)
            u_prev = [u.copy() for u in st.u]
            rf = self.rf_shared(st)
            if not (math.isfinite(rf) and math.isfinite(re)):
                raise DivergenceError(n)
            rec = ConvergenceRecord(n, rf, re)
            if on_iteration:
                on_iteration(rec)
            records.append(rec)
            if (rf <= cfg.tol_rf) if cfg.stop_rule == "rfactor" else (re <= cfg.tol_re):
                break
        probe, spec = self.project_support(st.w)
        return st.u, merge(st.u, self.plan), probe, spec, records


# ----------------------------------------------------------------------------- metrics.cpp
def r_factor(subs: Sequence[np.ndarray], frames: Sequence[np.ndarray], probe: np.ndarray,
             plan: DecompositionPlan) -> float:
    """metrics.cpp:11-27."""
    num = den = 0.0
    for d in range(plan.D):
        au = forward(probe, subs[d], plan.local_geometries[d])
        sf = np.sqrt(frames[d])
        num += float(np.sum(np.abs(np.abs(au) - sf)))
        den += float(np.sum(sf))
    if den <= 0.0:
        raise InvalidArgument("r_factor: all-zero data, metric undefined")
    return num / den


def relative_error(current: Sequence[np.ndarray], previous: Sequence[np.ndarray]) -> float:
    """metrics.cpp:29-46 (sqrt(diff/norm) form)."""
    if len(current) != len(previous):
        raise InvalidArgument("relative_error: subdomain count mismatch")
    worst = 0.0
    for a, b in zip(current, previous):
        if a.shape != b.shape:
            raise InvalidArgument("relative_error: shape mismatch")
        dd = a - b
        diff = float(np.sum(dd.real**2 + dd.imag**2))
        norm = float(np.sum(a.real**2 + a.imag**2))
        if norm <= 0.0:
            raise InvalidArgument("relative_error: zero current norm")
        worst = max(worst, math.sqrt(diff / norm))
    return worst


def snr_db(recovered: np.ndarray, truth: np.ndarray) -> float:
    """metrics.cpp:48-57."""
    dd = recovered - truth
    diff = float(np.sum(dd.real**2 + dd.imag**2))
    ref = float(np.sum(recovered.real**2 + recovered.imag**2))
    return math.inf if diff == 0.0 else -10.0 * math.log10(diff / ref)


def augmented_lagrangian(state: SolverState, au: list, frames: list, plan: DecompositionPlan,
                         eps: float, eta: float, r: float) -> float:
    """metrics.cpp:73-101."""
    total = 0.0
    for d in range(plan.D):
        total += stagm_value(state.z[d], frames[d], eps)
        res = au[d] - state.z[d]
        total += float(np.sum(eta * ((np.conj(state.gamma[d]) * res).real + 0.5 * (res.real**2 + res.imag**2))))
    for p, ov in enumerate(plan.overlaps):
        ds = (ov.d1, ov.d2)
        for side in range(2):
            ru = restrict_overlap(state.u[ds[side]], plan, ds[side], ds[1 - side])
            res = ru - state.v[p]
            total += float(np.sum(r * ((np.conj(state.lam[p][side]) * res).real + 0.5 * (res.real**2 + res.imag**2))))
    return total
