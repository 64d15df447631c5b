"""PTYA array files (the reference's on-disk container, proj/src/io.cpp:80-207)
and the dataset / run directories of its CLI (proj/tools/ptychodd_cli.cpp).

Format: b"PTYA", u16 version (1), u16 dtype (1 = float64, 2 = complex128),
u16 ndim (1..4), u64 dims, little-endian row-major payload; writes are atomic
(temporary file + rename, io.cpp:32-42).  Frame stacks handed to a solver are
not read here at all: the solvers stream frames.ptya from disk straight to the
device (PDD_DATA_PTYA_FRAMES_F64, csrc/ptya.cpp).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from typing import Sequence, Tuple

import numpy as np

from . import _lib as L

F64, C128 = 1, 2
_NP = {F64: np.dtype("<f8"), C128: np.dtype("<c16")}


def header(path: str, dtype: int) -> Tuple[Tuple[int, ...], int]:
    """(dims, payload byte offset); validated by the library (io.cpp:95-115)."""
    ndim = C.c_int32()
    dims = (C.c_int64 * 4)()
    off = C.c_int64()
    L.check(L.lib().pdd_ptya_header(os.fsencode(path), C.c_int32(dtype), C.byref(ndim), dims, C.byref(off)))
    return tuple(int(dims[i]) for i in range(ndim.value)), int(off.value)


def _read(path: str, dtype: int, ndim: int) -> np.ndarray:
    dims, off = header(path, dtype)
    if len(dims) != ndim:
        what = {2: "a 2-D " + ("real" if dtype == F64 else "complex") + " array", 3: "a 3-D frame stack"}[ndim]
        raise L.FormatError(f"expected {what} (byte offset 8)")
    n = int(np.prod(dims))
    size = os.path.getsize(path)
    need = off + n * _NP[dtype].itemsize
    if size < need:
        raise L.FormatError(f"truncated PTYA file (byte offset {size})")
    if size > need:
        raise L.FormatError(f"trailing bytes after payload (byte offset {need})")
    return np.fromfile(path, dtype=_NP[dtype], count=n, offset=off).reshape(dims)


def read_real_array(path: str) -> np.ndarray:
    """io.cpp:162-172."""
    return _read(path, F64, 2).astype(np.float64)


def read_complex_array(path: str) -> np.ndarray:
    """io.cpp:174-188."""
    return _read(path, C128, 2).astype(np.complex128)


def read_frames(path: str) -> np.ndarray:
    """io.cpp:190-204 as one [J, s, s] array (for host-side metrics; solvers
    stream the file instead)."""
    return _read(path, F64, 3).astype(np.float64)


def _write(path: str, dtype: int, arr: np.ndarray) -> None:
    arr = np.ascontiguousarray(arr, dtype=_NP[dtype])
    head = b"PTYA" + np.array([1, dtype, arr.ndim], "<u2").tobytes() + np.array(arr.shape, "<u8").tobytes()
    tmp = str(path) + ".tmp"
    with open(tmp, "wb") as f:
        f.write(head)
        arr.tofile(f)
    os.replace(tmp, path)  # atomic_write (io.cpp:32-42)


def write_array(path: str, field: np.ndarray) -> None:
    """io.cpp:136-160: float64 or complex128 2-D field by its numpy dtype."""
    field = np.asarray(field)
    if field.ndim != 2:
        raise L.InvalidArgument("write_array: 2-D field expected")
    _write(path, C128 if np.iscomplexobj(field) else F64, field)


def write_frames(path: str, frames: np.ndarray) -> None:
    """io.cpp:162-175: [J, s, s] float64 stack."""
    frames = np.asarray(frames)
    if frames.ndim != 3 or frames.shape[0] == 0:
        raise L.InvalidArgument("write_frames: empty stack")
    _write(path, F64, frames)


def write_json(path: str, obj) -> None:
    tmp = str(path) + ".tmp"
    with open(tmp, "w") as f:
        f.write(json.dumps(obj, indent=2) + "\n")
    os.replace(tmp, path)


def read_json(path: str):
    with open(path) as f:
        txt = f.read()
    try:
        return json.loads(txt)
    except json.JSONDecodeError as e:
        raise L.FormatError(f"invalid JSON in {path}: {e} (byte offset {e.pos})") from None


def geometry_to_json(g) -> dict:
    """io.cpp:223-233."""
    return {"frame_side": g.frame_side, "step": g.step, "image_height": g.image_height,
            "image_width": g.image_width, "grid_rows": g.grid_rows, "grid_cols": g.grid_cols,
            "positions": [[int(r), int(c)] for r, c in g.positions]}


def geometry_from_json(j: dict):
    """io.cpp:235-251 (then ScanGeometry::validate, scan.cpp:5-16)."""
    from .ptychodd import ScanGeometry

    try:
        pos = np.array([[int(p[0]), int(p[1])] for p in j["positions"]], np.int64).reshape(-1, 2)
        g = ScanGeometry(int(j["frame_side"]), int(j["step"]), int(j["image_height"]), int(j["image_width"]),
                         int(j["grid_rows"]), int(j["grid_cols"]), pos)
    except (KeyError, TypeError, ValueError, IndexError) as e:
        raise L.FormatError(f"bad geometry record: {e} (byte offset 0)") from None
    # ScanGeometry::validate (scan.cpp:5-16)
    if g.frame_side < 1 or g.step < 1:
        raise L.InvalidArgument("ScanGeometry: frame_side, step >= 1")
    if g.step >= g.frame_side:
        raise L.InvalidArgument("ScanGeometry: step must be < frame_side for sufficient overlap")
    if pos.shape[0] == 0:
        raise L.InvalidArgument("ScanGeometry: no scan positions")
    if pos.shape[0] != g.grid_rows * g.grid_cols:
        raise L.InvalidArgument("ScanGeometry: positions do not form the declared raster grid")
    if ((pos < 0).any() or (pos[:, 0] + g.frame_side > g.image_height).any()
            or (pos[:, 1] + g.frame_side > g.image_width).any()):
        raise L.InvalidArgument("ScanGeometry: window outside image bounds")
    return g


def write_convergence_csv(path: str, records: Sequence) -> None:
    """io.cpp:252-268."""
    if not records:
        raise L.InvalidArgument("write_convergence_csv: no records")
    D = len(records[0].t_sub_ms)
    lines = ["iter,rf,re,lagrangian" + "".join(f",t_sub_{d}_ms" for d in range(D)) + ",t_virtual_ms,t_actual_ms"]
    for r in records:
        lag = "" if r.lagrangian is None else repr(float(r.lagrangian))
        subs = "".join("," + repr(float(t)) for t in r.t_sub_ms)
        lines.append(f"{r.iteration},{float(r.rf)!r},{float(r.re)!r},{lag}{subs},{float(r.t_virtual_ms)!r},"
                     f"{float(r.t_actual_ms)!r}")
    tmp = str(path) + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(lines) + "\n")
    os.replace(tmp, path)
