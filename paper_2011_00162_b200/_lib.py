"""ctypes binding of the C-ABI (include/ptychodd_cuda.h) and the error mapping.

The library is built in-tree (``paper_2011_00162_b200/libptychodd_cuda.so``,
see build.py).  There is no fallback: if it is missing or fails to load, every
entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

LIB_PATH = os.environ.get("PDD_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                    "libptychodd_cuda.so")

PDD_F32, PDD_F64 = 1, 2
DATA_INTENSITY_F64, DATA_AMPLITUDE_F32, DATA_AMPLITUDE_F64, DATA_PTYA_FRAMES_F64 = 0, 1, 2, 3


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class OutOfRange(IndexError):
    """std::out_of_range in the reference."""


class PtychoRuntimeError(RuntimeError):
    """std::runtime_error in the reference (e.g. singular illumination)."""


class DivergenceError(RuntimeError):
    """ptychodd::DivergenceError (solver.hpp:62-68)."""

    def __init__(self, iteration: int, msg: str = ""):
        super().__init__(msg or f"solver diverged: non-finite iterate at iteration {iteration}")
        self.iteration = iteration


class CudaError(RuntimeError):
    """CUDA / NCCL failure."""


class FormatError(RuntimeError):
    """ptychodd::FormatError (io.hpp:12-18): malformed or truncated PTYA/JSON input."""


class PlanInfo(C.Structure):
    _fields_ = [("frame_side", C.c_int64), ("step", C.c_int64), ("image_height", C.c_int64),
                ("image_width", C.c_int64), ("grid_rows", C.c_int64), ("grid_cols", C.c_int64),
                ("n_frames", C.c_int64), ("n_sub", C.c_int32), ("n_pairs", C.c_int32)]


class NonblindConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("eta", C.c_double), ("r", C.c_double), ("tol_rf", C.c_double),
                ("tol_re", C.c_double), ("max_iters", C.c_int32), ("stop_rule", C.c_int32),
                ("record_lagrangian", C.c_int32), ("threads", C.c_int32)]


class BlindConfigC(C.Structure):
    _fields_ = [("epsilon", C.c_double), ("eta", C.c_double), ("r", C.c_double), ("mu", C.c_double),
                ("gamma", C.c_double), ("support_energy", C.c_double), ("tol_rf", C.c_double),
                ("tol_re", C.c_double), ("max_iters", C.c_int32), ("stop_rule", C.c_int32),
                ("threads", C.c_int32)]


class LayoutC(C.Structure):
    _fields_ = [("n_local_sub", C.c_int32), ("n_local_pairs", C.c_int32), ("frame_side", C.c_int64),
                ("image_elems", C.c_int64), ("frame_elems", C.c_int64), ("v_elems", C.c_int64),
                ("lambda_elems", C.c_int64)]


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run paper_2011_00162_b200/build.py (no CPU fallback exists)")
        _lib = C.CDLL(LIB_PATH)
        _lib.pdd_last_error.restype = C.c_char_p
    return _lib


def check(rc: int, iteration: int = 0) -> None:
    if rc == 0:
        return
    msg = lib().pdd_last_error().decode(errors="replace")
    if rc == 1:
        raise InvalidArgument(msg)
    if rc == 2:
        raise OutOfRange(msg)
    if rc == 3:
        raise PtychoRuntimeError(msg)
    if rc == 4:
        raise DivergenceError(iteration, msg)
    if rc == 6:
        raise FormatError(msg)
    raise CudaError(msg)


def ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):  # torch tensor
        return C.c_void_p(a.data_ptr())
    if isinstance(a, C.c_char_p):  # a path (PTYA frames)
        return C.cast(a, C.c_void_p)
    return a.ctypes.data_as(C.c_void_p)


def c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def dtype_code(dtype) -> int:
    if dtype in ("f32", "float32", "complex64", np.float32, np.complex64, PDD_F32):
        return PDD_F32
    if dtype in ("f64", "float64", "complex128", np.float64, np.complex128, PDD_F64):
        return PDD_F64
    raise InvalidArgument(f"unknown dtype {dtype!r}")


def exported_symbols():
    """Names declared PDD_API in include/ptychodd_cuda.h (for the export test)."""
    import re

    hdr = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ptychodd_cuda.h")
    with open(hdr) as f:
        return re.findall(r"PDD_API\s+[\w\s\*]*?\b(pdd_\w+)\s*\(", f.read())
