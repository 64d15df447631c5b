"""B200-native OD²P (arXiv 2011.00162): the overlapping-domain-decomposition
ADMM ptychography iteration as sm_100a CUDA kernels behind a C-ABI
(include/ptychodd_cuda.h), with a Python mirror of the reference ptychodd API.
"""
from ._lib import (LIB_PATH, CudaError, DivergenceError, FormatError, InvalidArgument, OutOfRange, PtychoRuntimeError,
                   exported_symbols, lib)
from .ptychodd import (BlindConfig, BlindResult, BlindSolver, BlindState, ConvergenceRecord, DecompositionPlan, NonblindConfig, NonblindResult, NonblindSolver, Region,
                       ScanGeometry, SolverState, adjoint, adjoint_probe, fft2_normalized, forward, ifft2_normalized,
                       illumination_density, intensity, make_raster_scan, merge, partition_frames, plan_from_arrays, plan_grid,
                       plan_stripes, probe_density, r_factor, relative_error, restrict_overlap, scan_coverage, snr_db,
                       stagm, disk_support_mask, estimate_support_mask)

__all__ = [n for n in dir() if not n.startswith("_")]
