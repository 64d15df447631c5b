"""The NCCL-backed solver path on one GPU: a single-rank communicator makes the
solver take every multi-GPU code path (D-vector all-reduces inside the captured
iteration graph, memsets of the reduction vectors, probe-tile all-reduce for the
blind solver).  Results must be bit-identical to the communicator-free solver
-- the GPU-count invariance the design promises."""
import ctypes as C

import numpy as np
import pytest

import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import _lib as L
from tests.golden import cases

pytestmark = pytest.mark.gpu


def _nccl_id():
    buf = C.create_string_buffer(128)
    L.check(L.lib().pdd_nccl_unique_id(buf))
    return bytes(buf.raw)


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_nonblind_nccl_single_rank_bit_identical(dtype):
    N, s, step, D, f, probe = cases.nonblind_inputs()["n96D2"]
    plan = P.plan_stripes(P.make_raster_scan(N, N, s, step), D)
    cfg = P.NonblindConfig(max_iters=12, tol_rf=1e-300)
    a = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype).run()
    b = P.NonblindSolver(plan, f, probe, cfg, dtype=dtype, rank=0, world=1, nccl_id=_nccl_id()).run()
    assert np.array_equal(a.merged, b.merged)
    assert [r.rf for r in a.records] == [r.rf for r in b.records]
    assert [r.re for r in a.records] == [r.re for r in b.records]


def test_blind_nccl_single_rank_bit_identical():
    N, s, step, D, f, w0 = cases.blind_inputs()["b96"]
    plan = P.plan_stripes(P.make_raster_scan(N, N, s, step), D)
    cfg = P.BlindConfig(r=1e3, max_iters=6, tol_rf=1e-300)
    a = P.BlindSolver(plan, f, cfg, dtype="f32").run()
    b = P.BlindSolver(plan, f, cfg, dtype="f32", rank=0, world=1, nccl_id=_nccl_id()).run()
    assert np.array_equal(a.merged, b.merged)
    assert np.array_equal(a.probe, b.probe)
    assert [r.rf for r in a.records] == [r.rf for r in b.records]
