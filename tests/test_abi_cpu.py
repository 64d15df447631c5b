"""Host-side checks (no GPU): the C-ABI library loads and exports every symbol
include/ptychodd_cuda.h declares; the C++ plan layer is bit-exact with the
oracle restatement (and through it with the reference, test_oracle_cpu.py)."""
import ctypes as C

import numpy as np
import pytest

from oracle import od2p as O
import paper_2011_00162_b200 as P
from paper_2011_00162_b200 import _lib as L


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    names = L.exported_symbols()
    assert len(names) >= 50
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_status_codes_and_error_text_without_gpu():
    h = C.c_void_p()
    rc = L.lib().pdd_plan_stripes(C.c_int64(64), C.c_int64(64), C.c_int64(16), C.c_int64(16), C.c_int32(1),
                                  C.c_int32(0), C.byref(h))
    assert rc == 1  # step >= frame_side -> std::invalid_argument
    assert b"step must be < frame_side" in L.lib().pdd_last_error()
    with pytest.raises(P.InvalidArgument):
        P.plan_stripes(P.make_raster_scan(128, 256, 64, 8), 10, "rows")  # test_ddplan.cpp:71


CASES = [(256, 256, 64, 8, D, "auto") for D in (1, 2, 4, 6, 8, 10)] + [
    (512, 512, 64, 16, 2, "auto"), (128, 128, 32, 8, 2, "auto"), (128, 256, 64, 8, 3, "rows"),
    (128, 256, 64, 8, 3, "auto"), (2048, 2048, 128, 32, 8, "rows"), (8192, 8192, 128, 32, 8, "rows"),
    (96, 96, 32, 8, 3, "auto")]


@pytest.mark.parametrize("H,W,s,step,D,axis", CASES)
def test_plan_stripes_bit_exact(H, W, s, step, D, axis):
    p = P.plan_stripes(P.make_raster_scan(H, W, s, step), D, axis)
    o = O.plan_stripes(O.make_raster_scan(H, W, s, step), D, axis)
    _same_plan(p, o)


@pytest.mark.parametrize("H,s,step,Dr,Dc", [(2048, 128, 32, 2, 4), (1024, 64, 16, 4, 2), (256, 32, 8, 2, 2),
                                             (512, 64, 16, 3, 3)])
def test_plan_grid_bit_exact(H, s, step, Dr, Dc):
    p = P.plan_grid(P.make_raster_scan(H, H, s, step), Dr, Dc)
    o = O.plan_grid(O.make_raster_scan(H, H, s, step), Dr, Dc)
    _same_plan(p, o)


def _same_plan(p, o):
    assert p.D == o.D
    assert np.array_equal(p.geometry.positions, o.geometry.positions)
    assert np.array_equal(p.frame_assignment, o.frame_assignment)
    assert [(r.row_start, r.row_end, r.col_start, r.col_end) for r in p.subdomains] == [tuple(x) for x in o.subdomains]
    assert [(ov.d1, ov.d2, (ov.region.row_start, ov.region.row_end, ov.region.col_start, ov.region.col_end))
            for ov in p.overlaps] == [(ov.d1, ov.d2, tuple(ov.region)) for ov in o.overlaps]
    for a, b in zip(p.local_geometries, o.local_geometries):
        assert np.array_equal(a.positions, b.positions)
        assert (a.grid_rows, a.grid_cols, a.image_height, a.image_width) == (b.grid_rows, b.grid_cols,
                                                                             b.image_height, b.image_width)
    for d in range(p.D):
        assert p.pairs_of(d) == o.pairs_of(d)


def test_known_plan_answers():
    # test_ddplan.cpp:9-37
    g = P.make_raster_scan(256, 256, 64, 8)
    assert (g.grid_rows, g.grid_cols, g.frame_count()) == (25, 25, 625)
    plan = P.plan_stripes(g, 2)
    assert plan.local_geometries[0].grid_cols == 13 and plan.local_geometries[1].grid_cols == 12
    assert (plan.subdomains[0].col_end, plan.subdomains[1].col_start) == (160, 104)
    assert plan.overlaps[0].region.width() == 56 and plan.overlaps[0].region.height() == 256
    assert P.plan_stripes(P.make_raster_scan(512, 512, 64, 16), 2).overlaps[0].region.width() == 48
    with pytest.raises(P.InvalidArgument):
        P.plan_stripes(P.make_raster_scan(512, 512, 64, 16), 6).pair_index(0, 5)


def test_merge_restrict_round_trip_exact():
    # test_ddplan.cpp:86-119 (merge runs in the C++ host layer)
    g = P.make_raster_scan(96, 96, 32, 8)
    plan = P.plan_stripes(g, 3)
    rng = np.random.default_rng(1)
    glob = rng.standard_normal((96, 96)) + 1j * rng.standard_normal((96, 96))
    subs = [glob[r.slices()].copy() for r in plan.subdomains]
    for ov in plan.overlaps:
        r1 = P.restrict_overlap(subs[ov.d1], plan, ov.d1, ov.d2)
        assert np.array_equal(r1, glob[ov.region.slices()])
    merged = P.merge(subs, plan)
    assert np.max(np.abs(merged - glob)) < 1e-12


def test_scan_coverage_matches_oracle():
    g = P.make_raster_scan(128, 96, 32, 8)
    assert np.array_equal(P.scan_coverage(g), O.scan_coverage(O.make_raster_scan(128, 96, 32, 8)))
