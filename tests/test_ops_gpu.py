"""GPU operator parity against the oracle (oracle/od2p.py) through the C-ABI.

Mirrors the reference's operator tests (proj/tests/test_field_fft.cpp,
test_forward.cpp, test_stagm.cpp): known answers, identities, and element-wise
agreement with the float64 restatement.  Tolerances: float64 compute <= 1e-10
(relative L2), float32 compute <= 1e-5 (the north-star operator bound).
"""
import numpy as np
import pytest

from tests.helpers import rel_l2
from oracle import od2p as O
import paper_2011_00162_b200 as P

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-10, "f32": 1e-5}


def rfield(shape, seed):
    r = np.random.default_rng(seed)
    return r.standard_normal(shape) + 1j * r.standard_normal(shape)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("s", [2, 4, 8, 16, 32, 64, 128])
def test_fft2_matches_numpy(dtype, s):
    x = rfield((s, s), s)
    assert rel_l2(P.fft2_normalized(x, dtype=dtype), O.fft2n(x)) < TOL[dtype]
    assert rel_l2(P.ifft2_normalized(x, dtype=dtype), O.ifft2n(x)) < TOL[dtype]


@pytest.mark.parametrize("shape", [(16, 12), (4, 5), (8, 8), (3, 7)])
def test_fft2_generic_shapes(shape):
    # test_field_fft.cpp:75-112: Parseval / inversion / direct DFT on non-square grids
    x = rfield(shape, 5)
    fx = P.fft2_normalized(x)
    assert rel_l2(fx, O.fft2n(x)) < 1e-12
    assert rel_l2(P.ifft2_normalized(fx), x) < 1e-12


def test_fft_dc_known_answer():
    # test_field_fft.cpp:89-94: constant (2 - i) on 8x8 -> DC = 8 (2 - i)
    x = np.full((8, 8), 2.0 - 1.0j)
    fx = P.fft2_normalized(x)
    assert abs(fx[0, 0] - (2.0 - 1.0j) * 8.0) < 1e-12
    assert np.abs(fx.ravel()[1:]).max() < 1e-12


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("H,s,step", [(12, 4, 2), (40, 8, 4), (128, 32, 8), (256, 64, 16), (384, 128, 32)])
def test_forward_adjoint_density(dtype, H, s, step):
    g = O.make_raster_scan(H, H, s, step)
    gp = P.make_raster_scan(H, H, s, step)
    probe, img = rfield((s, s), 1), rfield((H, H), 2)
    fr = O.forward(probe, img, g)
    assert rel_l2(P.forward(probe, img, gp, dtype=dtype), fr) < TOL[dtype]
    z = rfield(fr.shape, 3)
    assert rel_l2(P.adjoint(probe, z, gp, dtype=dtype), O.adjoint(probe, z, g)) < TOL[dtype]
    assert rel_l2(P.illumination_density(probe, gp, dtype=dtype), O.illumination_density(probe, g)) < TOL[dtype]
    assert rel_l2(P.probe_density(img, gp, dtype=dtype), O.probe_density(img, g)) < TOL[dtype]
    assert rel_l2(P.adjoint_probe(img, z, gp, dtype=dtype), O.adjoint_probe(img, z, g)) < TOL[dtype]
    assert rel_l2(P.intensity(fr, dtype=dtype), O.intensity(fr)) < TOL[dtype]


def test_adjoint_inner_product_identity():
    # test_forward.cpp:49-58: <A u, z> = <u, A* z>
    g = P.make_raster_scan(12, 12, 4, 2)
    probe, u = rfield((4, 4), 3), rfield((12, 12), 4)
    z = rfield((g.frame_count(), 4, 4), 5)
    lhs = np.vdot(P.forward(probe, u, g), z)
    rhs = np.vdot(u, P.adjoint(probe, z, g))
    assert abs(lhs - rhs) < 1e-10


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_prox_matches_oracle_general_and_fast(dtype):
    rng = np.random.default_rng(11)
    n = 20000
    y = rng.uniform(0, 4, n) * np.exp(1j * rng.uniform(-3.14, 3.14, n))
    b = rng.uniform(0, 4, n)
    for lam, eps in [(0.1, 0.5), (2.0, 0.5), (40.0, 0.3), (0.02, 0.95)]:
        got = P.stagm.pixel_prox(y, b, lam, eps, dtype=dtype)
        assert rel_l2(got, O.pixel_prox(y, b, lam, eps)) < (1e-12 if dtype == "f64" else 1e-5)


def test_prox_sign_zero_known_answer():
    # test_stagm.cpp:125-131
    p = P.stagm.pixel_prox(0.0 + 0.0j, 4.0, 0.01, 0.5)
    assert p.imag == 0.0
    assert abs(p.real - 2.0 / 1.01) < 1e-9


def test_value_gradient_match_oracle():
    rng = np.random.default_rng(3)
    x = rng.uniform(-2, 2, 500) + 1j * rng.uniform(-2, 2, 500)
    b = rng.uniform(0, 4, 500)
    assert np.allclose(P.stagm.pixel_value(x, b, 0.3), O.pixel_value(x, b, 0.3), rtol=1e-12, atol=1e-12)
    assert np.allclose(P.stagm.pixel_gradient(x, b, 0.3), O.pixel_gradient(x, b, 0.3), rtol=1e-12, atol=1e-12)


def test_errors_map_to_reference_exceptions():
    g = P.make_raster_scan(12, 12, 4, 2)
    with pytest.raises(ValueError):
        P.forward(np.ones((3, 3)), np.ones((12, 12)), g)
    with pytest.raises(ValueError):
        P.stagm.prox(np.ones(3), np.ones(3), 0.0, 0.5)
    with pytest.raises(ValueError):
        P.stagm.pixel_prox(np.ones(3), np.ones(3), 1.0, 1.5)
