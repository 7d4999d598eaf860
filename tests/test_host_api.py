"""CPU tests of the host side of the drop-in: C-ABI library load + exports,
geometry/validation rules and messages, quadrature and bound constants
(the reference's own known answers, pkg/tests/test_nnfft.py, test_bounds.py,
test_sinc_approx.py).  No GPU compute is called here."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2107_02671_b200 as sf
from paper_2107_02671_b200 import _lib, bounds
from paper_2107_02671_b200.fast_sinc import _even_bandwidth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "sincfft_b200.h")).read()
    declared = set(re.findall(r"\b(sincfft_[a-z_0-9]+)\s*\(", hdr))
    assert len(declared) >= 14
    lib = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), "ctypes table out of sync with the header"
    assert lib.sincfft_version() == 100


def test_status_mapping():
    with pytest.raises(sf.ParameterError):
        _lib.check(_lib.EPARAM)
    with pytest.raises(sf.PositivityError):
        _lib.check(_lib.EPOSITIVITY)
    with pytest.raises(MemoryError):
        _lib.check(_lib.ENOMEM)
    assert issubclass(sf.ParameterError, ValueError)
    assert issubclass(sf.PositivityError, ArithmeticError)


def test_c_abi_rejects_bad_arguments_without_gpu():
    h = ctypes.c_void_p()
    v = np.zeros(4)
    # sigma1*N odd -> EPARAM from the C geometry check, before any device work
    st = _lib.lib.sincfft_nnfft_plan_create(ctypes.byref(h), 10, 4, 4, 1.5, 2.0, 4, 4,
                                            v.ctypes.data, v.ctypes.data, 0, 0, None)
    assert st == _lib.EPARAM
    assert "even integer" in _lib.last_error()
    st = _lib.lib.sincfft_nnfft_plan_create(ctypes.byref(h), 128, 4, 4, 2.0, 2.0, 4, 4,
                                            v.ctypes.data, v.ctypes.data, 7, 0, None)
    assert st == _lib.EPARAM


def test_geometry_reference_cases(golden):
    geo = sf.NnfftGeometry.from_parameters(128, 64, 48, 2.0, 2.0, 4, 4)
    assert (geo.N1, geo.K, geo.N2, geo.a) == (256, 264, 528, 33 / 32)
    geo = sf.NnfftGeometry.from_parameters(128, 10, 10, 2.0, 1.5, 3, 3)
    assert geo.N2 == 394 and geo.sigma2 == pytest.approx(394 / 262, rel=1e-15)
    assert geo.sigma2_nominal == 1.5
    for N, s1, s2, m1, m2, N1, N2, a, sig1, sig2 in golden("geometry.npz")["rows"]:
        g = sf.NnfftGeometry.from_parameters(int(N), 1, 1, s1, s2, int(m1), int(m2))
        assert (g.N1, g.N2, g.a, g.sigma1, g.sigma2) == (int(N1), int(N2), a, sig1, sig2)


def test_geometry_rejects():
    bad = [(10, 8, 8, 1.5, 2.0, 4, 4), (127, 8, 8, 1.5, 2.0, 4, 4), (128, 8, 8, 1.0, 2.0, 4, 4),
           (128, 0, 8, 2.0, 2.0, 4, 4), (16, 8, 8, 1.25, 1.03125, 2, 3)]
    for args in bad:
        with pytest.raises(sf.ParameterError):
            sf.NnfftGeometry.from_parameters(*args)


def test_rescale_reference_case():
    v = np.array([-0.5, -0.1, 0.0, 0.37, 0.5])
    n_star, vs = sf.rescale_frequencies(100, v, 2.0, 4)
    assert n_star == 104
    assert np.array_equal(vs, v * (100 / 104))
    with pytest.raises(sf.ParameterError):
        sf.rescale_frequencies(100, np.array([0.6]), 2.0, 4)


def test_even_bandwidth_config5():
    assert _even_bandwidth(4096, 2.0, 8) == 4104


def test_window_spec_rules():
    with pytest.raises(sf.ParameterError):
        sf.WindowSpec("sinh", 4, 2.5, 64)
    with pytest.raises(sf.ParameterError):
        sf.WindowSpec("gauss", 4, 2.0, 64)
    with pytest.raises(sf.ParameterError, match="not implemented"):
        sf.WindowSpec("bspline", 4, 2.0, 64)
    assert sf.WindowSpec("sinh", 4, 2.0, 64).beta == pytest.approx(2 * np.pi * 4 * 0.75)


def test_quadrature_reference_values(golden):
    q = sf.cc_quadrature(2)
    assert np.max(np.abs(q.weights - np.array([1 / 6, 2 / 3, 1 / 6]))) <= 1e-15
    g = golden("sinc_cases.npz")
    q = sf.cc_quadrature(16384)
    assert np.array_equal(q.points, g["cc16384_z"])
    assert np.max(np.abs(q.weights - g["cc16384_w"])) <= 1e-16
    for n in (4, 16, 256, 4096):
        assert np.max(np.abs(sf.cc_weights_fast(n) - sf.cc_weights_direct(n))) <= 1e-13
        assert abs(sf.cc_quadrature(n).weights.sum() - 1.0) <= 1e-13


def test_bound_constants():
    # frozen values of the reference tests (pkg/tests/test_bounds.py:13-33)
    assert bounds.bound_nnfft_sinh(1200, 2.0, 2.0, 4, 4) == pytest.approx(0.010918764328663988,
                                                                         rel=1e-12)
    assert bounds.bound_nnfft_sinh(128, 2.0, 2.0, 6, 6) == pytest.approx(4.233675150056723e-07,
                                                                        rel=1e-12)
    assert bounds.bound_sinh_E(6, 2.0) == pytest.approx(9.60421890348206e-10, rel=1e-12)
    assert bounds.choose_n(128, 1e-8) == 512
