"""Exact quadratic-cost reference sums on the GPU -- drop-in for
``sincfft.direct`` (reference ``pkg/src/sincfft/direct.py``; SURVEY.md 8f
row f2).

Same names, arguments, validation and messages as the reference.  The sums
run on the device (``csrc/direct.cu``) with the phase carried in two doubles
and compensated accumulation, so they are at least as accurate as the
reference's fixed-order pairwise sums; ``compensated`` is accepted for API
compatibility (the device sum is always compensated).  At configs 3 and 5
these are the only affordable oracles (O(M1 M2) fp64 terms).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ParameterError
from .nnfft import _default_device


def _check_1d(name, arr):
    if arr.ndim != 1 or arr.size == 0:
        raise ParameterError(f"{name} must be a nonempty 1-d array")


def _vp(arr):
    return C.c_void_p(arr.ctypes.data)


def nndft_direct(f, v, x, N, compensated=False, *, device=None):
    """``out_j = sum_k f_k e^{-2 pi i N v_k x_j}`` (direct.py:28-64)."""
    _lib.require_gpu()
    f = np.ascontiguousarray(f, dtype=complex)
    v = np.ascontiguousarray(v, dtype=float)
    x = np.ascontiguousarray(x, dtype=float)
    _check_1d("f", f)
    _check_1d("x", x)
    if v.shape != f.shape:
        raise ParameterError("f and v must have the same length")
    out = np.empty(x.size, dtype=complex)
    _lib.check(_lib.lib.sincfft_nndft_direct(_vp(f), _vp(v), f.size, _vp(x), x.size, int(N),
                                             _vp(out), _lib.PTR_HOST, _default_device(device),
                                             None))
    return out


def ndft_direct(c, x, compensated=False, *, device=None):
    """``sum_{k in I_N} c_k e^{2 pi i k x_j}``, N = len(c) even (direct.py:67-90)."""
    _lib.require_gpu()
    c = np.ascontiguousarray(c, dtype=complex)
    x = np.ascontiguousarray(x, dtype=float)
    _check_1d("c", c)
    _check_1d("x", x)
    if c.size % 2:
        raise ParameterError("ndft_direct: len(c) must be even")
    out = np.empty(x.size, dtype=complex)
    _lib.check(_lib.lib.sincfft_ndft_direct(_vp(c), c.size, _vp(x), x.size, _vp(out),
                                            _lib.PTR_HOST, _default_device(device), None))
    return out


def sinc_transform_direct(c, a, b, N, compensated=False, *, device=None):
    """``sum_k c_k sinc(N pi (b_j - a_k))`` (direct.py:93-112)."""
    _lib.require_gpu()
    c = np.ascontiguousarray(c, dtype=complex)
    a = np.ascontiguousarray(a, dtype=float)
    b = np.ascontiguousarray(b, dtype=float)
    _check_1d("c", c)
    _check_1d("b", b)
    if a.shape != c.shape:
        raise ParameterError("c and a must have the same length")
    out = np.empty(b.size, dtype=complex)
    _lib.check(_lib.lib.sincfft_sinc_direct(_vp(c), _vp(a), c.size, _vp(b), b.size, int(N),
                                            _vp(out), _lib.PTR_HOST, _default_device(device),
                                            None))
    return out
