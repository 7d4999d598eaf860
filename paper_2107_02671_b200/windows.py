"""Window functions -- drop-in for ``sincfft.windows`` (reference
``pkg/src/sincfft/windows.py``), sinh kind.

``omega_eval``, ``omega_hat_eval``, ``phi_eval`` and ``phi_hat_eval`` keep the
reference's signatures (``spec``, array or scalar argument; a scalar in gives a
float out) and its closed forms; they are evaluated elementwise on the device
through ``sincfft_window_eval`` (``csrc/window.cu``), not on the host.  The
hot path does not call these: its spread and gather evaluate per-tap
polynomials validated against the same closed form (``csrc/window.cuh``).

``window_kinds()`` names the shapes this backend implements (the north star's
sinh windows); the reference's other three shapes are rejected by
``WindowSpec`` with a ``ParameterError``.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ParameterError
from .nnfft import WINDOW_KINDS, WindowSpec, _default_device

__all__ = ["WindowSpec", "window_kinds", "omega_eval", "omega_hat_eval", "phi_eval",
           "phi_hat_eval"]

_OMEGA, _OMEGA_HAT, _PHI, _PHI_HAT = 0, 1, 2, 3


def window_kinds():
    """Names of the available window shapes (windows.py:41-43)."""
    return WINDOW_KINDS


def _eval(func, spec, x):
    if not isinstance(spec, WindowSpec):
        raise ParameterError("spec must be a WindowSpec")
    _lib.require_gpu()
    arr = np.asarray(x, dtype=float)
    scalar = arr.ndim == 0
    flat = np.ascontiguousarray(arr.ravel())
    out = np.empty_like(flat)
    if flat.size:
        _lib.check(_lib.lib.sincfft_window_eval(
            func, float(spec.beta), int(spec.m), int(spec.n_grid),
            C.c_void_p(flat.ctypes.data), flat.size, C.c_void_p(out.ctypes.data),
            _lib.PTR_HOST, _default_device(None), None))
    return float(out[0]) if scalar else out.reshape(arr.shape)


def omega_eval(spec, x):
    """Shape function ``omega`` at ``x`` (windows.py:106-125)."""
    return _eval(_OMEGA, spec, x)


def omega_hat_eval(spec, v):
    """Fourier transform ``omega_hat`` at ``v`` (windows.py:135-160; all three
    branches: the series near w = 0, I1 for w > 0, J1 for w < 0)."""
    return _eval(_OMEGA_HAT, spec, v)


def phi_eval(spec, t):
    """Grid window ``phi(t) = omega(n_grid t / m)`` (windows.py:212-214)."""
    return _eval(_PHI, spec, t)


def phi_hat_eval(spec, v):
    """``(m / n_grid) omega_hat(m v / n_grid)`` (windows.py:217-220)."""
    return _eval(_PHI_HAT, spec, v)
