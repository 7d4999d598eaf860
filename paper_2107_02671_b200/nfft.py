"""Classical NFFT and adjoint NFFT on B200 -- drop-in for ``sincfft.nfft``
(reference ``pkg/src/sincfft/nfft.py``).

The forward transform evaluates ``p(x_j) = sum_{k in I_N} c_k e^{2 pi i k x_j}``
by deconvolution on an oversampled grid of ``sigma * N`` points, one FFT and
a short gather around each node; the adjoint is the exact conjugate
transpose of the same three stages.  Same names, signatures, defaults,
validation order, messages and exception classes as the reference; the
stages run on the GPU (``csrc/nfft.cu``, built from the NNFFT's spread,
pruned-DFT and gather kernels).  The reference's plan tables
(``spread_idx``, ``spread_val``, ``hat``) are exported lazily from the
device plan for parity checks.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import ParameterError
from .nnfft import WindowSpec, _default_device, _is_torch, _stream_handle

_DOMAIN_TOL = 1e-12


def _vp(arr):
    return C.c_void_p(arr.ctypes.data)


class NfftPlan:
    """Device-resident plan for one node set (reference ``NfftPlan``,
    nfft.py:18-50): degree, n_over, window, nodes, and -- exported on first
    access -- spread_idx, spread_val (M x 2m) and hat (N)."""

    def __init__(self, handle, degree, n_over, window, nodes, device):
        self._h = handle
        self.degree = degree
        self.n_over = n_over
        self.window = window
        self.nodes = nodes
        self.device = device
        self._tables = None

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:
            _lib.lib.sincfft_nfft_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    @property
    def node_count(self):
        return self.nodes.size

    def _export(self):
        if self._tables is None:
            M, m2 = self.nodes.size, 2 * self.window.m
            idx = np.empty((M, m2), dtype=np.int64)
            val = np.empty((M, m2), dtype=float)
            hat = np.empty(self.degree, dtype=float)
            _lib.check(_lib.lib.sincfft_nfft_export_tables(self._h, _vp(idx), _vp(val),
                                                           _vp(hat)))
            self._tables = (idx, val, hat)
        return self._tables

    @property
    def spread_idx(self):
        return self._export()[0]

    @property
    def spread_val(self):
        return self._export()[1]

    @property
    def hat(self):
        return self._export()[2]

    def backend_geometry(self):
        """FFT realisation of the trafo and adjoint stages."""
        n_over = C.c_int64()
        gt, ga = _lib.Geometry(), _lib.Geometry()
        _lib.check(_lib.lib.sincfft_nfft_plan_geometry(self._h, C.byref(n_over), C.byref(gt),
                                                       C.byref(ga)))
        conv = lambda g: {f: getattr(g, f) for f, _ in _lib.Geometry._fields_}  # noqa: E731
        return {"n_over": n_over.value, "trafo": conv(gt), "adjoint": conv(ga)}


def nfft_plan(N, nodes, *, sigma=2.0, m=4, window="sinh", device=None):
    """Build an :class:`NfftPlan` for polynomial degree ``N`` at ``nodes``
    (nfft.py:53-96).  ``sigma * N`` must be an even integer and
    ``2m <= sigma * N / 2``; nodes must satisfy ``|x| <= 1/2`` (a 1e-12
    overhang is clamped) and are treated 1-periodically."""
    _lib.require_gpu()
    if not isinstance(N, (int, np.integer)) or N <= 0 or N % 2:
        raise ParameterError("nfft_plan: N must be a positive even integer")
    n_over_f = sigma * N
    n_over = int(round(n_over_f))
    if abs(n_over_f - n_over) > 1e-9 or n_over % 2:
        raise ParameterError(f"nfft_plan: sigma*N must be an even integer, got {n_over_f}")
    if 2 * m > n_over // 2:
        raise ParameterError(f"nfft_plan: need 2*m <= sigma*N/2, got 2*{m} > {n_over // 2}")
    x = np.ascontiguousarray(nodes, dtype=float)
    if x.ndim != 1 or x.size == 0:
        raise ParameterError("nfft_plan: nodes must be a nonempty 1-d array")
    if np.max(np.abs(x)) > 0.5 + _DOMAIN_TOL:
        raise ParameterError("nfft_plan: nodes must lie in [-1/2, 1/2]")
    x = np.clip(x, -0.5, 0.5)
    spec = WindowSpec(window, int(m), float(sigma), n_over)
    dev = _default_device(device)
    h = C.c_void_p()
    _lib.check(_lib.lib.sincfft_nfft_plan_create(C.byref(h), int(N), x.size, float(sigma),
                                                 int(m), _vp(x), _lib.PTR_HOST, dev, None))
    return NfftPlan(h, int(N), n_over, spec, x, dev)


def _apply(fn, plan, arr, n_in, n_out, name):
    if _is_torch(arr):
        import torch
        if arr.device.type != "cuda" or arr.device.index != plan.device:
            raise ParameterError(f"{name}: tensor must live on the plan's device")
        if tuple(arr.shape) != (n_in,):
            raise ParameterError(f"{name}: expected {n_in} values, got {tuple(arr.shape)}")
        a = arr.to(torch.complex128).contiguous()
        out = torch.empty(n_out, dtype=torch.complex128, device=a.device)
        _lib.check(fn(plan.handle, C.c_void_p(a.data_ptr()), C.c_void_p(out.data_ptr()),
                      _lib.PTR_DEVICE, _stream_handle(a)))
        return out
    a = np.ascontiguousarray(arr, dtype=complex)
    if a.shape != (n_in,):
        raise ParameterError(f"{name}: expected {n_in} {'coefficients' if name == 'nfft_trafo' else 'values'}, got {a.shape}")
    out = np.empty(n_out, dtype=complex)
    _lib.check(fn(plan.handle, _vp(a), _vp(out), _lib.PTR_HOST, None))
    return out


def nfft_trafo(plan, c):
    """Evaluate ``sum_{k in I_N} c_k e^{2 pi i k x_j}`` for all plan nodes
    (nfft.py:99-109)."""
    return _apply(_lib.lib.sincfft_nfft_trafo, plan, c, plan.degree, plan.node_count,
                  "nfft_trafo")


def nfft_adjoint(plan, y):
    """Adjoint: ``h_k = sum_j y_j e^{-2 pi i k x_j}`` on ``I_N`` (nfft.py:112-123),
    the exact conjugate transpose of :func:`nfft_trafo` stage by stage."""
    return _apply(_lib.lib.sincfft_nfft_adjoint, plan, y, plan.node_count, plan.degree,
                  "nfft_adjoint")
