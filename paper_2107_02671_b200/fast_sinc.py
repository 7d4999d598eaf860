"""Fast discrete sinc transform (Algorithm 6.3 of arXiv 2107.02671) on B200 --
drop-in for ``sincfft.fast_sinc`` (reference: ``pkg/src/sincfft/fast_sinc.py``).

    h(b_l) = sum_k c_k sinc(N pi (b_l - a_k))
           ~ sum_j w_j e^{+pi i N z_j b_l} sum_k c_k e^{-pi i N z_j a_k}

computed as stage 1 (sources -> Chebyshev nodes z/2) -> times w -> stage 3
(Chebyshev nodes -> targets) on the GPU, with the weight multiply fused into
stage 1's gather.  Mode detection, forcing and validation follow the
reference exactly, and so does the route (fast_sinc.py:198-220): a stage runs
as an NNFFT, or -- when its node set is the even grid -- as the classical
NFFT trafo (equispaced sources) / NFFT adjoint (equispaced targets), which
skips one window stage (``paper_2107_02671_b200.nfft``).
"""

from __future__ import annotations

import ctypes as C
import enum
import math

import numpy as np

from . import _lib
from . import bounds as _bounds
from .errors import ParameterError
from .nnfft import NnfftGeometry, WindowSpec, _is_torch, _stream_handle, _default_device
from .quadrature import cc_quadrature

_GRID_TOL = 1e-12


class SincMode(enum.Enum):
    """Which stage runs on an even grid (fast_sinc.py:32-38)."""

    GENERAL = "general"
    EQUISPACED_SOURCES = "equispaced-sources"
    EQUISPACED_TARGETS = "equispaced-targets"
    EQUISPACED_BOTH = "equispaced-both"


_MODE_CODE = {SincMode.GENERAL: 0, SincMode.EQUISPACED_SOURCES: 1,
              SincMode.EQUISPACED_TARGETS: 2, SincMode.EQUISPACED_BOTH: 3}


def _even_bandwidth(N, sigma1, m1):
    """fast_sinc.py:97-107."""
    n_star = int(N) + math.ceil(2 * m1 / sigma1)
    for cand in range(n_star, n_star + 100000):
        n1 = sigma1 * cand
        if abs(n1 - round(n1)) < 1e-9 and round(n1) % 2 == 0:
            return cand
    raise ParameterError(f"no admissible rescaled bandwidth found for sigma1={sigma1}")


def _is_even_grid(nodes, L, scale):
    if nodes.size != L or L % 2:
        return False
    grid = (np.arange(L) - L // 2) / scale
    return bool(np.max(np.abs(nodes - grid)) <= _GRID_TOL)


class SincPlan:
    """Planned fast sinc transform (fast_sinc.py:41-94); the two inner NNFFT
    plans live on the GPU."""

    def __init__(self, handle, N, n, quad, a, b, mode, params, n_star, inner_geometry, device):
        self._h = handle
        self.N = N
        self.n = n
        self.quad = quad
        self.a = a
        self.b = b
        self.L1 = a.size
        self.L2 = b.size
        self.mode = mode
        (self.m1, self.m2, self.sigma1, self.sigma2, self.window1, self.window2) = params
        self.n_star = n_star
        self.inner_geometry = inner_geometry
        self.route = {SincMode.GENERAL: "nnfft/nnfft",
                      SincMode.EQUISPACED_SOURCES: "nfft/nnfft",
                      SincMode.EQUISPACED_TARGETS: "nnfft/adjoint",
                      SincMode.EQUISPACED_BOTH: "nfft/adjoint"}[mode]
        self.device = device

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:
            _lib.lib.sincfft_sinc_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def stage_geometry(self):
        g1, g3 = _lib.Geometry(), _lib.Geometry()
        _lib.check(_lib.lib.sincfft_sinc_plan_geometry(self._h, C.byref(g1), C.byref(g3)))
        conv = lambda g: {f: getattr(g, f) for f, _ in _lib.Geometry._fields_}  # noqa: E731
        return conv(g1), conv(g3)

    def error_bound(self):
        """Closed-form certificate (fast_sinc.py:63-94)."""
        if self.window1 != "sinh" or self.window2 != "sinh":
            raise ParameterError("error_bound: closed-form bounds require sinh windows")
        geo = self.inner_geometry
        epsilon = _bounds.bound_cc_sinc(self.N, self.n / self.N)
        e1 = _bounds.bound_sinh_E(self.m1, self.sigma1)
        e2 = _bounds.bound_sinh_E(self.m2, geo.sigma2)
        hat = _bounds.hat_phi_sinh_at_half(geo.N, self.sigma1, self.m1)
        b_term = e1 + geo.a * e2 / hat
        full = _bounds.bound_fast_sinc(epsilon, e1, e2, geo.a, hat)
        simplified = epsilon + 3.0 * e1 + 3.0 * geo.a * e2 / hat
        return {"epsilon": epsilon, "e1": e1, "e2": e2, "a": geo.a, "hat_phi1_half": hat,
                "b_term": b_term, "full": full, "simplified": simplified,
                "simplified_valid": bool(b_term <= 1.0)}


def sinc_plan(N, a, b, *, n=None, epsilon=None, m1=6, m2=6, sigma1=2.0, sigma2=2.0,
              window1="sinh", window2="sinh", mode=None, device=None):
    """Plan a fast sinc transform of bandwidth N (fast_sinc.py:123-223)."""
    _lib.require_gpu()
    if not isinstance(N, (int, np.integer)) or N <= 0:
        raise ParameterError("sinc_plan: N must be a positive integer")
    a = np.ascontiguousarray(a, dtype=float)
    b = np.ascontiguousarray(b, dtype=float)
    for name, arr in (("a", a), ("b", b)):
        if arr.ndim != 1 or arr.size == 0:
            raise ParameterError(f"sinc_plan: {name} must be a nonempty 1-d array")
        if arr.size % 2:
            raise ParameterError(f"sinc_plan: len({name}) must be even")
        if np.max(np.abs(arr)) > 0.5 + _GRID_TOL:
            raise ParameterError(f"sinc_plan: {name} must lie in [-1/2, 1/2]")
    a = np.clip(a, -0.5, 0.5)
    b = np.clip(b, -0.5, 0.5)
    if n is not None and epsilon is not None:
        raise ParameterError("sinc_plan: pass either n or epsilon, not both")
    if n is None:
        n = _bounds.choose_n(int(N), float(epsilon), shape="pow2") if epsilon is not None \
            else 4 * int(N)
    if not isinstance(n, (int, np.integer)) or n < 2:
        raise ParameterError("sinc_plan: n must be an integer >= 2")
    quad = cc_quadrature(int(n))
    z = quad.points
    sources_grid = _is_even_grid(a, a.size, a.size)
    targets_grid = (b.size == N) and (N % 2 == 0) and _is_even_grid(b, int(N), int(N))
    auto = (SincMode.EQUISPACED_BOTH if sources_grid and targets_grid
            else SincMode.EQUISPACED_SOURCES if sources_grid
            else SincMode.EQUISPACED_TARGETS if targets_grid
            else SincMode.GENERAL)
    if mode is None:
        mode = auto
    else:
        mode = SincMode(mode.value if isinstance(mode, SincMode) else mode)
        if mode in (SincMode.EQUISPACED_SOURCES, SincMode.EQUISPACED_BOTH) and not sources_grid:
            raise ParameterError("sinc_plan: equispaced-sources mode requires a_k = k/L1 on I_L1")
        if mode in (SincMode.EQUISPACED_TARGETS, SincMode.EQUISPACED_BOTH) and not targets_grid:
            raise ParameterError(
                "sinc_plan: equispaced-targets mode requires L2 = N even and b_l = l/N")
    params = (int(m1), int(m2), float(sigma1), float(sigma2), window1, window2)
    n_star = _even_bandwidth(int(N), float(sigma1), int(m1))
    inner = NnfftGeometry.from_parameters(n_star, a.size, z.size, float(sigma1), float(sigma2),
                                          int(m1), int(m2))
    WindowSpec(window1, inner.m1, inner.sigma1, inner.N1)
    WindowSpec(window2, inner.m2, inner.sigma2, inner.N2)
    dev = _default_device(device)
    h = C.c_void_p()
    w = np.ascontiguousarray(quad.weights, dtype=float)
    _lib.check(_lib.lib.sincfft_sinc_plan_create(
        C.byref(h), int(N), n_star, a.size, b.size, int(n),
        C.c_void_p(z.ctypes.data), C.c_void_p(w.ctypes.data),
        C.c_void_p(a.ctypes.data), C.c_void_p(b.ctypes.data),
        float(sigma1), float(sigma2), int(m1), int(m2), _MODE_CODE[mode], _lib.PTR_HOST, dev,
        None))
    return SincPlan(h, int(N), int(n), quad, a, b, mode, params, n_star, inner, dev)


def fast_sinc_transform(plan, c):
    """Apply the planned transform (fast_sinc.py:226-249).  ``c``: (L1,) real
    or complex numpy array, or a CUDA float64/complex128 tensor."""
    if _is_torch(c):
        import torch
        if c.device.type != "cuda" or c.device.index != plan.device:
            raise ParameterError("fast_sinc_transform: tensor must live on the plan's device")
        if tuple(c.shape) != (plan.L1,):
            raise ParameterError(
                f"fast_sinc_transform: expected {plan.L1} coefficients, got {tuple(c.shape)}")
        real = not c.is_complex()
        c = c.to(torch.float64 if real else torch.complex128).contiguous()
        out = torch.empty(plan.L2, dtype=torch.complex128, device=c.device)
        _lib.check(_lib.lib.sincfft_sinc_execute(plan.handle, C.c_void_p(c.data_ptr()), int(real),
                                                 C.c_void_p(out.data_ptr()), _lib.PTR_DEVICE,
                                                 _stream_handle(c)))
        return out
    real = np.isrealobj(c)
    c = np.ascontiguousarray(c, dtype=float if real else complex)
    if c.shape != (plan.L1,):
        raise ParameterError(
            f"fast_sinc_transform: expected {plan.L1} coefficients, got {c.shape}")
    out = np.empty(plan.L2, dtype=complex)
    _lib.check(_lib.lib.sincfft_sinc_execute(plan.handle, C.c_void_p(c.ctypes.data), int(real),
                                             C.c_void_p(out.ctypes.data), _lib.PTR_HOST, None))
    return out
