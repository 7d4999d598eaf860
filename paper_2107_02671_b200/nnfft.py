"""NNFFT (Algorithm 2.1 of arXiv 2107.02671) on B200 -- drop-in for
``sincfft.nnfft`` (reference: ``pkg/src/sincfft/nnfft.py``).

Same names, signatures, defaults, validation order, messages and exception
classes as the reference; the plan and the transform run in the CUDA library
(``include/sincfft_b200.h``) -- there is no CPU path.

Extensions (additive): ``nnfft_trafo`` accepts ``f`` of shape ``(M1, B)``
(B columns sharing one plan, the reference applied column by column), and
CUDA ``torch.Tensor`` inputs/outputs (device pointers, current stream).
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ParameterError, PositivityError  # noqa: F401  (re-exported)

_DOMAIN_TOL = 1e-12  # nnfft.py:25
_SIGMA_TOL = 1e-9    # windows.py:37
WINDOW_KINDS = ("sinh",)


@dataclass(frozen=True)
class WindowSpec:
    """Window description (reference ``windows.WindowSpec``, windows.py:46-98);
    the B200 backend implements the sinh shape only (north star)."""

    kind: str
    m: int
    sigma: float
    n_grid: int

    def __post_init__(self):
        if self.kind not in ("sinh", "bspline", "algebraic", "kaiser-bessel"):
            raise ParameterError(
                f"unknown window kind {self.kind!r}; expected one of "
                "('sinh', 'bspline', 'algebraic', 'kaiser-bessel')")
        if self.kind != "sinh":
            raise ParameterError(
                f"window kind {self.kind!r} is not implemented by the B200 backend "
                "(sinh windows only)")
        if not isinstance(self.m, (int, np.integer)) or self.m < 2:
            raise ParameterError("window cut-off m must be an integer >= 2")
        if not self.sigma > 1.0:
            raise ParameterError("window oversampling sigma must be > 1")
        if not (1.25 - _SIGMA_TOL <= self.sigma <= 2.0 + _SIGMA_TOL):
            raise ParameterError(
                f"sinh window requires 5/4 <= sigma <= 2, got sigma={self.sigma}")
        if (not isinstance(self.n_grid, (int, np.integer))
                or self.n_grid <= 0 or self.n_grid % 2):
            raise ParameterError("n_grid must be a positive even integer")
        if 2 * self.m > self.n_grid:
            raise ParameterError(
                f"window needs 2*m <= n_grid, got m={self.m}, n_grid={self.n_grid}")

    @property
    def beta(self):
        return 2.0 * np.pi * self.m * (1.0 - 1.0 / (2.0 * self.sigma))


@dataclass(frozen=True)
class NnfftGeometry:
    """Grid sizes of one NNFFT configuration (nnfft.py:30-89)."""

    N: int
    M1: int
    M2: int
    sigma1: float
    sigma2: float
    m1: int
    m2: int
    N1: int
    N2: int
    a: float
    sigma2_nominal: float

    @classmethod
    def from_parameters(cls, N, M1, M2, sigma1, sigma2, m1, m2):
        if not isinstance(N, (int, np.integer)) or N <= 0:
            raise ParameterError("N must be a positive integer")
        for name, val in (("M1", M1), ("M2", M2)):
            if not isinstance(val, (int, np.integer)) or val <= 0:
                raise ParameterError(f"{name} must be a positive integer")
        for name, val in (("m1", m1), ("m2", m2)):
            if not isinstance(val, (int, np.integer)) or val < 2:
                raise ParameterError(f"{name} must be an integer >= 2")
        if not sigma1 > 1.0 or not sigma2 > 1.0:
            raise ParameterError("sigma1 and sigma2 must be > 1")
        prod = sigma1 * N
        N1 = int(round(prod))
        if abs(prod - N1) > 1e-9 or N1 % 2:
            raise ParameterError(f"sigma1*N must be an even integer, got {prod}")
        if 2 * m1 > N1 // 2:
            raise ParameterError(f"need 2*m1 <= N1/2, got 2*{m1} > {N1 // 2}")
        K = N1 + 2 * m1
        prod2 = sigma2 * K
        N2 = int(round(prod2))
        if abs(prod2 - N2) > 1e-9:
            N2 = math.ceil(prod2)
        N2 += N2 % 2
        limit = (1.0 - N / N1) * N2
        if 2 * m2 > limit + 1e-9:
            raise ParameterError(f"need 2*m2 <= (1 - 1/sigma1)*N2, got 2*{m2} > {limit:g}")
        return cls(int(N), int(M1), int(M2), N1 / N, N2 / K, int(m1), int(m2),
                   N1, N2, K / N1, float(sigma2))

    @property
    def K(self):
        return self.N1 + 2 * self.m1


def rescale_frequencies(N, v, sigma1, m1):
    """Map frequencies on [-1/2, 1/2] into the admissible band (nnfft.py:110-128):
    ``N* = N + ceil(2 m1/sigma1)``, ``v* = v * (N/N*)``."""
    if not isinstance(N, (int, np.integer)) or N <= 0:
        raise ParameterError("rescale_frequencies: N must be a positive integer")
    if not sigma1 > 1.0:
        raise ParameterError("rescale_frequencies: sigma1 must be > 1")
    if not isinstance(m1, (int, np.integer)) or m1 < 2:
        raise ParameterError("rescale_frequencies: m1 must be an integer >= 2")
    arr = np.asarray(v, dtype=float)
    if arr.size and np.max(np.abs(arr)) > 0.5 + _DOMAIN_TOL:
        raise ParameterError("rescale_frequencies: frequencies must lie in [-1/2, 1/2]")
    n_star = int(N) + math.ceil(2 * m1 / sigma1)
    return n_star, arr * (N / n_star)


# ------------------------------------------------------------------ helpers
def _is_torch(a):
    return type(a).__module__.startswith("torch")


def _stream_handle(dev_tensor):
    import torch
    return C.c_void_p(torch.cuda.current_stream(dev_tensor.device).cuda_stream)


def _vp(arr):
    return C.c_void_p(arr.ctypes.data)


class NnfftPlan:
    """Device-resident plan (reference ``NnfftPlan``, nnfft.py:92-107).

    Holds the sorted/binned nodes, the phi_hat tables and the FFT tables on the
    GPU.  The reference's M x 2m step-0 tables (``spread_idx``,
    ``spread_val``, ``gather_idx``, ``gather_val``) and ``hat1``/``hat2``
    are materialised on first access from the device plan (the kernels never
    read them; they evaluate windows from per-tap polynomials).
    """

    def __init__(self, handle, geometry, window1, window2, v, x, device):
        self._h = handle
        self.geometry = geometry
        self.window1 = window1
        self.window2 = window2
        # host copies of the clipped nodes (the reference's plan.v / plan.x):
        # numpy inputs are clipped on first access (the device clips its own
        # copy), so a plan does not pay two M-sized host passes it may never use
        self._v, self._x = v, x
        self._vlim = None
        self.device = device
        self._tables = None
        g = _lib.Geometry()
        _lib.check(_lib.lib.sincfft_nnfft_plan_geometry(self._h, C.byref(g)))
        self.backend_geometry = {f: getattr(g, f) for f, _ in _lib.Geometry._fields_}

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and _lib is not None and getattr(_lib, "lib", None) is not None:
            _lib.lib.sincfft_nnfft_plan_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def _clip_host(self):
        if self._vlim is not None:
            self._v = np.clip(self._v, -self._vlim, self._vlim)
            self._x = np.clip(self._x, -0.5, 0.5)
            self._vlim = None

    @property
    def v(self):
        self._clip_host()
        return self._v

    @property
    def x(self):
        self._clip_host()
        return self._x

    def _export(self):
        if self._tables is None:
            geo = self.geometry
            K = geo.N1 + 2 * geo.m1
            si = np.empty((geo.M1, 2 * geo.m1), np.int64)
            sv = np.empty((geo.M1, 2 * geo.m1), np.float64)
            gi = np.empty((geo.M2, 2 * geo.m2), np.int64)
            gv = np.empty((geo.M2, 2 * geo.m2), np.float64)
            h1 = np.empty(geo.M2, np.float64)
            h2 = np.empty(K, np.float64)
            _lib.check(_lib.lib.sincfft_nnfft_export_tables(
                self._h, _vp(si), _vp(sv), _vp(gi), _vp(gv), _vp(h1), _vp(h2)))
            self._tables = (si, sv, gi, gv, h1, h2)
        return self._tables

    spread_idx = property(lambda self: self._export()[0])
    spread_val = property(lambda self: self._export()[1])
    gather_idx = property(lambda self: self._export()[2])
    gather_val = property(lambda self: self._export()[3])
    hat1 = property(lambda self: self._export()[4])
    hat2 = property(lambda self: self._export()[5])


def nnfft_plan(N, v, x, *, sigma1=2.0, sigma2=2.0, m1=4, m2=4,
               window1="sinh", window2="sinh", device=None, h_window="data"):
    """Build an :class:`NnfftPlan` (reference nnfft.py:131-207).

    ``v``/``x`` may be numpy arrays (copied to the GPU) or CUDA float64 torch
    tensors (validated and clipped on the device).  ``device`` selects the
    GPU (default: the tensor's device, else the current torch device or 0).
    ``h_window`` (additive): "data" sizes the FFT output window from the
    targets (default), "full" from the geometry, so plans over different
    target shards of one problem share one FFT (the distributed FFT of
    ``sharding.DistributedFftNnfft`` requires it).
    """
    _lib.require_gpu()
    if h_window not in ("data", "full"):
        raise ParameterError("nnfft_plan: h_window must be 'data' or 'full'")
    flags = _lib.PLAN_FULL_WINDOW if h_window == "full" else 0
    if _is_torch(v) or _is_torch(x):
        return _plan_from_torch(N, v, x, sigma1, sigma2, m1, m2, window1, window2, device,
                                flags)
    v = np.ascontiguousarray(v, dtype=float)
    x = np.ascontiguousarray(x, dtype=float)
    if v.ndim != 1 or v.size == 0:
        raise ParameterError("nnfft_plan: v must be a nonempty 1-d array")
    if x.ndim != 1 or x.size == 0:
        raise ParameterError("nnfft_plan: x must be a nonempty 1-d array")
    geo = NnfftGeometry.from_parameters(N, v.size, x.size, float(sigma1), float(sigma2),
                                        int(m1), int(m2))
    vmax = 0.5 / geo.a
    # max |.| without an M-sized temporary (same NaN behaviour as np.max(np.abs(.)))
    if _absmax(v) > vmax + _DOMAIN_TOL:
        raise ParameterError(
            "nnfft_plan: frequencies exceed 1/(2a) = {:.6g}; apply "
            "rescale_frequencies to map [-1/2, 1/2] data into the band".format(vmax))
    if _absmax(x) > 0.5 + _DOMAIN_TOL:
        raise ParameterError("nnfft_plan: spatial nodes must lie in [-1/2, 1/2]")
    w1 = WindowSpec(window1, geo.m1, geo.sigma1, geo.N1)
    w2 = WindowSpec(window2, geo.m2, geo.sigma2, geo.N2)
    dev = _default_device(device)
    h = C.c_void_p()
    _lib.check(_lib.lib.sincfft_nnfft_plan_create_ex(
        C.byref(h), geo.N, geo.M1, geo.M2, float(sigma1), float(sigma2), geo.m1, geo.m2,
        _vp(v), _vp(x), _lib.PTR_HOST, dev, flags, None))
    plan = NnfftPlan(h, geo, w1, w2, v, x, dev)
    plan._vlim = vmax  # host copies clipped lazily (NnfftPlan.v / .x)
    return plan


def _absmax(a):
    hi, lo = a.max(), a.min()
    return hi if hi != hi or lo != lo or hi >= -lo else -lo


def _default_device(device):
    if device is not None:
        return int(device)
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except ImportError:  # pragma: no cover
        pass
    return 0


def _plan_from_torch(N, v, x, sigma1, sigma2, m1, m2, window1, window2, device, flags=0):
    import torch
    if not (isinstance(v, torch.Tensor) and isinstance(x, torch.Tensor)):
        raise ParameterError("nnfft_plan: pass both v and x as CUDA tensors (or both as arrays)")
    if v.device != x.device or v.device.type != "cuda":
        raise ParameterError("nnfft_plan: v and x must be CUDA tensors on one device")
    if v.ndim != 1 or v.numel() == 0:
        raise ParameterError("nnfft_plan: v must be a nonempty 1-d array")
    if x.ndim != 1 or x.numel() == 0:
        raise ParameterError("nnfft_plan: x must be a nonempty 1-d array")
    v = v.to(torch.float64).contiguous()
    x = x.to(torch.float64).contiguous()
    geo = NnfftGeometry.from_parameters(N, v.numel(), x.numel(), float(sigma1), float(sigma2),
                                        int(m1), int(m2))
    w1 = WindowSpec(window1, geo.m1, geo.sigma1, geo.N1)
    w2 = WindowSpec(window2, geo.m2, geo.sigma2, geo.N2)
    dev = v.device.index if device is None else int(device)
    h = C.c_void_p()
    # the C side checks the band (message names rescale_frequencies) and clips
    _lib.check(_lib.lib.sincfft_nnfft_plan_create_ex(
        C.byref(h), geo.N, geo.M1, geo.M2, float(sigma1), float(sigma2), geo.m1, geo.m2,
        C.c_void_p(v.data_ptr()), C.c_void_p(x.data_ptr()), _lib.PTR_DEVICE, dev, flags,
        _stream_handle(v)))
    return NnfftPlan(h, geo, w1, w2, None, None, dev)


def nnfft_trafo(plan, f):
    """Evaluate ``sum_k f_k e^{-2 pi i N v_k x_j}`` at all plan nodes
    (reference nnfft.py:210-243).  ``f``: shape (M1,) or (M1, B)."""
    geo = plan.geometry
    if _is_torch(f):
        return _trafo_torch(plan, f)
    f = np.ascontiguousarray(f, dtype=complex)
    if f.shape == (geo.M1,):
        batch = 1
        out = np.empty(geo.M2, dtype=complex)
    elif f.ndim == 2 and f.shape[0] == geo.M1 and f.shape[1] >= 1:
        batch = f.shape[1]
        out = np.empty((geo.M2, batch), dtype=complex)
    else:
        raise ParameterError(f"nnfft_trafo: expected {geo.M1} coefficients, got {f.shape}")
    _lib.check(_lib.lib.sincfft_nnfft_execute(plan.handle, _vp(f), _vp(out), batch,
                                              _lib.PTR_HOST, None))
    return out


def _trafo_torch(plan, f):
    import torch
    geo = plan.geometry
    if f.device.type != "cuda" or f.device.index != plan.device:
        raise ParameterError("nnfft_trafo: tensor must live on the plan's CUDA device")
    f = f.to(torch.complex128).contiguous()
    if tuple(f.shape) == (geo.M1,):
        batch, oshape = 1, (geo.M2,)
    elif f.ndim == 2 and f.shape[0] == geo.M1:
        batch, oshape = f.shape[1], (geo.M2, f.shape[1])
    else:
        raise ParameterError(f"nnfft_trafo: expected {geo.M1} coefficients, got {tuple(f.shape)}")
    out = torch.empty(oshape, dtype=torch.complex128, device=f.device)
    _lib.check(_lib.lib.sincfft_nnfft_execute(plan.handle, C.c_void_p(f.data_ptr()),
                                              C.c_void_p(out.data_ptr()), batch,
                                              _lib.PTR_DEVICE, _stream_handle(f)))
    return out


def nnfft_adjoint(plan, y):
    """Adjoint NNFFT: ``sum_j y_j e^{+2 pi i N v_k x_j}`` at every frequency
    node, the exact conjugate transpose of :func:`nnfft_trafo` on the same
    plan (BASELINE north star's adjoint-NNFFT entry point; not in the
    reference).  ``y``: shape (M2,) or (M2, B), numpy or
    CUDA tensor; returns shape (M1,) or (M1, B)."""
    geo = plan.geometry
    if _is_torch(y):
        import torch
        if y.device.type != "cuda" or y.device.index != plan.device:
            raise ParameterError("nnfft_adjoint: tensor must live on the plan's CUDA device")
        y = y.to(torch.complex128).contiguous()
        if tuple(y.shape) == (geo.M2,):
            batch, oshape = 1, (geo.M1,)
        elif y.ndim == 2 and y.shape[0] == geo.M2:
            batch, oshape = y.shape[1], (geo.M1, y.shape[1])
        else:
            raise ParameterError(f"nnfft_adjoint: expected {geo.M2} values, got {tuple(y.shape)}")
        out = torch.empty(oshape, dtype=torch.complex128, device=y.device)
        _lib.check(_lib.lib.sincfft_nnfft_adjoint(plan.handle, C.c_void_p(y.data_ptr()),
                                                  C.c_void_p(out.data_ptr()), batch,
                                                  _lib.PTR_DEVICE, _stream_handle(y)))
        return out
    y = np.ascontiguousarray(y, dtype=complex)
    if y.shape == (geo.M2,):
        batch = 1
        out = np.empty(geo.M1, dtype=complex)
    elif y.ndim == 2 and y.shape[0] == geo.M2 and y.shape[1] >= 1:
        batch = y.shape[1]
        out = np.empty((geo.M1, batch), dtype=complex)
    else:
        raise ParameterError(f"nnfft_adjoint: expected {geo.M2} values, got {y.shape}")
    _lib.check(_lib.lib.sincfft_nnfft_adjoint(plan.handle, _vp(y), _vp(out), batch,
                                              _lib.PTR_HOST, None))
    return out


def nnfft_trafo_into(plan, f, out, stream=None, blocking=True):
    """Extension for pipelined host-side use: write the transform of ``f`` into
    ``out`` (CPU torch tensors, ideally page-locked, or numpy arrays).  With
    ``blocking=False`` the H2D copy, the kernels and the D2H copy are only
    enqueued on ``stream`` (a ``torch.cuda.Stream``; default: current) via
    ``SINCFFT_PTR_HOST_ASYNC`` and the caller synchronizes the stream before
    reading ``out`` or reusing ``f`` -- alternating two streams overlaps the
    copies of consecutive transforms."""
    import torch
    geo = plan.geometry
    if isinstance(f, np.ndarray):
        f = torch.from_numpy(np.ascontiguousarray(f, dtype=complex))
    if isinstance(out, np.ndarray):
        out = torch.from_numpy(out)
    if f.dtype != torch.complex128 or out.dtype != torch.complex128:
        raise ParameterError("nnfft_trafo_into: f and out must be complex128")
    if f.device.type != "cpu" or out.device.type != "cpu":
        raise ParameterError("nnfft_trafo_into: f and out must be host tensors")
    if not (f.is_contiguous() and out.is_contiguous()):
        raise ParameterError("nnfft_trafo_into: f and out must be contiguous")
    batch = 1 if f.ndim == 1 else f.shape[1]
    if f.shape[0] != geo.M1 or tuple(out.shape) != ((geo.M2,) if f.ndim == 1 else (geo.M2, batch)):
        raise ParameterError("nnfft_trafo_into: shape mismatch with the plan")
    st = stream if stream is not None else torch.cuda.current_stream(plan.device)
    kind = _lib.PTR_HOST if blocking else _lib.PTR_HOST_ASYNC
    _lib.check(_lib.lib.sincfft_nnfft_execute(plan.handle, C.c_void_p(f.data_ptr()),
                                              C.c_void_p(out.data_ptr()), batch, kind,
                                              C.c_void_p(st.cuda_stream)))
    return out
