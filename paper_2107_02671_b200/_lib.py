"""ctypes binding of the C ABI in ``include/sincfft_b200.h``.

The shared library ``paper_2107_02671_b200/lib/libsincfft_b200.so`` is built
in-tree by ``__graft_entry__.build()`` (``make -C paper_2107_02671_b200/csrc``).
There is no fallback: if the library is missing, importing this module raises.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import ParameterError, PositivityError

LIB_PATH = os.environ.get("SINCFFT_B200_LIB") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libsincfft_b200.so")

OK, EPARAM, EPOSITIVITY, ECUDA, ENOMEM, EUNSUPPORTED = range(6)
PTR_HOST, PTR_DEVICE, PTR_HOST_ASYNC = 0, 1, 2
PLAN_FULL_WINDOW = 1  # sincfft_nnfft_plan_create_ex flags


class Geometry(C.Structure):
    """Mirror of ``sincfft_geometry``."""

    _fields_ = [
        ("N", C.c_int64), ("M1", C.c_int64), ("M2", C.c_int64),
        ("N1", C.c_int64), ("K", C.c_int64), ("N2", C.c_int64),
        ("m1", C.c_int32), ("m2", C.c_int32),
        ("sigma1", C.c_double), ("sigma2", C.c_double), ("a", C.c_double),
        ("beta1", C.c_double), ("beta2", C.c_double),
        ("L", C.c_int64), ("L1", C.c_int64), ("L2", C.c_int64),
        ("Kout", C.c_int64), ("s_lo", C.c_int64),
    ]


class BackendError(RuntimeError):
    """A CUDA-side failure (status SINCFFT_ECUDA)."""


class UnsupportedError(ParameterError):
    """Input outside the envelope the B200 kernels implement (e.g. m > 16)."""


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_vp = C.c_void_p

# name -> (restype, argtypes); every function declared in include/sincfft_b200.h
SIGNATURES = {
    "sincfft_last_error": (C.c_char_p, []),
    "sincfft_version": (C.c_int, []),
    "sincfft_device_count": (C.c_int, []),
    "sincfft_nnfft_plan_create": (C.c_int, [C.POINTER(_vp), C.c_int64, C.c_int64, C.c_int64,
                                            C.c_double, C.c_double, C.c_int32, C.c_int32,
                                            _vp, _vp, C.c_int32, C.c_int32, _vp]),
    "sincfft_nnfft_plan_create_ex": (C.c_int, [C.POINTER(_vp), C.c_int64, C.c_int64,
                                               C.c_int64, C.c_double, C.c_double, C.c_int32,
                                               C.c_int32, _vp, _vp, C.c_int32, C.c_int32,
                                               C.c_int32, _vp]),
    "sincfft_nnfft_plan_destroy": (C.c_int, [_vp]),
    "sincfft_nnfft_dist_layout": (C.c_int, [_vp, C.c_int32, _i64p]),
    "sincfft_nnfft_dist_pack": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp]),
    "sincfft_nnfft_dist_colfwd": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp]),
    "sincfft_nnfft_dist_rowmul": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp]),
    "sincfft_nnfft_dist_colinv": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp, _vp, _vp]),
    "sincfft_nnfft_dist_gather": (C.c_int, [_vp, C.c_int32, _vp, _vp, _vp]),
    "sincfft_nnfft_dist_support": (C.c_int, [_vp, _i64p, _vp]),
    "sincfft_ipc_alloc": (C.c_int, [C.c_int32, C.c_int64, C.POINTER(_vp)]),
    "sincfft_ipc_free": (C.c_int, [_vp]),
    "sincfft_ipc_handle": (C.c_int, [_vp, C.POINTER(C.c_uint8)]),
    "sincfft_ipc_open": (C.c_int, [C.c_int32, C.POINTER(C.c_uint8), C.POINTER(_vp)]),
    "sincfft_ipc_close": (C.c_int, [_vp]),
    "sincfft_nnfft_dist_colfwd_peer": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp,
                                                 C.POINTER(C.c_uint64), _vp]),
    "sincfft_nnfft_dist_rowmul_peer": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp,
                                                 C.POINTER(C.c_uint64), _vp]),
    "sincfft_nnfft_dist_pack_rows_peer": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, C.c_int64,
                                                    C.c_int64, C.POINTER(C.c_uint64), _i64p,
                                                    _vp]),
    "sincfft_nnfft_dist_colinv_peer": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _vp,
                                                 C.POINTER(C.c_uint64), _i64p, _i64p, _vp]),
    "sincfft_nnfft_dist_pack_rows": (C.c_int, [_vp, C.c_int32, _vp, C.c_int64, C.c_int64, _vp,
                                               _vp]),
    "sincfft_nnfft_dist_unpack_rows": (C.c_int, [_vp, C.c_int32, C.c_int32, _vp, _i64p, _i64p,
                                                 _vp, _vp]),
    "sincfft_nnfft_dist_pack_hrows": (C.c_int, [_vp, C.c_int32, _vp, _i64p, _i64p, _vp, _vp]),
    "sincfft_nnfft_dist_gather_rows": (C.c_int, [_vp, C.c_int32, _vp, C.c_int64, C.c_int64, _vp,
                                                 _vp]),
    "sincfft_nnfft_plan_geometry": (C.c_int, [_vp, C.POINTER(Geometry)]),
    "sincfft_nnfft_execute": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, _vp]),
    "sincfft_nnfft_spread": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, _vp]),
    "sincfft_nnfft_finish": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, _vp]),
    "sincfft_nnfft_export_tables": (C.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sincfft_nnfft_execute_profiled": (C.c_int, [_vp, _vp, _vp, C.c_int64, _vp, _vp]),
    "sincfft_nnfft_launches_per_execute": (C.c_int, [_vp, C.c_int64]),
    "sincfft_sinc_plan_create": (C.c_int, [C.POINTER(_vp), C.c_int64, C.c_int64, C.c_int64,
                                           C.c_int64, C.c_int64, _vp, _vp, _vp, _vp,
                                           C.c_double, C.c_double, C.c_int32, C.c_int32,
                                           C.c_int32, C.c_int32, C.c_int32, _vp]),
    "sincfft_sinc_plan_destroy": (C.c_int, [_vp]),
    "sincfft_sinc_plan_geometry": (C.c_int, [_vp, C.POINTER(Geometry), C.POINTER(Geometry)]),
    "sincfft_sinc_execute": (C.c_int, [_vp, _vp, C.c_int32, _vp, C.c_int32, _vp]),
    "sincfft_sinc_stage1": (C.c_int, [_vp, _vp, C.c_int32, _vp, _vp]),
    "sincfft_sinc_stage3": (C.c_int, [_vp, _vp, _vp, _vp]),
    "sincfft_nnfft_adjoint": (C.c_int, [_vp, _vp, _vp, C.c_int64, C.c_int32, _vp]),
    "sincfft_nfft_plan_create": (C.c_int, [C.POINTER(_vp), C.c_int64, C.c_int64, C.c_double,
                                           C.c_int32, _vp, C.c_int32, C.c_int32, _vp]),
    "sincfft_nfft_plan_destroy": (C.c_int, [_vp]),
    "sincfft_nfft_plan_geometry": (C.c_int, [_vp, C.POINTER(C.c_int64), C.POINTER(Geometry),
                                             C.POINTER(Geometry)]),
    "sincfft_nfft_trafo": (C.c_int, [_vp, _vp, _vp, C.c_int32, _vp]),
    "sincfft_nfft_adjoint": (C.c_int, [_vp, _vp, _vp, C.c_int32, _vp]),
    "sincfft_nfft_export_tables": (C.c_int, [_vp, _vp, _vp, _vp]),
    "sincfft_nndft_direct": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int64, _vp,
                                       C.c_int32, C.c_int32, _vp]),
    "sincfft_ndft_direct": (C.c_int, [_vp, C.c_int64, _vp, C.c_int64, _vp, C.c_int32,
                                      C.c_int32, _vp]),
    "sincfft_sinc_direct": (C.c_int, [_vp, _vp, C.c_int64, _vp, C.c_int64, C.c_int64, _vp,
                                      C.c_int32, C.c_int32, _vp]),
    "sincfft_window_eval": (C.c_int, [C.c_int32, C.c_double, C.c_int32, C.c_int64, _vp,
                                      C.c_int64, _vp, C.c_int32, C.c_int32, _vp]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or make -C "
            "paper_2107_02671_b200/csrc); there is no CPU fallback")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.sincfft_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Map a status code to the reference's exception classes."""
    if status == OK:
        return
    msg = last_error()
    if status == EPARAM:
        raise ParameterError(msg)
    if status == EPOSITIVITY:
        raise PositivityError(msg)
    if status == EUNSUPPORTED:
        raise UnsupportedError(msg)
    if status == ENOMEM:
        raise MemoryError(msg)
    raise BackendError(msg or f"sincfft status {status}")


def device_count() -> int:
    return int(lib.sincfft_device_count())


def require_gpu() -> None:
    if device_count() < 1:
        raise BackendError("no CUDA device visible: the B200 backend has no CPU fallback")
