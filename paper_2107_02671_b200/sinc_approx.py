"""The Clenshaw-Curtis exponential-sum surrogate of sinc, evaluated on the GPU.

Drop-in for the evaluation half of ``sincfft.sinc_approx`` (reference
``pkg/src/sincfft/sinc_approx.py:109-153``; the quadrature half lives in
``quadrature.py``).  ``sinc(pi N x) ~ (1/2) sum_k w_k e^{-i pi N z_k x}``
(Lemma 6.1) with the Clenshaw-Curtis nodes ``z_k`` and weights ``w_k``.

* ``sinc_expsum_eval`` -- the exponential sum at arbitrary ``x`` as the exact
  NNDFT ``sum_k w_k e^{-2 pi i N (z_k / 2) x}`` on the device
  (``direct.nndft_direct``; the reference sums the same terms in chunks of
  2048 targets on the CPU).
* ``sinc_expsum_eval_grid`` -- the same sum on the even grid ``x_r = 2r/R``
  as ONE adjoint NFFT of degree ``R`` at the nodes ``z_k N / R`` with the
  reference's internal window (sinh, sigma = 2, m = 12), on the device
  (``nfft.nfft_adjoint``).
* ``sinc_expsum_max_error`` -- ``max_r |surrogate(x_r) - sinc(pi N x_r)|``.
"""

from __future__ import annotations

import numpy as np

from .direct import nndft_direct
from .errors import ParameterError
from .nfft import nfft_adjoint, nfft_plan

_DOMAIN_TOL = 1e-12  # sinc_approx.py:26


def sinc(y):
    """Unnormalised sinc ``sin(y)/y`` with value 1 at 0 (special.py:88-93)."""
    arr = np.asarray(y, dtype=float)
    with np.errstate(invalid="ignore", divide="ignore"):
        out = np.where(arr == 0.0, 1.0, np.sin(arr) / np.where(arr == 0.0, 1.0, arr))
    return float(out) if np.ndim(y) == 0 else out


def sinc_expsum_eval(quad, N, x, *, device=None):
    """Surrogate at arbitrary ``x in [-1, 1]`` (sinc_approx.py:109-127)."""
    arr = np.atleast_1d(np.asarray(x, dtype=float))
    if arr.size and np.max(np.abs(arr)) > 1.0 + _DOMAIN_TOL:
        raise ParameterError("sinc_expsum_eval: x must lie in [-1, 1]")
    arr = np.clip(arr, -1.0, 1.0)
    out = nndft_direct(quad.weights.astype(complex), quad.points / 2.0, arr, int(N), device=device)
    if np.ndim(x) == 0:
        return out[0]
    return out


def sinc_expsum_eval_grid(quad, N, R, *, device=None):
    """Surrogate on ``x_r = 2r/R``, ``r = -R/2 .. R/2 - 1`` (sinc_approx.py:130-147);
    requires even ``R >= 2N``."""
    if not isinstance(R, (int, np.integer)) or R < 2 or R % 2:
        raise ParameterError("sinc_expsum_eval_grid: R must be a positive even integer")
    if R < 2 * N:
        raise ParameterError("sinc_expsum_eval_grid: need R >= 2*N")
    plan = nfft_plan(int(R), quad.points * (N / R), sigma=2.0, m=12, window="sinh",
                     device=device)
    return nfft_adjoint(plan, quad.weights.astype(complex))


def sinc_expsum_max_error(quad, N, R, *, device=None):
    """``max_r |surrogate(x_r) - sinc(pi N x_r)|`` on ``x_r = 2r/R``
    (sinc_approx.py:150-155)."""
    approx = sinc_expsum_eval_grid(quad, N, R, device=device)
    x = 2.0 * (np.arange(R) - R // 2) / R
    return float(np.max(np.abs(approx - sinc(np.pi * N * x))))
