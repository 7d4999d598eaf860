"""Clenshaw-Curtis nodes and weights for the sinc surrogate (host, plan time).

The fast sinc transform needs the n+1 Chebyshev points z_k = cos(k pi/n) and
positive weights w_k summing to 1 (reference: ``pkg/src/sincfft/
sinc_approx.py:30-106``, one orthonormal DCT-I when n is a power of two,
``fft_core.py:31-42``).  This is O(n log n) plan-time input data (n = 16384
at config 5), computed on the host like the reference and copied to the GPU
by ``sinc_plan``; it is not a hot-path kernel.
"""

from dataclasses import dataclass

import numpy as np
import scipy.fft

from .errors import ParameterError


@dataclass(frozen=True)
class CcQuadrature:
    n: int
    points: np.ndarray
    weights: np.ndarray


def _eps(n, idx):
    return np.where((idx == 0) | (idx == n), np.sqrt(0.5), 1.0)


def chebyshev_points(n):
    """cos(k pi/n), exact zero at n/2, mirrored so z_k = -z_{n-k} exactly
    (sinc_approx.py:48-57)."""
    k = np.arange(n // 2 + 1)
    half = np.cos(np.pi * k / n)
    if n % 2 == 0:
        half[n // 2] = 0.0
    z = np.empty(n + 1)
    z[:half.size] = half
    z[n + 1 - half.size:] = -half[::-1]
    return z


def cc_weights_direct(n):
    """Explicit cosine sum with exact integer phase reduction (sinc_approx.py:60-75)."""
    if not isinstance(n, (int, np.integer)) or n < 2:
        raise ParameterError("cc_weights_direct: n must be an integer >= 2")
    jmax = n // 2
    j = np.arange(jmax + 1)
    coef = _eps(n, 2 * j) ** 2 * (2.0 / (1.0 - 4.0 * j * j))
    k = np.arange(n + 1)
    phase = (2 * np.outer(j, k)) % (2 * n)
    return (_eps(n, k) ** 2 / n) * (coef @ np.cos((np.pi / n) * phase))


def cc_weights_fast(n):
    """One orthonormal DCT-I, n = 2^t >= 4 (sinc_approx.py:78-94)."""
    if not isinstance(n, (int, np.integer)) or n < 4 or n & (n - 1):
        raise ParameterError("cc_weights_fast: n must be a power of two >= 4")
    a = np.zeros(n + 1)
    j = np.arange(n // 2 + 1)
    a[::2] = _eps(n, 2 * j) * (2.0 / (1.0 - 4.0 * j * j))
    ahat = scipy.fft.dct(a, type=1, norm="ortho")
    return _eps(n, np.arange(n + 1)) / np.sqrt(2.0 * n) * ahat


def cc_quadrature(n):
    """sinc_approx.py:97-106."""
    if not isinstance(n, (int, np.integer)) or n < 2:
        raise ParameterError("cc_quadrature: n must be an integer >= 2")
    w = cc_weights_fast(n) if (n >= 4 and (n & (n - 1)) == 0) else cc_weights_direct(n)
    return CcQuadrature(int(n), chebyshev_points(n), np.asarray(w, dtype=float))


def cc_export_csv(quad, path):
    """Write the quadrature to ``path`` as CSV with columns k, z_k, w_k
    (sinc_approx.py:157-165: a ``# schema=1`` line, the header, then one row
    per node with both floats printed to 17 significant digits)."""
    with open(path, "w", encoding="utf-8", newline="") as fh:
        fh.write("# schema=1\nk,z_k,w_k\n")
        fh.writelines(f"{k},{format(z, '.17g')},{format(w, '.17g')}\n"
                      for k, (z, w) in enumerate(zip(quad.points[:quad.n + 1],
                                                     quad.weights[:quad.n + 1])))
