"""Golden vectors for the public window functions, produced by the REFERENCE.

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_windows_golden.py

Imports ``/root/reference/pkg/src/sincfft`` and evaluates ``omega_eval``,
``omega_hat_eval``, ``phi_eval`` and ``phi_hat_eval`` (windows.py:106-220) for
sinh specs over the BASELINE cut-offs and oversampling range, on arguments
that hit every branch: inside / on / outside the support, the series seam
w = 0 of omega_hat, and the J1 branch (w < 0).  Writes ``windows.npz``.
"""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
from sincfft import windows as W  # noqa: E402  (the reference itself)

SPECS = [(2, 2.0, 64), (4, 2.0, 64), (6, 1.25, 64), (6, 2.0, 262192), (8, 2.0, 2097168),
         (8, 1.5, 4096), (10, 2.0, 16464), (16, 1.25, 1024)]


def main():
    rng = np.random.default_rng(7)
    out = {"specs": np.array([(m, s, n) for m, s, n in SPECS], dtype=float)}
    for i, (m, sigma, n_grid) in enumerate(SPECS):
        spec = W.WindowSpec("sinh", m, sigma, n_grid)
        x = np.concatenate([rng.uniform(-1.2, 1.2, 400), np.linspace(-1.0, 1.0, 201),
                            [0.0, 1.0, -1.0, 1.0 - 1e-12, -1.0 + 1e-15, 1.0 + 1e-9, 3.0]])
        v0 = spec.beta / (2.0 * np.pi)  # w = 0 seam
        v = np.concatenate([rng.uniform(0.0, 2.0 * m, 300),
                            np.linspace(0.0, m / (2.0 * sigma), 41),
                            v0 + np.linspace(-1e-4, 1e-4, 9), -rng.uniform(0, m, 20)])
        t = x * (m / n_grid)
        vg = v * (n_grid / m)
        out[f"s{i}_x"], out[f"s{i}_omega"] = x, W.omega_eval(spec, x)
        out[f"s{i}_v"], out[f"s{i}_omega_hat"] = v, W.omega_hat_eval(spec, v)
        out[f"s{i}_t"], out[f"s{i}_phi"] = t, W.phi_eval(spec, t)
        out[f"s{i}_vg"], out[f"s{i}_phi_hat"] = vg, W.phi_hat_eval(spec, vg)
        out[f"s{i}_scalar"] = np.array([W.omega_eval(spec, 0.25), W.omega_hat_eval(spec, 0.5),
                                        W.phi_eval(spec, 1.0 / n_grid),
                                        W.phi_hat_eval(spec, 3.0)])
    np.savez_compressed(os.path.join(HERE, "windows.npz"), **out)


if __name__ == "__main__":
    main()
