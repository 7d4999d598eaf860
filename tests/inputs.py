"""Seeded input generators shared by tests and bench (BASELINE.md 3 recipe:
np.random.default_rng(seed); first node set, second node set, coefficient
real parts, coefficient imaginary parts)."""

import hashlib

import numpy as np


def nodes_and_coeffs(seed, M1, M2, clustered=False, batch=0):
    rng = np.random.default_rng(seed)
    if clustered:
        v = 0.5 * np.cos(np.pi * rng.uniform(0.0, 1.0, M1))
        x = 0.5 * np.cos(np.pi * rng.uniform(0.0, 1.0, M2))
    else:
        v = rng.uniform(-0.5, 0.5, M1)
        x = rng.uniform(-0.5, 0.5, M2)
    if batch:
        f = rng.standard_normal((M1, batch)) + 1j * rng.standard_normal((M1, batch))
    else:
        f = rng.standard_normal(M1) + 1j * rng.standard_normal(M1)
    return v, x, f


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()
