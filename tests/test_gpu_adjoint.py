"""Adjoint NNFFT on the GPU (BASELINE north star's adjoint-NNFFT entry point;
SURVEY.md 8f row f4).  The reference has no adjoint NNFFT, so parity is
pinned by (1) the inner-product identity with the GPU forward transform
(which is pinned to the reference), (2) the oracle's stage-by-stage
conjugate transpose of the reference's trafo, and (3) the exact adjoint sum
on the GPU within the NNFFT's error bound.
"""

import numpy as np
import pytest

import paper_2107_02671_b200 as sf
from oracle import sincfft_oracle as O
from tests.inputs import nodes_and_coeffs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def l1err(a, b, f):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.sum(np.abs(f)))


CASES = [(256, 1024, 1500, 4, 2.0, 2.0, False), (4096, 65536, 65536, 8, 2.0, 2.0, False),
         (700, 5000, 3000, 6, 1.5, 1.25, True), (1 << 16, 1 << 18, 1 << 18, 8, 2.0, 2.0, True),
         (124, 300, 200, 2, 1.25, 2.0, False)]


@pytest.mark.parametrize("N,M1,M2,m,s1,s2,clustered", CASES)
def test_adjoint_vs_oracle_and_identity(N, M1, M2, m, s1, s2, clustered):
    v, x, f = nodes_and_coeffs(N + M2, M1, M2, clustered=clustered)
    y = np.random.default_rng(M1).standard_normal(M2) * (1 - 0.5j)
    n, vs = sf.rescale_frequencies(N, v, s1, m)
    plan = sf.nnfft_plan(n, vs, x, sigma1=s1, sigma2=s2, m1=m, m2=m)
    adj = sf.nnfft_adjoint(plan, y)
    assert adj.shape == (M1,)
    tab = O.plan(n, vs, x, s1, s2, m, m)
    assert l1err(adj, O.adjoint(tab, y), y) <= TOL
    fw = sf.nnfft_trafo(plan, f)
    lhs, rhs = np.vdot(y, fw), np.vdot(adj, f)
    assert abs(lhs - rhs) <= 1e-13 * np.linalg.norm(f) * np.linalg.norm(y) * np.sqrt(M1 + M2)


def test_adjoint_vs_exact_sum():
    """out_k ~ sum_j y_j e^{+2 pi i N v_k x_j} within the NNFFT's bound."""
    v, x, _ = nodes_and_coeffs(3, 20000, 30000)
    y = np.random.default_rng(4).standard_normal(30000) + 1j
    N, m = 2048, 8
    n, vs = sf.rescale_frequencies(N, v, 2.0, m)
    plan = sf.nnfft_plan(n, vs, x, m1=m, m2=m)
    adj = sf.nnfft_adjoint(plan, y)
    idx = np.r_[0:256]
    exact = sf.nndft_direct(y, x, v[idx], -N)
    err = np.max(np.abs(adj[idx] - exact)) / np.sum(np.abs(y))
    assert err <= O.bound_nnfft_sinh(n, 2.0, 2.0, m, m)


def test_adjoint_batch_and_torch():
    import torch
    v, x, _ = nodes_and_coeffs(9, 3000, 2500)
    Y = np.random.default_rng(5).standard_normal((2500, 3)) + 0.25j
    n, vs = sf.rescale_frequencies(512, v, 2.0, 6)
    plan = sf.nnfft_plan(n, vs, x, m1=6, m2=6)
    out = sf.nnfft_adjoint(plan, Y)
    assert out.shape == (3000, 3)
    for b in range(3):
        col = sf.nnfft_adjoint(plan, np.ascontiguousarray(Y[:, b]))
        assert np.max(np.abs(out[:, b] - col)) <= 1e-15 * np.sum(np.abs(Y[:, b]))
    tout = sf.nnfft_adjoint(plan, torch.from_numpy(Y).cuda())
    assert tout.is_cuda and np.max(np.abs(tout.cpu().numpy() - out)) <= 1e-15 * np.sum(np.abs(Y))
    with pytest.raises(sf.ParameterError, match="expected 2500 values"):
        sf.nnfft_adjoint(plan, np.ones(7, dtype=complex))


@pytest.mark.slow
def test_adjoint_config3_full_size():
    """Config 3 (2^24 + 2^24 clustered nodes): the identity at full size."""
    v, x, f = nodes_and_coeffs(0, 1 << 24, 1 << 24, clustered=True)
    y = np.random.default_rng(1).standard_normal(1 << 24) * (1 + 1j)
    n, vs = sf.rescale_frequencies(1 << 20, v, 2.0, 8)
    plan = sf.nnfft_plan(n, vs, x, m1=8, m2=8)
    lhs = np.vdot(y, sf.nnfft_trafo(plan, f))
    rhs = np.vdot(sf.nnfft_adjoint(plan, y), f)
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(f) * np.linalg.norm(y)
