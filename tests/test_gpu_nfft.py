"""GPU parity of the classical NFFT / adjoint NFFT and the equispaced
fast-sinc layouts against the reference.

Oracles: fixtures from running the reference (tests/golden/nfft_cases.npz,
sinc_modes.npz; make_golden.py main_nfft), the CPU restatement run live,
the GPU direct sums (tests/test_gpu_direct.py pins those), and the
properties the reference's own tests assert (tests/test_nfft.py,
test_fast_sinc.py, test_acceptance.py c08/c09).  Tolerance as for the
NNFFT: 1e-12 * sum|input| against the reference's outputs.
"""

import numpy as np
import pytest

import paper_2107_02671_b200 as sf
from oracle import sincfft_oracle as O

pytestmark = pytest.mark.gpu
TOL = 1e-12


def l1err(a, b, f):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.sum(np.abs(f)))


def test_nfft_against_reference_fixtures(golden):
    g = golden("nfft_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g[f"c{k}_{key}"]  # noqa: E731
        plan = sf.nfft_plan(int(c("N")), c("x"), sigma=float(c("sigma")), m=int(c("m")))
        assert plan.n_over == round(float(c("sigma")) * int(c("N")))
        assert l1err(sf.nfft_trafo(plan, c("c")), c("trafo"), c("c")) <= TOL, k
        assert l1err(sf.nfft_adjoint(plan, c("y")), c("adjoint"), c("y")) <= TOL, k
        assert np.max(np.abs(plan.hat / c("hat") - 1)) <= 1e-13, k
        if f"c{k}_spread_idx" in g.files:
            assert np.array_equal(plan.spread_idx, c("spread_idx")), k
            # d = n_over x - floor(n_over x) carries the rounding of n_over x
            # (|n_over x| <= n_over/2), the reference's x - l/n_over a comparable one
            tol = 1e-13 * max(1.0, float(c("N")) / 64)
            assert np.max(np.abs(plan.spread_val - c("spread_val"))) <= tol, k


@pytest.mark.parametrize("N,M,m,clustered", [(1 << 14, 1 << 18, 8, False), (4096, 16385, 6, True),
                                             (1 << 20, 1 << 16, 4, False)])
def test_nfft_vs_oracle_live(N, M, m, clustered):
    rng = np.random.default_rng(N + M)
    x = 0.5 * np.cos(np.pi * rng.uniform(0, 1, M)) if clustered else rng.uniform(-0.5, 0.5, M)
    c = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    plan = sf.nfft_plan(N, x, m=m)
    t = O.nfft_plan(N, x, 2.0, m)
    assert l1err(sf.nfft_trafo(plan, c), O.nfft_trafo(t, c), c) <= TOL
    assert l1err(sf.nfft_adjoint(plan, y), O.nfft_adjoint(t, y), y) <= TOL


@pytest.mark.parametrize("m", [2, 4, 6])
def test_trafo_error_below_window_bound(m):
    """tests/test_nfft.py:18-26 -- against the (GPU) exact polynomial."""
    rng = np.random.default_rng(100 + m)
    N, M = 64, 129
    x = rng.uniform(-0.5, 0.5, M)
    c = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
    plan = sf.nfft_plan(N, x, sigma=2.0, m=m)
    err = np.max(np.abs(sf.nfft_trafo(plan, c) - sf.ndft_direct(c, x)))
    assert err <= sf.bounds.bound_sinh_E(m, 2.0) * np.sum(np.abs(c))


def test_spread_rows_have_fixed_width():
    """tests/test_nfft.py:29-38: 2m entries per node, the last one of a node
    on a grid point carries the window's exact zero."""
    plan = sf.nfft_plan(16, np.array([0.0, 0.24, -0.5]), sigma=2.0, m=4)
    assert plan.spread_idx.shape == (3, 8) and plan.spread_val.shape == (3, 8)
    assert np.all((plan.spread_idx >= 0) & (plan.spread_idx < plan.n_over))
    assert np.all(plan.spread_val >= 0.0)
    row = plan.spread_val[0]
    assert row[-1] == 0.0 and np.count_nonzero(row) == 7


def test_adjoint_matches_conjugate_sum():
    rng = np.random.default_rng(17)
    N, M = 12, 29
    x = rng.uniform(-0.5, 0.5, M)
    y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    plan = sf.nfft_plan(N, x, sigma=2.0, m=6)
    k = np.arange(N) - N // 2
    ref = np.exp(-2j * np.pi * np.outer(k, x)) @ y
    assert np.max(np.abs(sf.nfft_adjoint(plan, y) - ref)) <= \
        sf.bounds.bound_sinh_E(6, 2.0) * np.sum(np.abs(y))


def test_adjoint_inner_product_identity():
    """<A c, y> = <c, A* y> to rounding (test_nfft.py:52-63, acceptance c09)."""
    rng = np.random.default_rng(909)
    worst = 0.0
    for _ in range(50):
        N = 2 * int(rng.integers(4, 33))
        M = int(rng.integers(5, 80))
        x = rng.uniform(-0.5, 0.5, M)
        c = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        plan = sf.nfft_plan(N, x, sigma=2.0, m=4)
        lhs = np.vdot(y, sf.nfft_trafo(plan, c))
        rhs = np.vdot(sf.nfft_adjoint(plan, y), c)
        worst = max(worst, abs(lhs - rhs) / (np.linalg.norm(c) * np.linalg.norm(y)))
    assert worst <= 1e-12
    # and at a size where the device FFT is the multi-kernel Bluestein
    N, M = 1 << 16, 100000
    x = rng.uniform(-0.5, 0.5, M)
    c = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
    plan = sf.nfft_plan(N, x, m=8)
    lhs = np.vdot(y, sf.nfft_trafo(plan, c))
    rhs = np.vdot(sf.nfft_adjoint(plan, y), c)
    assert abs(lhs - rhs) <= 1e-13 * np.linalg.norm(c) * np.linalg.norm(y) * np.sqrt(N)


def test_periodic_wrap_at_half():
    c = np.random.default_rng(2).standard_normal(16) + 0j
    left = sf.nfft_trafo(sf.nfft_plan(16, np.array([-0.5])), c)
    right = sf.nfft_trafo(sf.nfft_plan(16, np.array([0.5])), c)
    assert abs(left[0] - right[0]) < 1e-12 * np.sum(np.abs(c))


def test_plan_rejects_like_reference():
    with pytest.raises(sf.ParameterError, match="positive even integer"):
        sf.nfft_plan(15, np.zeros(3))
    with pytest.raises(sf.ParameterError, match="even integer"):
        sf.nfft_plan(16, np.zeros(3), sigma=1.3)
    with pytest.raises(sf.ParameterError, match="lie in"):
        sf.nfft_plan(16, np.array([0.6]))
    with pytest.raises(sf.ParameterError, match="2\\*m"):
        sf.nfft_plan(8, np.zeros(3), sigma=2.0, m=6)
    with pytest.raises(sf.ParameterError, match="expected 16 coefficients"):
        sf.nfft_trafo(sf.nfft_plan(16, np.zeros(3)), np.ones(8, dtype=complex))
    with pytest.raises(sf.ParameterError, match="expected 3 values"):
        sf.nfft_adjoint(sf.nfft_plan(16, np.zeros(3)), np.ones(8, dtype=complex))
    with pytest.raises((sf.PositivityError, sf.ParameterError)):
        sf.nfft_plan(64, np.zeros(2), sigma=1.0, m=4, window="bspline")


def test_nfft_torch_device_path():
    import torch
    rng = np.random.default_rng(4)
    N, M = 256, 1000
    x = rng.uniform(-0.5, 0.5, M)
    c = rng.standard_normal(N) + 1j * rng.standard_normal(N)
    plan = sf.nfft_plan(N, x, m=6)
    ct = torch.from_numpy(c).cuda()
    out = sf.nfft_trafo(plan, ct)
    assert out.is_cuda and out.shape == (M,)
    assert l1err(out.cpu().numpy(), sf.nfft_trafo(plan, c), c) <= 1e-15
    back = sf.nfft_adjoint(plan, out)
    assert l1err(back.cpu().numpy(), sf.nfft_adjoint(plan, out.cpu().numpy()), out.cpu().numpy()) \
        <= 1e-15


def test_sinc_modes_against_reference_fixtures(golden):
    g = golden("sinc_modes.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g[f"s{k}_{key}"]  # noqa: E731
        N, m = int(s("N")), int(s("m"))
        plan = sf.sinc_plan(N, s("a"), s("b"), m1=m, m2=m, mode=str(s("forced")) or None)
        assert plan.mode.value == str(s("mode")), k
        out = sf.fast_sinc_transform(plan, s("c"))
        assert l1err(out, s("out"), s("c")) <= TOL, k
        err = np.max(np.abs(out - s("direct"))) / np.sum(np.abs(s("c")))
        assert err <= float(s("bound_full")), k


def test_special_case_equivalence():
    """Acceptance c08 (test_acceptance.py:161-177): the equispaced-targets
    route equals the forced GENERAL route to 1e-11 * sum|c|."""
    rng = np.random.default_rng(808)
    N, L1 = 128, 64
    a = rng.uniform(-0.5, 0.5, L1)
    b = (np.arange(N) - N // 2) / N
    c = rng.uniform(-1, 1, L1) + 1j * rng.uniform(-1, 1, L1)
    fast = sf.sinc_plan(N, a, b, n=4 * N, m1=10, m2=10)
    general = sf.sinc_plan(N, a, b, n=4 * N, m1=10, m2=10, mode="general")
    assert fast.mode is sf.SincMode.EQUISPACED_TARGETS
    assert fast.route == "nnfft/adjoint" and general.route == "nnfft/nnfft"
    gap = np.max(np.abs(sf.fast_sinc_transform(fast, c) - sf.fast_sinc_transform(general, c)))
    assert gap / np.sum(np.abs(c)) <= 1e-11


@pytest.mark.parametrize("layout", ["equispaced-sources", "equispaced-both"])
def test_large_equispaced_layouts_vs_oracle(layout):
    """Config-5-sized equispaced layouts: L1 = 2^18 grid sources (an NFFT of
    degree 2^18) against the live oracle and the GPU exact sum."""
    rng = np.random.default_rng(55)
    N, L1 = 4096, 1 << 18
    a = (np.arange(L1) - L1 // 2) / L1
    b = (np.arange(N) - N // 2) / N if layout == "equispaced-both" else rng.uniform(-0.5, 0.5, 5000)
    c = rng.standard_normal(L1)
    plan = sf.sinc_plan(N, a, b, m1=8, m2=8)
    assert plan.mode.value == layout
    out = sf.fast_sinc_transform(plan, c)
    ref = O.sinc_transform(O.sinc_plan(N, a, b, m1=8, m2=8), c)
    assert l1err(out, ref, c) <= TOL
    idx = rng.integers(0, b.size, 256)
    direct = sf.sinc_transform_direct(c, a, b[idx], N)
    assert np.max(np.abs(out[idx] - direct)) / np.sum(np.abs(c)) <= plan.error_bound()["full"]
