"""GPU parity of the B200 NNFFT / fast sinc path against the reference.

Two oracles: the golden fixtures produced by running the reference
(tests/golden/make_golden.py) and the pinned CPU restatement
(oracle/sincfft_oracle.py) run live on the same seeded inputs.  Tolerance:
max-abs error <= 1e-12 * ||f||_1 (north star), plus the paper's bound against
the direct NDFT on target subsets.  All calls go through the C ABI.
"""

import numpy as np
import pytest

import paper_2107_02671_b200 as sf
from oracle import sincfft_oracle as O
from tests.inputs import digest, nodes_and_coeffs

pytestmark = pytest.mark.gpu
TOL = 1e-12


def relerr(a, b, f):
    return float(np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.sum(np.abs(f)))


def gpu_nnfft(N, v, x, f, m, sigma=2.0, rescale=True, m2=None, sigma2=None):
    m2 = m if m2 is None else m2
    sigma2 = sigma if sigma2 is None else sigma2
    if rescale:
        N, v = sf.rescale_frequencies(N, v, sigma, m)
    plan = sf.nnfft_plan(N, v, x, sigma1=sigma, sigma2=sigma2, m1=m, m2=m2)
    return plan, sf.nnfft_trafo(plan, f)


def test_config1_against_reference_fixture(golden):
    g = golden("nnfft_config1.npz")
    plan, out = gpu_nnfft(int(g["N"]), g["v"], g["x"], g["f"], int(g["m"]))
    assert relerr(out, g["out"], g["f"]) <= TOL
    assert relerr(out, g["direct"], g["f"]) <= float(g["bound"])


def test_config1_step0_tables(golden):
    """The device plan's windows/indices equal the reference's step-0 tables."""
    g = golden("nnfft_config1.npz")
    plan, _ = gpu_nnfft(int(g["N"]), g["v"], g["x"], g["f"], int(g["m"]))
    assert np.array_equal(plan.spread_idx, g["spread_idx"])
    assert np.array_equal(plan.gather_idx, g["gather_idx"])
    # the node offset d = N1 v - floor(N1 v) carries the rounding of N1 v
    # (|N1 v| <= 260 here: ulp 5.7e-14 grid units) and the reference's argument
    # l/N1 - v a comparable one; |d omega/d d| <= beta/m ~ 5 gives ~1e-13
    assert np.max(np.abs(plan.spread_val - g["spread_val"])) <= 1e-13
    assert np.max(np.abs(plan.gather_val - g["gather_val"])) <= 1e-13
    assert np.max(np.abs(plan.hat1 / g["hat1"] - 1)) <= 1e-13
    assert np.max(np.abs(plan.hat2 / g["hat2"] - 1)) <= 1e-13


def test_small_reference_geometries(golden):
    g = golden("nnfft_small_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g[f"c{k}_{key}"]  # noqa: E731
        plan = sf.nnfft_plan(int(c("N")), c("v"), c("x"), sigma1=float(c("sigma1")),
                             sigma2=float(c("sigma2")), m1=int(c("m1")), m2=int(c("m2")))
        out = sf.nnfft_trafo(plan, c("f"))
        assert relerr(out, c("out"), c("f")) <= TOL, k


@pytest.mark.parametrize("m", [2, 4, 6, 8, 10])
def test_config2_full_vs_oracle(golden, m):
    g = golden("nnfft_config2.npz")
    v, x, f = nodes_and_coeffs(0, 65536, 65536)
    assert digest(v, x, f) == str(g["input_digest"])
    plan, out = gpu_nnfft(4096, v, x, f, m)
    assert relerr(out[:2048], g[f"m{m}_head"], f) <= TOL
    n_star, vs = O.rescale_frequencies(4096, v, 2.0, m)
    ref = O.trafo(O.plan(n_star, vs, x, m1=m, m2=m), f)
    assert relerr(out, ref, f) <= TOL
    # the paper's bound against the direct NDFT on 1024 targets
    err = np.max(np.abs(out[:1024] - g["direct_head"])) / np.sum(np.abs(f))
    assert err <= float(g[f"m{m}_bound"])


@pytest.mark.parametrize("name,batch", [("nnfft_config3_small.npz", 0),
                                        ("nnfft_config4_small.npz", 4)])
def test_scaled_configs(golden, name, batch):
    g = golden(name)
    plan, out = gpu_nnfft(int(g["N"]), g["v"], g["x"], g["f"], int(g["m"]))
    assert out.shape == g["out"].shape
    assert relerr(out, g["out"], g["f"]) <= TOL


def test_batch_equals_columns():
    v, x, f = nodes_and_coeffs(11, 3000, 2500, batch=3)
    N, vs = sf.rescale_frequencies(512, v, 2.0, 6)
    plan = sf.nnfft_plan(N, vs, x, m1=6, m2=6)
    out = sf.nnfft_trafo(plan, f)
    for b in range(3):
        col = sf.nnfft_trafo(plan, np.ascontiguousarray(f[:, b]))
        assert np.max(np.abs(out[:, b] - col)) <= 1e-15 * np.sum(np.abs(f[:, b]))


def test_sinc_against_reference_fixture(golden):
    g = golden("sinc_cases.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g[f"s{k}_{key}"]  # noqa: E731
        plan = sf.sinc_plan(int(s("N")), s("a"), s("b"), m1=int(s("m")), m2=int(s("m")))
        assert plan.mode is sf.SincMode.GENERAL
        assert plan.n_star == int(s("n_star"))
        out = sf.fast_sinc_transform(plan, s("c"))
        assert relerr(out, s("out"), s("c")) <= TOL, k
        out_c = sf.fast_sinc_transform(plan, s("c").astype(complex))
        assert relerr(out_c, out, s("c")) <= 1e-15
        err = np.max(np.abs(out[:64] - s("direct"))) / np.sum(np.abs(s("c")))
        assert err <= plan.error_bound()["full"]


def test_out_of_band_rejected_by_name():
    with pytest.raises(sf.ParameterError, match="rescale_frequencies"):
        sf.nnfft_plan(32, np.array([0.5]), np.zeros(4))
    with pytest.raises(sf.ParameterError):
        sf.nnfft_plan(32, np.zeros(4), np.array([0.7]))


def test_torch_device_path(golden):
    torch = pytest.importorskip("torch")
    g = golden("nnfft_config1.npz")
    n_star, vs = sf.rescale_frequencies(int(g["N"]), g["v"], 2.0, 4)
    dv = torch.from_numpy(vs).cuda()
    dx = torch.from_numpy(g["x"]).cuda()
    df = torch.from_numpy(g["f"]).cuda()
    plan = sf.nnfft_plan(n_star, dv, dx, m1=4, m2=4)
    out = sf.nnfft_trafo(plan, df)
    torch.cuda.synchronize()
    assert relerr(out.cpu().numpy(), g["out"], g["f"]) <= TOL
    with pytest.raises(sf.ParameterError, match="rescale_frequencies"):
        sf.nnfft_plan(n_star, torch.full((4,), 0.5, dtype=torch.float64, device="cuda"), dx)


def test_single_wave_known_answer():
    # pkg/tests/test_nnfft.py:87-93
    v = np.array([0.21])
    x = np.linspace(-0.5, 0.5, 33)
    plan = sf.nnfft_plan(32, v, x, m1=6, m2=6)
    out = sf.nnfft_trafo(plan, np.array([1.0 + 0j]))
    assert np.max(np.abs(out - np.exp(-2j * np.pi * 32 * v[0] * x))) < 1e-9


def test_host_node_copies_are_clipped_lazily():
    """plan.v / plan.x are the reference's clipped nodes (nnfft.py:168-170);
    numpy inputs within the 1e-12 domain tolerance are clipped on first access,
    the device plan clips its own copy."""
    vlim = 0.5 / sf.NnfftGeometry.from_parameters(32, 3, 4, 2.0, 2.0, 4, 4).a
    v = np.array([-vlim - 5e-13, 0.1, vlim + 5e-13])
    x = np.array([-0.5 - 5e-13, 0.0, 0.25, 0.5 + 5e-13])
    plan = sf.nnfft_plan(32, v, x, m1=4, m2=4)
    out = sf.nnfft_trafo(plan, np.ones(3, complex))
    assert np.all(np.isfinite(out))
    assert plan.v.max() == vlim and plan.v.min() == -vlim
    assert plan.x.max() == 0.5 and plan.x.min() == -0.5
    ref = sf.nnfft_trafo(sf.nnfft_plan(32, np.clip(v, -vlim, vlim), np.clip(x, -0.5, 0.5),
                                       m1=4, m2=4), np.ones(3, complex))
    assert np.array_equal(out, ref)
