"""Pin the CPU oracle (oracle/sincfft_oracle.py) against fixtures produced by
the reference itself (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import sincfft_oracle as O
from tests.inputs import digest, nodes_and_coeffs


def rel(a, b, f):
    return np.max(np.abs(np.asarray(a) - np.asarray(b))) / np.sum(np.abs(f))


def test_config1_tables_and_output(golden):
    g = golden("nnfft_config1.npz")
    n_star, vs = O.rescale_frequencies(int(g["N"]), g["v"], 2.0, int(g["m"]))
    assert n_star == int(g["n_star"])
    assert np.array_equal(vs, g["v_star"])
    t = O.plan(n_star, vs, g["x"], m1=4, m2=4)
    assert np.array_equal(t.spread_idx, g["spread_idx"])
    assert np.array_equal(t.gather_idx, g["gather_idx"])
    assert np.array_equal(t.spread_val, g["spread_val"])
    assert np.array_equal(t.gather_val, g["gather_val"])
    assert np.array_equal(t.hat1, g["hat1"])
    assert np.array_equal(t.hat2, g["hat2"])
    out = O.trafo(t, g["f"])
    assert rel(out, g["out"], g["f"]) <= 1e-15
    # the reference's accuracy at config 1 (6.1e-8) is within the paper bound
    err = rel(out, g["direct"], g["f"])
    assert err <= float(g["bound"])


def test_config2_all_m(golden):
    g = golden("nnfft_config2.npz")
    v, x, f = nodes_and_coeffs(0, 65536, 65536)
    assert digest(v, x, f) == str(g["input_digest"]), "numpy RNG stream changed"
    for m in (2, 4, 6, 8, 10):
        n_star, vs = O.rescale_frequencies(4096, v, 2.0, m)
        assert n_star == int(g[f"m{m}_n_star"])
        out = O.trafo(O.plan(n_star, vs, x, m1=m, m2=m), f)
        assert rel(out[:2048], g[f"m{m}_head"], f) <= 1e-15
        j = np.arange(out.size)
        l1 = np.sum(np.abs(f))
        assert abs(out.sum() - g[f"m{m}_sum"]) <= 1e-13 * l1
        assert abs((out * np.cos(0.001 * j)).sum() - g[f"m{m}_wsum"]) <= 1e-13 * l1
        err = np.max(np.abs(out[:1024] - g["direct_head"])) / l1
        assert err <= float(g[f"m{m}_bound"])


@pytest.mark.parametrize("name,clustered,batch", [("nnfft_config3_small.npz", True, 0),
                                                  ("nnfft_config4_small.npz", False, 4)])
def test_scaled_configs(golden, name, clustered, batch):
    g = golden(name)
    N, m = int(g["N"]), int(g["m"])
    n_star, vs = O.rescale_frequencies(N, g["v"], 2.0, m)
    t = O.plan(n_star, vs, g["x"], m1=m, m2=m)
    f = g["f"]
    if batch:
        out = np.stack([O.trafo(t, f[:, b]) for b in range(batch)], axis=1)
    else:
        out = O.trafo(t, f)
    assert rel(out, g["out"], f) <= 1e-15


def test_small_cases(golden):
    g = golden("nnfft_small_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g[f"c{k}_{key}"]  # noqa: E731
        t = O.plan(int(c("N")), c("v"), c("x"), float(c("sigma1")), float(c("sigma2")),
                   int(c("m1")), int(c("m2")))
        out = O.trafo(t, c("f"))
        assert rel(out, c("out"), c("f")) <= 1e-15, k


def test_geometry_rows(golden):
    rows = golden("geometry.npz")["rows"]
    for N, s1, s2, m1, m2, N1, N2, a, sig1, sig2 in rows:
        geo = O.geometry(int(N), 1, 1, s1, s2, int(m1), int(m2))
        assert (geo.N1, geo.N2) == (int(N1), int(N2))
        assert geo.a == a and geo.sigma1 == sig1 and geo.sigma2 == sig2


def test_sinc_cases(golden):
    g = golden("sinc_cases.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g[f"s{k}_{key}"]  # noqa: E731
        st = O.sinc_plan(int(s("N")), s("a"), s("b"), m1=int(s("m")), m2=int(s("m")))
        assert st.n_star == int(s("n_star"))
        out = O.sinc_transform(st, s("c"))
        assert rel(out, s("out"), s("c")) <= 1e-15, k
        err = np.max(np.abs(out[:64] - s("direct"))) / np.sum(np.abs(s("c")))
        assert err <= float(s("bound_full"))
    z, w = O.cc_quadrature(16384)
    assert np.array_equal(z, g["cc16384_z"])
    assert np.max(np.abs(w - g["cc16384_w"])) <= 1e-16
    assert np.max(np.abs(O.cc_quadrature(6)[1] - g["cc_w6"])) <= 1e-16


def test_nfft_cases(golden):
    """Classical NFFT restatement (ref:nfft.py) against the reference's own
    trafo / adjoint outputs, plan tables and hat values."""
    g = golden("nfft_cases.npz")
    for k in range(int(g["ncases"])):
        c = lambda key: g[f"c{k}_{key}"]  # noqa: E731
        t = O.nfft_plan(int(c("N")), c("x"), float(c("sigma")), int(c("m")))
        assert np.array_equal(t.hat, c("hat")), k
        if f"c{k}_spread_idx" in g.files:
            assert np.array_equal(t.spread_idx, c("spread_idx")), k
            assert np.array_equal(t.spread_val, c("spread_val")), k
        assert rel(O.nfft_trafo(t, c("c")), c("trafo"), c("c")) <= 1e-15, k
        assert rel(O.nfft_adjoint(t, c("y")), c("adjoint"), c("y")) <= 1e-15, k


def test_sinc_modes(golden):
    """All four fast-sinc layouts (ref:fast_sinc.py:171-248)."""
    g = golden("sinc_modes.npz")
    for k in range(int(g["ncases"])):
        s = lambda key: g[f"s{k}_{key}"]  # noqa: E731
        N = int(s("N"))
        assert O.sinc_mode(N, s("a"), s("b")) == str(s("mode")) or str(s("forced")), k
        st = O.sinc_plan(N, s("a"), s("b"), m1=int(s("m")), m2=int(s("m")),
                         mode=str(s("forced")) or None)
        assert st.mode == str(s("mode")), k
        out = O.sinc_transform(st, s("c"))
        assert rel(out, s("out"), s("c")) <= 1e-15, k
        err = np.max(np.abs(out - s("direct"))) / np.sum(np.abs(s("c")))
        assert err <= float(s("bound_full")), k


def test_oracle_adjoint_is_the_conjugate_transpose(golden):
    """The oracle's adjoint NNFFT (no reference counterpart) is pinned through
    the pinned trafo: <A f, y> = <f, A^H y> to rounding on config 1's plan."""
    g = golden("nnfft_config1.npz")
    t = O.plan(int(g["n_star"]), g["v_star"], g["x"], m1=int(g["m"]), m2=int(g["m"]))
    y = np.random.default_rng(3).standard_normal(g["x"].size) * (1 + 2j)
    lhs = np.vdot(y, O.trafo(t, g["f"]))
    rhs = np.vdot(O.adjoint(t, y), g["f"])
    assert abs(lhs - rhs) <= 1e-14 * np.linalg.norm(g["f"]) * np.linalg.norm(y) * 64


def test_chunked_oracle_matches_reference(golden):
    """trafo_chunked (the bounded-memory oracle the full-size config-3 parity
    test uses) against the reference's own output; chunks far smaller than
    the inputs so every chunk boundary path runs."""
    for name in ("nnfft_config3_small.npz", "nnfft_config1.npz"):
        g = golden(name)
        N, m = int(g["N"]), int(g["m"])
        n_star, vs = O.rescale_frequencies(N, g["v"], 2.0, m)
        out = O.trafo_chunked(n_star, vs, g["x"], g["f"], m1=m, m2=m, chunk=777)
        assert rel(out, g["out"], g["f"]) <= 1e-15, name
