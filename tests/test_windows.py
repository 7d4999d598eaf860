"""Public window functions (drop-in for the reference's ``sincfft.windows``,
windows.py:41-220, sinh kind).

CPU: the oracle's window restatement against golden vectors the reference
produced (tests/golden/make_windows_golden.py), and the API surface.
GPU: ``omega_eval`` / ``omega_hat_eval`` / ``phi_eval`` / ``phi_hat_eval``
(device kernels behind ``sincfft_window_eval``) against the same vectors, plus
the reference's own window tests (tests/test_windows.py:20-98) restated."""

import numpy as np
import pytest

from oracle import sincfft_oracle as O


def _specs(golden):
    g = golden("windows.npz")
    for i, (m, sigma, n_grid) in enumerate(g["specs"]):
        yield g, i, int(m), float(sigma), int(n_grid)


def _close(a, b, rtol, scale):
    return np.max(np.abs(np.asarray(a) - np.asarray(b)) / (rtol * (np.abs(b) + scale)))


def test_oracle_windows_match_reference(golden):
    for g, i, m, sigma, n_grid in _specs(golden):
        beta = O.sinh_beta(m, sigma)
        assert np.array_equal(O.omega_sinh(beta, g[f"s{i}_x"]), g[f"s{i}_omega"])
        assert np.array_equal(O.phi_sinh(beta, m, n_grid, g[f"s{i}_t"]), g[f"s{i}_phi"])
        assert np.array_equal(O.omega_hat_sinh(beta, g[f"s{i}_v"]), g[f"s{i}_omega_hat"])
        assert np.array_equal(O.phi_hat_sinh(beta, m, n_grid, g[f"s{i}_vg"]), g[f"s{i}_phi_hat"])


def test_api_surface():
    import paper_2107_02671_b200 as sf
    for name in ("omega_eval", "omega_hat_eval", "phi_eval", "phi_hat_eval", "window_kinds",
                 "cc_export_csv", "WindowSpec"):
        assert name in sf.__all__ and callable(getattr(sf, name))
    assert sf.window_kinds() == ("sinh",)
    with pytest.raises(sf.ParameterError):
        sf.WindowSpec("gauss", 4, 2.0, 64)
    with pytest.raises(sf.ParameterError):
        sf.WindowSpec("sinh", 4, 2.5, 64)
    with pytest.raises(sf.ParameterError):
        sf.WindowSpec("bspline", 4, 2.0, 64)  # kind the B200 backend does not implement


def test_cc_export_csv_format(tmp_path):
    """sinc_approx.py:157-165 / reference tests/test_sinc_approx.py:95-103."""
    import paper_2107_02671_b200 as sf
    quad = sf.cc_quadrature(64)
    out = tmp_path / "weights.csv"
    sf.cc_export_csv(quad, str(out))
    lines = out.read_text().splitlines()
    assert lines[0] == "# schema=1"
    assert lines[1] == "k,z_k,w_k"
    assert len(lines) == quad.n + 3
    k, z, w = lines[2].split(",")
    assert int(k) == 0 and float(z) == 1.0
    assert float(w) == pytest.approx(quad.weights[0], rel=1e-16)
    rows = [ln.split(",") for ln in lines[2:]]
    assert np.array_equal([float(r[1]) for r in rows], quad.points)
    assert np.array_equal([float(r[2]) for r in rows], quad.weights)


@pytest.mark.gpu
def test_gpu_windows_match_reference(golden):
    import paper_2107_02671_b200 as sf
    worst = {}
    for g, i, m, sigma, n_grid in _specs(golden):
        spec = sf.WindowSpec("sinh", m, sigma, n_grid)
        pref = 2.0 * np.pi * spec.beta * np.exp(-spec.beta) / -np.expm1(-2.0 * spec.beta)
        cases = [
            ("omega", sf.omega_eval(spec, g[f"s{i}_x"]), g[f"s{i}_omega"], 1e-16),
            ("phi", sf.phi_eval(spec, g[f"s{i}_t"]), g[f"s{i}_phi"], 1e-16),
            # omega_hat spans e^{-beta}..1: relative, with an absolute floor of
            # 1e-13 of the series prefactor for the oscillating J1 branch
            ("omega_hat", sf.omega_hat_eval(spec, g[f"s{i}_v"]), g[f"s{i}_omega_hat"], pref),
            ("phi_hat", sf.phi_hat_eval(spec, g[f"s{i}_vg"]), g[f"s{i}_phi_hat"],
             pref * m / n_grid),
        ]
        for name, got, ref, scale in cases:
            assert got.shape == ref.shape
            # support edges are exact: zero where the reference is zero
            assert np.array_equal(got == 0.0, ref == 0.0), (name, m, sigma)
            worst[name] = max(worst.get(name, 0.0), _close(got, ref, 1e-13, scale))
        sc = g[f"s{i}_scalar"]
        got_sc = [sf.omega_eval(spec, 0.25), sf.omega_hat_eval(spec, 0.5),
                  sf.phi_eval(spec, 1.0 / n_grid), sf.phi_hat_eval(spec, 3.0)]
        assert all(isinstance(s, float) for s in got_sc)
        assert np.max(np.abs(np.array(got_sc) - sc) / np.abs(sc)) <= 1e-13
    print("window parity (units of 1e-13 relative):", worst)
    assert max(worst.values()) <= 1.0


@pytest.mark.gpu
def test_gpu_window_properties():
    """The reference's own window tests (tests/test_windows.py:20-98), sinh kind."""
    import paper_2107_02671_b200 as sf
    spec = sf.WindowSpec("sinh", 4, 2.0, 64)
    x = np.linspace(0.0, 1.0, 501)
    vals = sf.omega_eval(spec, x)
    assert sf.omega_eval(spec, 0.0) == pytest.approx(1.0, abs=1e-14)
    assert np.allclose(sf.omega_eval(spec, -x), vals, atol=1e-15)
    assert np.all(np.diff(vals) <= 1e-14)
    assert np.all(vals >= 0.0)
    assert sf.omega_eval(spec, 1.2) == 0.0
    assert np.all(sf.omega_eval(spec, np.array([-3.0, 1.0 + 1e-9])) == 0.0)
    v = np.linspace(0.0, spec.m / (2.0 * spec.sigma), 41)
    hat = sf.omega_hat_eval(spec, v)
    assert np.all(hat > 0.0) and np.all(np.diff(hat) < 1e-13)
    v0 = spec.beta / (2.0 * np.pi)
    seam = sf.omega_hat_eval(spec, v0 + np.linspace(-1e-4, 1e-4, 9))
    assert np.all(np.isfinite(seam)) and np.max(np.abs(np.diff(seam, 2))) < 1e-10
    t = np.array([0.0, 0.01, -0.03, 0.06])
    assert np.allclose(sf.phi_eval(spec, t), sf.omega_eval(spec, t * spec.n_grid / spec.m),
                       atol=0)
    vv = np.array([0.0, 1.0, 5.0, 31.0])
    assert np.allclose(sf.phi_hat_eval(spec, vv), (spec.m / spec.n_grid)
                       * sf.omega_hat_eval(spec, vv * spec.m / spec.n_grid), atol=0)
    assert sf.omega_eval(spec, np.zeros((3, 0))).shape == (3, 0)
    assert sf.omega_eval(spec, np.zeros((2, 3))).shape == (2, 3)
