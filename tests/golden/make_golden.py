"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

The reference package has no frozen output vectors for ``nnfft_trafo`` or
``fast_sinc_transform``, so these fixtures are produced by
importing ``/root/reference/pkg/src/sincfft`` and calling its public API on
seeded inputs.  Tests never import the reference: they read these files.

Input recipe (BASELINE.md 3 / SURVEY.md 8d): ``np.random.default_rng(seed)``,
drawn in the order first node set, second node set, coefficient real parts,
coefficient imaginary parts; frequencies in [-1/2, 1/2) pass through
``rescale_frequencies`` before ``nnfft_plan``.
"""

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")
import sincfft  # noqa: E402  (the reference itself)
from sincfft import bounds as rbounds  # noqa: E402


def digest(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def uniform_case(seed, N, M1, M2, clustered=False, batch=0):
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


def nnfft_ref(N, v, x, f, m, sigma=2.0, rescale=True, m2=None):
    m2 = m if m2 is None else m2
    if rescale:
        n_star, vs = sincfft.rescale_frequencies(N, v, sigma, m)
    else:
        n_star, vs = N, v
    plan = sincfft.nnfft_plan(n_star, vs, x, sigma1=sigma, sigma2=sigma, m1=m, m2=m2)
    if f.ndim == 2:
        out = np.stack([sincfft.nnfft_trafo(plan, f[:, b]) for b in range(f.shape[1])], axis=1)
    else:
        out = sincfft.nnfft_trafo(plan, f)
    return n_star, vs, plan, out


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: {os.path.getsize(path) / 1024:.1f} KiB")


def main():
    # --- config 1: full tables + output (BASELINE.json configs[0], seed 0)
    v, x, f = uniform_case(0, 256, 1024, 1024)
    n_star, vs, plan, out = nnfft_ref(256, v, x, f, 4)
    save("nnfft_config1.npz", N=256, m=4, n_star=n_star, v=v, x=x, f=f, v_star=vs, out=out,
         spread_idx=plan.spread_idx.astype(np.int32), spread_val=plan.spread_val,
         gather_idx=plan.gather_idx.astype(np.int32), gather_val=plan.gather_val,
         hat1=plan.hat1, hat2=plan.hat2,
         direct=sincfft.nndft_direct(f, v, x, 256),
         bound=rbounds.bound_nnfft_sinh(n_star, 2.0, 2.0, 4, 4))

    # --- config 2: N=4096, M1=M2=65536, m in {2,4,6,8,10}; inputs regenerated from seed 0,
    #     pinned by digest; outputs: first 2048 values + whole-vector checksums
    v, x, f = uniform_case(0, 4096, 65536, 65536)
    d2 = {"input_digest": digest(v, x, f)}
    direct = sincfft.nndft_direct(f, v, x[:1024], 4096)
    d2["direct_head"] = direct
    for m in (2, 4, 6, 8, 10):
        n_star, vs, plan, out = nnfft_ref(4096, v, x, f, m)
        j = np.arange(out.size)
        d2[f"m{m}_n_star"] = n_star
        d2[f"m{m}_head"] = out[:2048]
        d2[f"m{m}_sum"] = out.sum()
        d2[f"m{m}_wsum"] = (out * np.cos(0.001 * j)).sum()
        d2[f"m{m}_l1"] = np.abs(out).sum()
        d2[f"m{m}_bound"] = rbounds.bound_nnfft_sinh(n_star, 2.0, 2.0, m, m)
    save("nnfft_config2.npz", **d2)

    # --- scaled config 3 (clustered cos nodes), scaled config 4 (batched) --- full outputs
    v, x, f = uniform_case(3, 1 << 12, 1 << 14, 1 << 14, clustered=True)
    n_star, vs, plan, out = nnfft_ref(1 << 12, v, x, f, 8)
    save("nnfft_config3_small.npz", N=1 << 12, m=8, v=v, x=x, f=f, out=out)
    v, x, f = uniform_case(4, 1024, 1 << 12, 1 << 12, batch=4)
    n_star, vs, plan, out = nnfft_ref(1024, v, x, f, 6)
    save("nnfft_config4_small.npz", N=1024, m=6, v=v, x=x, f=f, out=out)

    # --- small reference-test geometries (tests/test_nnfft.py) and edge cases
    cases = {}
    k = 0
    for sigma in (1.25, 1.5, 2.0):
        for m in (2, 3, 4, 5):
            rng = np.random.default_rng(1000 * m + int(4 * sigma))
            N, M1, M2 = 64, 40, 50
            geo = sincfft.NnfftGeometry.from_parameters(N, M1, M2, sigma, sigma, m, m)
            v = rng.uniform(-0.5 / geo.a, 0.5 / geo.a, M1)
            x = rng.uniform(-0.5, 0.5, M2)
            f = rng.uniform(-1, 1, M1) + 1j * rng.uniform(-1, 1, M1)
            plan = sincfft.nnfft_plan(N, v, x, sigma1=sigma, sigma2=sigma, m1=m, m2=m)
            out = sincfft.nnfft_trafo(plan, f)
            cases[f"c{k}"] = dict(N=N, sigma1=sigma, sigma2=sigma, m1=m, m2=m, v=v, x=x, f=f, out=out)
            k += 1
    # loop-reference geometry (tests/test_nnfft.py:116-126)
    rng = np.random.default_rng(77)
    geo = sincfft.NnfftGeometry.from_parameters(16, 9, 11, 2.0, 2.0, 3, 3)
    v = rng.uniform(-0.5 / geo.a, 0.5 / geo.a, 9)
    x = rng.uniform(-0.5, 0.5, 11)
    f = rng.uniform(-1, 1, 9) + 1j * rng.uniform(-1, 1, 9)
    plan = sincfft.nnfft_plan(16, v, x, m1=3, m2=3)
    cases[f"c{k}"] = dict(N=16, sigma1=2.0, sigma2=2.0, m1=3, m2=3, v=v, x=x, f=f,
                          out=sincfft.nnfft_trafo(plan, f)); k += 1
    # edge case: band-edge frequencies, x = +-1/2 and 0, exact grid coincidences, m1 != m2
    N = 128
    geo = sincfft.NnfftGeometry.from_parameters(N, 8, 8, 2.0, 2.0, 4, 6)
    lim = 0.5 / geo.a
    v = np.array([-lim, lim, 0.0, 3.0 / geo.N1, -7.0 / geo.N1, 0.123, -0.31, lim * (1 - 1e-16)])
    x = np.array([-0.5, 0.5, 0.0, 0.25, -0.25, 5.0 / geo.N2 * 2, 0.4999999, -0.3])
    f = np.array([1, -2, 0.5, 1.5, 1j, -1j, 2 + 1j, 0.25])
    plan = sincfft.nnfft_plan(N, v, x, m1=4, m2=6)
    cases[f"c{k}"] = dict(N=N, sigma1=2.0, sigma2=2.0, m1=4, m2=6, v=v, x=x, f=f,
                          out=sincfft.nnfft_trafo(plan, f)); k += 1
    # odd counts (tests/test_nnfft.py:139-144) and sigma2 rounding to even N2 (394)
    plan = sincfft.nnfft_plan(16, np.array([0.1, -0.2, 0.3]), np.array([0.4, -0.4]), m1=3, m2=3)
    cases[f"c{k}"] = dict(N=16, sigma1=2.0, sigma2=2.0, m1=3, m2=3, v=np.array([0.1, -0.2, 0.3]),
                          x=np.array([0.4, -0.4]), f=np.ones(3, complex),
                          out=sincfft.nnfft_trafo(plan, np.ones(3, complex))); k += 1
    rng = np.random.default_rng(5)
    geo = sincfft.NnfftGeometry.from_parameters(128, 30, 20, 2.0, 1.5, 3, 3)
    v = rng.uniform(-0.5 / geo.a, 0.5 / geo.a, 30)
    x = rng.uniform(-0.5, 0.5, 20)
    f = rng.standard_normal(30) + 1j * rng.standard_normal(30)
    plan = sincfft.nnfft_plan(128, v, x, sigma1=2.0, sigma2=1.5, m1=3, m2=3)
    cases[f"c{k}"] = dict(N=128, sigma1=2.0, sigma2=1.5, m1=3, m2=3, v=v, x=x, f=f,
                          out=sincfft.nnfft_trafo(plan, f), N2=plan.geometry.N2); k += 1
    flat = {}
    for name, d in cases.items():
        for key, val in d.items():
            flat[f"{name}_{key}"] = val
    flat["ncases"] = k
    save("nnfft_small_cases.npz", **flat)

    # --- geometry known answers (tests/test_nnfft.py:13-31) and window transform values
    geos = []
    for args in [(128, 64, 48, 2.0, 2.0, 4, 4), (128, 10, 10, 2.0, 1.5, 3, 3),
                 (4096 + 4, 1, 1, 2.0, 2.0, 8, 8), (1048584, 1, 1, 2.0, 2.0, 8, 8),
                 (65542, 1, 1, 2.0, 2.0, 6, 6), (260, 1, 1, 2.0, 2.0, 4, 4)]:
        g = sincfft.NnfftGeometry.from_parameters(*args)
        geos.append([args[0], args[3], args[4], args[5], args[6], g.N1, g.N2, g.a, g.sigma1, g.sigma2])
    save("geometry.npz", rows=np.array(geos, dtype=float))

    # --- fast sinc, GENERAL mode (config 5 scaled down + reference-test shapes)
    sc = {}
    k = 0
    for (N, L1, L2, m, seed) in [(48, 24, 30, 6, 11), (64, 32, 40, 8, 5), (256, 4096, 4096, 8, 5),
                                 (16, 4, 10, 6, 7)]:
        rng = np.random.default_rng(seed)
        a = rng.uniform(-0.5, 0.5, L1)
        b = rng.uniform(-0.5, 0.5, L2)
        if L1 == 4:
            a = np.array([-0.5, -0.2, 0.3, 0.5])
        c = rng.standard_normal(L1)
        plan = sincfft.sinc_plan(N, a, b, m1=m, m2=m)
        assert plan.mode is sincfft.SincMode.GENERAL
        out = sincfft.fast_sinc_transform(plan, c)
        sc[f"s{k}_N"] = N
        sc[f"s{k}_m"] = m
        sc[f"s{k}_a"] = a
        sc[f"s{k}_b"] = b
        sc[f"s{k}_c"] = c
        sc[f"s{k}_out"] = out
        sc[f"s{k}_n_star"] = plan.n_star
        sc[f"s{k}_bound_full"] = plan.error_bound()["full"]
        sc[f"s{k}_direct"] = sincfft.sinc_transform_direct(c, a, b[:64], N)
        k += 1
    sc["ncases"] = k
    q = sincfft.cc_quadrature(16384)
    sc["cc16384_w"] = q.weights
    sc["cc16384_z"] = q.points
    sc["cc_w6"] = sincfft.cc_quadrature(6).weights  # non-power-of-two direct path
    save("sinc_cases.npz", **sc)


def main_nfft():
    """Classical NFFT (nfft.py) and the equispaced fast-sinc routes
    (fast_sinc.py:200-248): SURVEY.md 8f row f1."""
    nf = {}
    k = 0
    # (N, M, sigma, m, seed): reference-test shapes (tests/test_nfft.py),
    # sigma 5/4 and 3/2, nodes at +-1/2 and on grid points, larger sizes
    for (N, M, sigma, m, seed) in [(64, 129, 2.0, 2, 102), (64, 129, 2.0, 4, 104),
                                   (64, 129, 2.0, 6, 106), (12, 29, 2.0, 6, 17),
                                   (32, 47, 2.0, 4, 0), (16, 3, 2.0, 4, 1), (128, 200, 1.5, 5, 3),
                                   (160, 333, 1.25, 3, 4), (4096, 16385, 2.0, 8, 9),
                                   (1024, 5000, 2.0, 10, 10)]:
        rng = np.random.default_rng(seed)
        x = rng.uniform(-0.5, 0.5, M)
        if M == 3:
            x = np.array([0.0, 0.24, -0.5])
        if M == 333:
            x[:4] = [-0.5, 0.5, 0.0, 1.0 / (sigma * N)]
        c = rng.uniform(-1, 1, N) + 1j * rng.uniform(-1, 1, N)
        y = rng.standard_normal(M) + 1j * rng.standard_normal(M)
        plan = sincfft.nfft_plan(N, x, sigma=sigma, m=m)
        nf[f"c{k}_N"] = N
        nf[f"c{k}_sigma"] = sigma
        nf[f"c{k}_m"] = m
        nf[f"c{k}_x"] = x
        nf[f"c{k}_c"] = c
        nf[f"c{k}_y"] = y
        nf[f"c{k}_trafo"] = sincfft.nfft_trafo(plan, c)
        nf[f"c{k}_adjoint"] = sincfft.nfft_adjoint(plan, y)
        nf[f"c{k}_hat"] = plan.hat
        if M * 2 * m <= 4096:
            nf[f"c{k}_spread_idx"] = plan.spread_idx.astype(np.int32)
            nf[f"c{k}_spread_val"] = plan.spread_val
        k += 1
    nf["ncases"] = k
    save("nfft_cases.npz", **nf)

    # --- fast sinc: all four layouts on grid node sets
    sm = {}
    k = 0
    # (N, L1, L2, m, seed, a on grid, b on grid, forced modes)
    for (N, L1, L2, m, seed, agrid, bgrid, modes) in [
            (32, 24, 32, 6, 21, True, True, None), (48, 16, 40, 6, 22, True, False, None),
            (64, 50, 64, 8, 23, False, True, None), (256, 512, 256, 8, 24, True, True, None),
            (40, 40, 30, 6, 25, False, False, None),
            (64, 64, 64, 8, 26, True, True,
             ("general", "equispaced-sources", "equispaced-targets", "equispaced-both"))]:
        rng = np.random.default_rng(seed)
        a = (np.arange(L1) - L1 // 2) / L1 if agrid else rng.uniform(-0.5, 0.5, L1)
        b = (np.arange(L2) - L2 // 2) / L2 if bgrid else rng.uniform(-0.5, 0.5, L2)
        c = rng.standard_normal(L1) + (1j * rng.standard_normal(L1) if seed % 2 else 0.0)
        for mode in (modes or (None,)):
            plan = sincfft.sinc_plan(N, a, b, m1=m, m2=m, mode=mode)
            sm[f"s{k}_N"] = N
            sm[f"s{k}_m"] = m
            sm[f"s{k}_a"] = a
            sm[f"s{k}_b"] = b
            sm[f"s{k}_c"] = c
            sm[f"s{k}_mode"] = plan.mode.value
            sm[f"s{k}_forced"] = mode or ""
            sm[f"s{k}_out"] = sincfft.fast_sinc_transform(plan, c)
            sm[f"s{k}_direct"] = sincfft.sinc_transform_direct(c, a, b, N)
            sm[f"s{k}_bound_full"] = plan.error_bound()["full"]
            k += 1
    sm["ncases"] = k
    save("sinc_modes.npz", **sm)


if __name__ == "__main__":
    if sys.argv[1:] == ["nfft"]:
        main_nfft()
    else:
        main()
        main_nfft()
