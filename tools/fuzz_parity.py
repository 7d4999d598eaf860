"""dev helper (GPU box): randomized parity of the whole public surface against
the CPU oracle -- NNFFT (single column and batched), adjoint NNFFT, NFFT /
adjoint NFFT and the fast sinc transform -- over random bandwidths (even, odd
multiples, primes times two, powers of two: every FFT realisation the planner
can pick), node counts, cut-offs, oversampling factors and node layouts
(uniform, clustered, a few cells, duplicates, band edges).  Test
infrastructure: imports oracle/.

    python tools/fuzz_parity.py [cases] [seed] [large]

"large": bandwidths 2^17 .. 2^20 (and non-power-of-two neighbours) with 2e5 ..
2^21 nodes -- the persistent spread, the dense moment spread, the four-step
Bluestein shapes and the TMA gather at sizes where every SM is busy.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_02671_b200 as sf  # noqa: E402
from oracle import sincfft_oracle as O  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
LARGE = len(sys.argv) > 3 and sys.argv[3] == "large"
TOL = 1e-12
worst = {}


def nodes(M, kind):
    u = rng.random(M)
    if kind == 0:
        return u - 0.5
    if kind == 1:
        return 0.5 * np.cos(np.pi * u)
    if kind == 2:  # a few cells
        return (u - 0.5) * 1e-3 + rng.choice([-0.4, 0.0, 0.3])
    if kind == 3:  # duplicates and the band edges
        a = rng.choice(np.array([-0.5, 0.5, 0.0, 0.25, -0.125]), M)
        return a
    return np.sort(u - 0.5)


def edge_noise(m, sigma, G):
    """The window's edge taps behave like C sqrt(d), C = beta sqrt(2/m) / sinh(beta), in
    the cell offset d, which either implementation knows to ~eps * G cells on a grid of
    G points: a node sitting exactly on a grid point (d = 0) sees C sqrt(eps G) of
    tap noise -- 2e-9 at m = 2, 1e-11 at m = 3, nothing from m = 4 on."""
    beta = 2.0 * np.pi * m * (1.0 - 0.5 / sigma)
    return beta * np.sqrt(2.0 / m) / np.sinh(beta) * np.sqrt(4e-16 * G)


def note(kind, err, desc, tol=TOL):
    worst[kind] = max(worst.get(kind, 0.0), err)
    ok = err <= tol
    print(f"{'ok ' if ok else 'BAD'} {kind:12s} {err:.2e}  {desc}", flush=True)
    if not ok:
        raise SystemExit(f"parity failure: {kind} {desc}")


rejected = 0


def one_case(c):
    N = int(rng.choice([8, 12, 30, 64, 100, 254, 256, 1000, 1024, 2 * 1031, 4096, 6 * 1001,
                        10000, 16384, 2 * 16411, 65536, 100000]))
    m1, m2 = int(rng.integers(2, 17)), int(rng.integers(2, 17))  # kMaxM = 16
    s1, s2 = float(rng.choice([1.25, 1.5, 2.0])), float(rng.choice([1.25, 1.5, 2.0]))
    M1 = int(rng.choice([1, 2, 31, 33, 100, 257, 1000, 4097, 20000, 100000]))
    M2 = int(rng.choice([1, 3, 64, 65, 999, 5000, 30000, 100000]))
    if LARGE:
        N = int(rng.choice([1 << 17, 3 << 16, 1 << 18, 2 * 131101, 1 << 19, 1000000, 1 << 20]))
        M1 = int(rng.choice([200000, 1000000, 1 << 21, 3000001]))
        M2 = int(rng.choice([65, 200000, 1000000, 1 << 21]))
    kv, kx = int(rng.integers(0, 5)), int(rng.integers(0, 5))
    v, x = nodes(M1, kv), nodes(M2, kx)
    B = int(rng.choice([0, 0, 0, 2, 5, 16, 33]))
    if LARGE and B > 5:
        B = 16 if M1 <= 1000000 and M2 <= 1000000 else 0
    desc = f"N={N} m=({m1},{m2}) s=({s1},{s2}) M=({M1},{M2}) kinds=({kv},{kx}) B={B}"
    route = int(rng.integers(0, 10))
    if route <= 5:  # NNFFT forward (+ adjoint on some)
        n, vs = sf.rescale_frequencies(N, v, s1, m1)
        plan = sf.nnfft_plan(n, vs, x, sigma1=s1, sigma2=s2, m1=m1, m2=m2)
        tab = O.plan(n, vs, x, sigma1=s1, sigma2=s2, m1=m1, m2=m2)
        shape = (M1, B) if B else (M1,)
        f = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        if rng.integers(0, 3) == 0:
            # device pointers: plan from CUDA tensors, the execute captured into a CUDA
            # graph on the first call and replayed on the second (capi.cu launch_graph)
            import torch
            plan = sf.nnfft_plan(n, torch.from_numpy(vs).cuda(), torch.from_numpy(x).cuda(),
                                 sigma1=s1, sigma2=s2, m1=m1, m2=m2)
            df = torch.from_numpy(f).cuda()
            first = sf.nnfft_trafo(plan, df).cpu().numpy()
            out = sf.nnfft_trafo(plan, df).cpu().numpy()
            rep = float(np.max(np.abs(out - first)) / np.sum(np.abs(f)) * max(B, 1))
            # run-to-run: the grid is summed with fp64 atomics, so the last bits of the
            # grid vary, amplified by 1/phi_hat like any rounding of the grid
            amp_r = float(tab.hat2.max() / tab.hat2.min() * tab.hat1.max() / tab.hat1.min())
            note("graph_replay", rep, desc + f" amp={amp_r:.1e}", 1e-15 + 1e-16 * amp_r)
            desc += " device"
        else:
            out = sf.nnfft_trafo(plan, f)
        cols = sorted({0, B - 1}) if B else [None]
        err = 0.0
        for b in cols:
            fb = f if b is None else np.ascontiguousarray(f[:, b])
            ob = out if b is None else out[:, b]
            ref = O.trafo(tab, fb)
            e = float(np.max(np.abs(ob - ref)) / np.sum(np.abs(fb)))
            if e > TOL:
                # ill-conditioned parameter sets -- phi_hat_2 spanning 1e4+ (sigma2 = 5/4
                # with a long window), or m1 = 2 with sources exactly on grid points (the
                # edge tap ~ sqrt(d) turns the 1e-11 rounding of the cell offset d into
                # 1e-9 of tap value): the reference's own rounding noise exceeds 1e-12.
                # Then the GPU must be as close to the EXACT sum as the reference is (to
                # within a tenth of that noise: with one or two nodes either side may be
                # the luckier one) and the mismatch must be explained by the noise
                sel = np.unique(np.linspace(0, M2 - 1, 200).astype(int))
                exact = O.nndft_direct(fb, vs, x[sel], n)
                ge = float(np.max(np.abs(ob[sel] - exact)) / np.sum(np.abs(fb)))
                oe = float(np.max(np.abs(ref[sel] - exact)) / np.sum(np.abs(fb)))
                amp = float(tab.hat2.max() / tab.hat2.min() * tab.hat1.max() / tab.hat1.min())
                print(f"cond: gpu-oracle {e:.2e} (amplification {amp:.1e}); vs exact sum: "
                      f"gpu {ge:.2e}, oracle {oe:.2e}", flush=True)
                worst["cond_gpu_vs_exact"] = max(worst.get("cond_gpu_vs_exact", 0.0), ge)
                # (noise model as for the NFFT below: window arguments known to
                # ~eps * grid size cells, times the 1/phi_hat amplification)
                G = tab.geo
                noise = amp * (max(1e-13, 4e-16 * max(G.N1, G.N2)) +
                               edge_noise(G.m1, G.sigma1, G.N1) + edge_noise(G.m2, G.sigma2, G.N2))
                e = 0.0 if ge <= 1.5 * oe + 1e-12 + 1e-16 * amp + noise / 10 and e <= noise else e
            err = max(err, e)
        note("nnfft", err, desc)
        if route == 5 and not B:
            y = rng.standard_normal(M2) + 1j * rng.standard_normal(M2)
            adj = sf.nnfft_adjoint(plan, y)
            err = float(np.max(np.abs(adj - O.adjoint(tab, y))) / np.sum(np.abs(y)))
            G = tab.geo  # the same conditioning as the forward transform (see above)
            amp = float(tab.hat2.max() / tab.hat2.min() * tab.hat1.max() / tab.hat1.min())
            noise = amp * (max(1e-13, 4e-16 * max(G.N1, G.N2)) +
                           edge_noise(G.m1, G.sigma1, G.N1) + edge_noise(G.m2, G.sigma2, G.N2))
            if err > TOL:  # as for the forward transform: both against the exact adjoint sum
                sel = np.unique(np.linspace(0, M1 - 1, 200).astype(int))
                exact = np.conj(O.nndft_direct(np.conj(y), x, vs[sel], n))
                ge = float(np.max(np.abs(adj[sel] - exact)) / np.sum(np.abs(y)))
                oe = float(np.max(np.abs(O.adjoint(tab, y)[sel] - exact)) / np.sum(np.abs(y)))
                print(f"cond: adjoint gpu-oracle {err:.2e} (amplification {amp:.1e}); vs exact "
                      f"sum: gpu {ge:.2e}, oracle {oe:.2e}", flush=True)
                err = 0.0 if ge <= 1.5 * oe + 1e-12 + 1e-16 * amp + noise / 10 and err <= noise else err
            note("nnfft_adjoint", err, desc + f" amp={amp:.1e}")
    elif route <= 7:  # NFFT trafo and adjoint
        s, m = s1, m1
        plan = sf.nfft_plan(N, x, sigma=s, m=m)
        tab = O.nfft_plan(N, x, sigma=s, m=m)
        cc = rng.standard_normal(N) + 1j * rng.standard_normal(N)
        err = float(np.max(np.abs(sf.nfft_trafo(plan, cc) - O.nfft_trafo(tab, cc))) /
                    np.sum(np.abs(cc)))
        # what two correct fp64 implementations can differ by: 1/phi_hat spans amp, so
        # the window values' rounding is worth ~amp * 1e-13; and half an ulp of a node
        # position (the cell offset is n_over x - floor(n_over x) here, x - l / n_over
        # in the reference) moves the phase at |k| = N/2 by ~pi N eps / 2 -- visible
        # when a handful of nodes carry all of sum |y|
        amp = float(tab.hat.max() / tab.hat.min())
        # -- and the window ARGUMENT of a node is only known to ~eps * n_over cells
        # on either side (the reference rounds l / n_over, the GPU n_over x), which
        # the O(1) window slope and 1/phi_hat turn into amp * eps * n_over per node
        tol = max(TOL, amp * (max(1e-13, 2.5e-16 * s * N) + edge_noise(m, s, s * N)))
        note("nfft", err, f"N={N} m={m} s={s} M={M2} kind={kx} amp={amp:.1e}", tol)
        y = rng.standard_normal(M2) + 1j * rng.standard_normal(M2)
        err = float(np.max(np.abs(sf.nfft_adjoint(plan, y) - O.nfft_adjoint(tab, y))) /
                    np.sum(np.abs(y)))
        note("nfft_adjoint", err, f"N={N} m={m} s={s} M={M2} kind={kx} amp={amp:.1e}", tol)
    else:  # fast sinc transform (general layout; the equispaced ones have fixtures)
        Ns = int(rng.choice([8, 30, 64, 200, 1000]))
        if LARGE:  # dense moment spread: hundreds of sources per cell
            M1, M2 = min(M1, 1000000), min(M2, 200000)
        a = nodes(2 * ((min(M1, 1000000 if LARGE else 20000) + 1) // 2), kv)  # even lengths (fast_sinc.py:131)
        b = nodes(2 * ((min(M2, 200000 if LARGE else 20000) + 1) // 2), kx)
        m = int(rng.integers(3, 11))
        sp = sf.sinc_plan(Ns, a, b, m1=m, m2=m)
        st = O.sinc_plan(Ns, a, b, m1=m, m2=m)
        cv = rng.standard_normal(a.size)
        err = float(np.max(np.abs(sf.fast_sinc_transform(sp, cv) - O.sinc_transform(st, cv))) /
                    np.sum(np.abs(cv)))
        note("fast_sinc", err, f"N={Ns} m={m} L=({a.size},{b.size}) kinds=({kv},{kx})")

c = 0
while c - rejected < cases and c < 20 * cases:  # `cases` accepted parameter sets
    c += 1
    try:
        one_case(c)
    except sf.ParameterError as e:
        # a parameter set the reference rejects (error parity has its own tests)
        rejected += 1
        print(f"rej {type(e).__name__}: {e}", flush=True)
print("fuzz ok:", cases, "cases,", rejected, "rejected by the parameter checks; worst", {k: f"{v:.2e}" for k, v in worst.items()})
