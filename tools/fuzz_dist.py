"""dev helper (GPU box): randomized check of the three distributed-FFT
realisations (dense reduce-scatter / all-gather, sparse row exchange, fused
peer transposes) with every rank of a P-way split run in THIS process
(sharding.run_*_in_process), against the unsharded transform of the same
inputs: random bandwidths (whatever FFT shape the planner picks), cut-offs,
oversampling factors, node counts and layouts, P in {2, 4, 8}, index and
position partitions.  Plans the distributed kernels do not cover
(dist_layout None) are counted, not failed.

    python tools/fuzz_dist.py [cases] [seed]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_02671_b200 as sf  # noqa: E402
from paper_2107_02671_b200 import sharding as sh  # noqa: E402
from oracle import sincfft_oracle as O  # noqa: E402  (phi_hat for the tolerance)

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 3)
worst, done, skipped = 0.0, 0, 0
attempt = 0
while done < cases and attempt < 20 * cases:
    attempt += 1
    # (the distributed kernels cover the 4096 x 1024 Bluestein shape, fft.cu dist_shape():
    # bandwidths around 2^20 at sigma = 2 and their neighbours; the rest is skipped)
    N = int(rng.choice([1 << 19, 3 << 18, 1000000, (1 << 20) - 64, 1 << 20, 1 << 20, 1 << 20]))
    m1, m2 = int(rng.integers(2, 13)), int(rng.integers(2, 13))
    s1, s2 = float(rng.choice([1.5, 2.0, 2.0])), float(rng.choice([1.25, 1.5, 2.0, 2.0]))
    M1 = int(rng.choice([64, 1000, 4097, 50000, 300000]))
    M2 = int(rng.choice([64, 999, 5000, 60000, 300000]))
    world = int(rng.choice([2, 4, 8]))
    clustered = bool(rng.integers(0, 2))
    u, w = rng.random(M1), rng.random(M2)
    v = 0.5 * np.cos(np.pi * u) if clustered else u - 0.5
    x = 0.5 * np.cos(np.pi * w) if clustered else w - 0.5
    if rng.integers(0, 4) == 0:
        x = 0.2 + 1e-3 * (w - 0.5)  # targets in a few cells
    f = rng.standard_normal(M1) + 1j * rng.standard_normal(M1)
    try:
        n, vs = sf.rescale_frequencies(N, v, s1, m1)
        full = sf.nnfft_plan(n, vs, x, sigma1=s1, sigma2=s2, m1=m1, m2=m2, device=0)
    except sf.ParameterError:
        continue
    ref = sf.nnfft_trafo(full, f)
    by_pos = bool(rng.integers(0, 2))
    sv = np.argsort(vs, kind="stable") if by_pos else np.arange(M1)
    sx = np.argsort(x, kind="stable") if by_pos else np.arange(M2)
    kind = int(rng.integers(0, 3))
    cls, run = [(sh.DistFftRank, sh.run_ranks_in_process),
                (sh.SparseDistFftRank, sh.run_sparse_ranks_in_process),
                (sh.PeerDistFftRank, sh.run_peer_ranks_in_process)][kind]
    ranks, shards, tidx = [], [], []
    ok = True
    for r in range(world):
        s0, s1_ = sh.shard_range(M1, world, r)
        t0, t1 = sh.shard_range(M2, world, r)
        si, ti = sv[s0:s1_], sx[t0:t1]
        if si.size == 0 or ti.size == 0:
            ok = False
            break
        plan = sf.nnfft_plan(n, vs[si], x[ti], sigma1=s1, sigma2=s2, m1=m1, m2=m2, device=0,
                             h_window="full")
        if sh.dist_layout(plan, world) is None:
            ok = False
            break
        ranks.append(cls(plan, world, r))
        shards.append(torch.from_numpy(np.ascontiguousarray(f[si])).to("cuda:0"))
        tidx.append(ti)
    desc = (f"N={N} m=({m1},{m2}) s=({s1},{s2}) M=({M1},{M2}) P={world} "
            f"{'pos' if by_pos else 'idx'} {cls.__name__}")
    if not ok:
        skipped += 1
        print("skip (no distributed layout)", desc, flush=True)
        continue
    outs = run(ranks, shards)
    err = max(float(np.max(np.abs(o.cpu().numpy() - ref[ti]))) for o, ti in zip(outs, tidx))
    err /= float(np.sum(np.abs(f)))
    # sharded vs unsharded runs of the SAME kernels: only the summation order of
    # the grid differs, amplified by 1/phi_hat_2 like any rounding of the grid
    g = full.backend_geometry
    geo = full.geometry
    K = geo.N1 + 2 * geo.m1
    hat = O.phi_hat_sinh(O.sinh_beta(geo.m2, geo.sigma2), geo.m2, geo.N2,
                         np.array([0.0, float(K // 2)]))
    tol = 1e-13 * max(1.0, float(hat[0] / hat[1]) / 100.0)
    done += 1
    worst = max(worst, err)
    print(f"{'ok ' if err <= tol else 'BAD'} {err:.2e} (tol {tol:.1e}) {desc} "
          f"L={g['L1']}x{g['L2']}", flush=True)
    if err > tol:
        raise SystemExit("distributed result differs from the unsharded transform")
print(f"dist fuzz ok: {done} cases ({skipped} plans without a distributed layout), "
      f"worst {worst:.2e}")
