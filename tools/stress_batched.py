"""dev helper (GPU box): randomized stress of the column-vectorised path
(k_spread_bw / k_*_b / k_gather_b) against the single-column kernels on the
same plan: random N, node counts, cut-offs, batch widths, clustered or
uniform nodes; every column must agree to rounding.

    python tools/stress_batched.py [cases] [seed]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_02671_b200 as sf  # noqa: E402

cases = int(sys.argv[1]) if len(sys.argv) > 1 else 40
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
worst = 0.0
for c in range(cases):
    N = int(rng.choice([64, 200, 700, 1024, 5000, 65536]))
    m = int(rng.integers(2, 17))
    M1 = int(rng.choice([1, 5, 31, 33, 257, 1000, 4097, 30000, 200000]))
    M2 = int(rng.choice([1, 7, 64, 65, 999, 5000, 50000]))
    B = int(rng.choice([16, 17, 31, 32, 33, 64, 127, 128, 129, 200, 256, 257]))
    clustered = bool(rng.integers(0, 2))
    u, w = rng.random(M1), rng.random(M2)
    v = 0.5 * np.cos(np.pi * u) if clustered else u - 0.5
    x = 0.5 * np.cos(np.pi * w) if clustered else w - 0.5
    if rng.integers(0, 4) == 0:  # all sources in a few cells
        v = v * 1e-3
    f = rng.standard_normal((M1, B)) + 1j * rng.standard_normal((M1, B))
    n, vs = sf.rescale_frequencies(N, v, 2.0, m)
    plan = sf.nnfft_plan(n, vs, x, m1=m, m2=m)
    out = sf.nnfft_trafo(plan, f)
    cols = sorted({0, B - 1, int(rng.integers(0, B)), min(B - 1, 128)})
    err = 0.0
    for b in cols:
        one = sf.nnfft_trafo(plan, np.ascontiguousarray(f[:, b]))
        err = max(err, float(np.max(np.abs(out[:, b] - one)) / np.sum(np.abs(f[:, b]))))
    worst = max(worst, err)
    print(f"case {c}: N={N} m={m} M1={M1} M2={M2} B={B} clustered={clustered} err={err:.2e}",
          flush=True)
    assert err <= 1e-13, "batched and single-column paths disagree"
print(f"stress ok: {cases} cases, worst {worst:.2e}")
