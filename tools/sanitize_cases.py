"""GPU box, under compute-sanitizer (one --tool per gpurun call) or with the
bounds-checked library (make EXTRA=-DSFB_BOUNDS=1, SINCFFT_B200_LIB=...):
small invocations that launch every hot kernel once, each checked against
the oracle so a silent corruption also fails the run.

    compute-sanitizer --tool memcheck|racecheck|synccheck python tools/sanitize_cases.py

Kernels covered: k_spread (per-source spread), k_spread_dense (moment spread,
forced with SFB_SPREAD_DENSE=1), k_spread_small, the register FFT passes of
the config-3 shape (k_colfwd_r1 / k_rowmul_r1 / k_colinv_r1 + k_bluestein_fix:
N = 2^20 gives the 4096 x 1024 Bluestein regardless of the node count),
k_gather2 (TMA-staged span), the batched path of the config-4 shape
(k_spread_bw, k_*_rb, k_gather_b), and the fast sinc transform."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_02671_b200 as sf  # noqa: E402
from oracle import sincfft_oracle as O  # noqa: E402
from tests.inputs import nodes_and_coeffs  # noqa: E402


def check(name, got, ref, f, tol=1e-12):
    err = float(np.max(np.abs(got - ref)) / np.sum(np.abs(f)))
    print(f"{name}: rel err {err:.2e}", flush=True)
    assert err <= tol, name


def nnfft(name, N, M, m, clustered=False, batch=0, env=None):
    for k, v in (env or {}).items():
        os.environ[k] = v
    v, x, f = nodes_and_coeffs(N + M, M, M, clustered=clustered, batch=batch)
    n_star, vs = sf.rescale_frequencies(N, v, 2.0, m)
    plan = sf.nnfft_plan(n_star, vs, x, m1=m, m2=m, device=0)
    out = sf.nnfft_trafo(plan, f)
    tab = O.plan(n_star, vs, x, m1=m, m2=m)
    if batch:
        for b in (0, batch - 1):
            check(f"{name} col {b}", out[:, b], O.trafo(tab, f[:, b]), f[:, b])
    else:
        check(name, out, O.trafo(tab, f), f)
    for k in (env or {}):
        del os.environ[k]


which = sys.argv[1:] or ["c3shape", "dense", "small", "c4shape", "sinc"]
if "c3shape" in which:   # k_spread, register FFT passes (4096 x 1024), k_gather2
    nnfft("config-3 shape, 2^18 nodes", 1 << 20, 1 << 18, 8, clustered=True)
if "dense" in which:     # k_spread_dense forced
    nnfft("moment spread", 256, 1 << 14, 8, env={"SFB_SPREAD_DENSE": "1"})
if "small" in which:     # k_spread_small + direct FFT (k_dstep1/2)
    nnfft("config-1", 256, 1024, 4)
if "c4shape" in which:   # batched path: k_spread_b, k_*_rb passes, k_gather_b
    nnfft("config-4 shape, 16 columns", 65536, 1 << 12, 6, batch=16)
if "sinc" in which:
    rng = np.random.default_rng(5)
    a, b = rng.uniform(-0.5, 0.5, 1 << 14), rng.uniform(-0.5, 0.5, 1 << 12)
    c = rng.standard_normal(1 << 14)
    got = sf.fast_sinc_transform(sf.sinc_plan(256, a, b, m1=8, m2=8, device=0), c)
    check("fast sinc", got, O.sinc_transform(O.sinc_plan(256, a, b, m1=8, m2=8), c), c)
print("sanitize cases done")
