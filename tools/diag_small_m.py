"""dev diagnostic (GPU box): error split for a large grid with few nodes
(N = 2^20, M = 2^15, m = 8, clustered): GPU vs oracle, and both vs the exact
direct sum on 256 targets, relative to sum|f| and to |f|_2."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2107_02671_b200 as sf  # noqa: E402
from oracle import sincfft_oracle as O  # noqa: E402
from tests.inputs import nodes_and_coeffs  # noqa: E402

for N, M in ((1 << 20, 1 << 15), (1 << 20, 1 << 18), (1 << 16, 1 << 12)):
    v, x, f = nodes_and_coeffs(N + M, M, M, clustered=True)
    n_star, vs = sf.rescale_frequencies(N, v, 2.0, 8)
    out = sf.nnfft_trafo(sf.nnfft_plan(n_star, vs, x, m1=8, m2=8, device=0), f)
    ref = O.trafo(O.plan(n_star, vs, x, m1=8, m2=8), f)
    idx = np.arange(0, M, M // 256)
    ex = sf.nndft_direct(f, v, x[idx], N)
    l1, l2 = np.abs(f).sum(), np.linalg.norm(f)
    print(f"N={N} M={M}: gpu-oracle {np.max(np.abs(out-ref))/l1:.2e} (|f|_1) "
          f"{np.max(np.abs(out-ref))/l2:.2e} (|f|_2); gpu-exact {np.max(np.abs(out[idx]-ex))/l1:.2e}; "
          f"oracle-exact {np.max(np.abs(ref[idx]-ex))/l1:.2e}; bound "
          f"{O.bound_nnfft_sinh(n_star, 2.0, 2.0, 8, 8):.2e}", flush=True)
