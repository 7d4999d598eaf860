"""dev helper (GPU box): per-call host latency of the pipelined host-buffer
e2e loop (config 3 shapes) to locate sporadic stalls."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2107_02671_b200 as sf  # noqa: E402
from paper_2107_02671_b200 import _lib  # noqa: E402
from tests.inputs import nodes_and_coeffs  # noqa: E402

M = 1 << 24
v, x, f = nodes_and_coeffs(0, M, M, clustered=True)
N, vs = sf.rescale_frequencies(1 << 20, v, 2.0, 8)
plan = sf.nnfft_plan(N, vs, x, m1=8, m2=8)
nb = int(sys.argv[1]) if len(sys.argv) > 1 else 4
hf = [torch.from_numpy(f).pin_memory() for _ in range(nb)]
ho = [torch.empty(M, dtype=torch.complex128).pin_memory() for _ in range(nb)]
st = [torch.cuda.Stream() for _ in range(nb)]
L = _lib.lib
for rep in range(int(sys.argv[2]) if len(sys.argv) > 2 else 3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    lat = []
    for k in range(40):
        a = time.perf_counter()
        _lib.check(L.sincfft_nnfft_execute(plan.handle, hf[k % nb].data_ptr(), ho[k % nb].data_ptr(),
                                           1, _lib.PTR_HOST_ASYNC, C.c_void_p(st[k % nb].cuda_stream)))
        lat.append((time.perf_counter() - a) * 1e3)
    torch.cuda.synchronize()
    tot = (time.perf_counter() - t0) * 1e3 / 40
    print(f"rep {rep}: {tot:.3f} ms/step; host call ms: max {max(lat):.3f} "
          f"median {np.median(lat):.3f} top {sorted(lat)[-4:]}")
