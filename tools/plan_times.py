"""dev helper (GPU box): where the plan time goes.  Times nnfft_plan at one
config from numpy inputs (host checks + H2D + device build) and from CUDA
tensors (device build only), with SFB_PLAN_TIMING=1 printing the C-side stages.

    python tools/plan_times.py 3
"""
import os
import sys
import time

os.environ.setdefault("SFB_PLAN_TIMING", "1")
import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2107_02671_b200 as sf  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "3"]
v, x, f = bench.make_inputs(cfg)
n_star, vs = sf.rescale_frequencies(cfg["N"], v, 2.0, cfg["m"])
torch.cuda.init()
torch.zeros(1, device="cuda")
for rep in range(3):
    t0 = time.perf_counter()
    plan = sf.nnfft_plan(n_star, vs, x, m1=cfg["m"], m2=cfg["m"], device=0)
    torch.cuda.synchronize()
    print(f"numpy inputs, rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del plan
dv = torch.from_numpy(vs).cuda()
dx = torch.from_numpy(x).cuda()
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = sf.nnfft_plan(n_star, dv, dx, m1=cfg["m"], m2=cfg["m"])
    torch.cuda.synchronize()
    print(f"CUDA tensors, rep {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    del plan
