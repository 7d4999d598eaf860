"""dev helper: in-stream kernel durations (CUPTI via torch.profiler, no
serialisation or cache flushing, unlike ncu) of one config's step.

    python tools/kernel_times.py 5      # fast sinc, config 5
    python tools/kernel_times.py 3      # NNFFT, config 3
"""
import ctypes as C
import os
import sys
from collections import defaultdict

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2107_02671_b200 as sf  # noqa: E402
from paper_2107_02671_b200 import _lib  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "5"]
dev = torch.device("cuda", 0)
s = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
v, x, f = bench.make_inputs(cfg)
# ablation: KT_SORT=v / x / vx presents the sources / targets already sorted by
# position, so the spread's f gather / the gather's output scatter are sequential
srt = os.environ.get("KT_SORT", "")
if "v" in srt:
    o = np.argsort(v, kind="stable")
    v, f = v[o], f[o]
if "x" in srt:
    x = np.sort(x)
if cfg.get("sinc"):
    plan = sf.sinc_plan(cfg["N"], v, x, m1=cfg["m"], m2=cfg["m"], device=0)
    d_c = torch.from_numpy(np.ascontiguousarray(f.real)).to(dev)
    d_out = torch.empty(cfg["M2"], dtype=torch.complex128, device=dev)

    def step():
        _lib.check(_lib.lib.sincfft_sinc_execute(plan.handle, d_c.data_ptr(), 1,
                                                 d_out.data_ptr(), _lib.PTR_DEVICE, s))
else:
    n_star, vs = sf.rescale_frequencies(cfg["N"], v, 2.0, cfg["m"])
    plan = sf.nnfft_plan(n_star, vs, x, m1=cfg["m"], m2=cfg["m"], device=0)
    d_f = torch.from_numpy(np.ascontiguousarray(f)).to(dev)
    B = max(cfg["batch"], 1)
    d_out = torch.empty((cfg["M2"],) + ((B,) if cfg["batch"] else ()), dtype=torch.complex128,
                        device=dev)

    def step():
        _lib.check(_lib.lib.sincfft_nnfft_execute(plan.handle, d_f.data_ptr(), d_out.data_ptr(),
                                                  B, _lib.PTR_DEVICE, s))
for _ in range(5):
    step()
torch.cuda.synchronize()
steps = 20
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
tot = defaultdict(float)
cnt = defaultdict(int)
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        tot[e.name] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
        cnt[e.name] += 1
for k, t in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{t / steps:9.2f} us/step  x{cnt[k] // steps}  {k[:100]}")
print(f"{sum(tot.values()) / steps:9.2f} us/step total kernel time")
# variant runs (tools/run_variants.sh): the first run saves its output, later
# runs report their max deviation from it (relative to sum|f|)
ref = os.environ.get("VAR_REF")
if ref:
    out = d_out.cpu().numpy()
    if os.path.exists(ref):
        base = np.load(ref)
        fl1 = float(np.abs(np.asarray(d_c.cpu() if cfg.get("sinc") else d_f.cpu())).sum())
        print(f"max|out - base| / sum|f| = {float(np.max(np.abs(out - base))) / fl1:.3e}")
    else:
        np.save(ref, out)
