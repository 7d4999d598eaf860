#!/usr/bin/env python
"""Benchmark of the B200 NNFFT hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config 3|1|2|4|5]

A "step" is one NNFFT execute (Algorithm 2.1 steps 1-4, ``nnfft_trafo``) over
the workload's nodes with the plan (step 0) built beforehand, exactly how the
reference is used (plan once, transform many).  Default workload: config 3 of
BASELINE.json (N = 2^20, M1 = M2 = 2^24, m1 = m2 = 8, sigma = 2, clustered
nodes 0.5 cos(pi u), complex128) -- the largest single-GPU configuration and
the one the north star's scaling target names.

* ``value``: (M1 + M2) nodes/s over K device-timed steps, inputs resident in
  HBM, CUDA events on the launching stream, max over ranks.
* ``e2e``: same metric through the C ABI with pinned HOST buffers (H2D of f
  and D2H of the output inside the timed region); the K-step region is timed
  E2E_REPEATS times and the median reported (every repeat in ``repeats_ms``).
* ``roofline``: algorithmic bytes of the dominant kernel over
  its CUDA-event duration measured live, against MEASURED_PEAKS.json.
* ``cpu_baseline``: the CPU oracle (a restatement of the reference; the
  reference itself is pure single-threaded numpy/scipy) on a bounded sample.

N > 1 (torchrun): the one config-3 problem is split -- each rank spreads
M1/N sources and gathers M2/N targets; the partial K-grids are summed with
one NCCL all-reduce (the path's only exchange step); the FFT is
replicated.  ``scaling`` is "strong".
"""

import argparse
import ctypes as C
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
E2E_REPEATS = 3  # timed e2e regions per run; the median is reported
sys.path.insert(0, ROOT)

METRIC = "NNFFT (M1+M2) nodes/sec fp64 at 1/2/4/8 B200; % of HBM roofline"

CONFIGS = {
    "1": dict(N=256, M1=1024, M2=1024, m=4, clustered=False, batch=0,
              desc="config1: NNFFT N=256, M1=M2=1024, m1=m2=4, sigma=2, uniform nodes"),
    "2": dict(N=4096, M1=65536, M2=65536, m=8, clustered=False, batch=0,
              desc="config2: NNFFT N=4096, M1=M2=65536, m1=m2=8, sigma=2, uniform nodes"),
    "3": dict(N=1 << 20, M1=1 << 24, M2=1 << 24, m=8, clustered=True, batch=0,
              desc="config3: NNFFT N=2^20, M1=M2=2^24, m1=m2=8, sigma=2, clustered nodes "
                   "0.5cos(pi u), complex128"),
    "4": dict(N=65536, M1=1 << 20, M2=1 << 20, m=6, clustered=False, batch=256,
              desc="config4: batched NNFFT N=65536, M1=M2=2^20, 256 columns, m1=m2=6"),
    "5": dict(N=4096, M1=1 << 22, M2=1 << 22, m=8, clustered=False, batch=0, sinc=True,
              desc="config5: fast sinc transform N=4096, L1=L2=2^22 uniform nodes, c real, "
                   "n=4N Clenshaw-Curtis, m1=m2=8, sigma=2"),
}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """Polls NVML during the timed region (sm clock, max clock, throttle reasons)."""

    REASONS = {
        "hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "sw_power_cap": 0x4, "sync_boost": 0x10,
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_inputs(cfg, seed=0):
    from tests.inputs import nodes_and_coeffs
    return nodes_and_coeffs(seed, cfg["M1"], cfg["M2"], clustered=cfg["clustered"],
                            batch=cfg["batch"])


def cpu_info():
    """The host the CPU leg ran on: core count, model, and the core this
    process is pinned to (os.sched_setaffinity, i.e. taskset -c)."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    aff = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None
    return {"nproc": os.cpu_count(), "cpu_model": model, "affinity": aff}


def pin_one_core():
    """taskset -c <core>: the reference is single-threaded numpy/scipy
    (SURVEY.md 8d), so it is timed on one pinned core; the first core of the
    inherited affinity set is used."""
    if hasattr(os, "sched_setaffinity"):
        core = min(os.sched_getaffinity(0))
        os.sched_setaffinity(0, {core})


def cpu_sample_rate(cfg, steps=1, warmup=0, sample_nodes=1 << 22, budget_s=None):
    """Time the CPU oracle's trafo (single-threaded numpy/scipy, like the
    reference) pinned to one core: the workload's geometry (N, m) with
    sample_nodes sources and targets drawn the same way (the full workload
    when sample_nodes >= M1, with the workload's own seed).  With budget_s the
    run is bounded in wall time on a slow host: warm-ups stop (after one) at a
    quarter of the budget, timed steps (after two) at the budget; the counts
    actually run are reported."""
    from oracle import sincfft_oracle as O
    pin_one_core()
    M = min(sample_nodes, cfg["M1"])
    full = M == cfg["M1"]
    sub = dict(cfg, M1=M, M2=M, batch=0)
    t_start = time.perf_counter()
    v, x, f = make_inputs(sub, seed=0 if full else 1)
    n_star, vs = O.rescale_frequencies(cfg["N"], v, 2.0, cfg["m"])
    t0 = time.perf_counter()
    tab = O.plan(n_star, vs, x, m1=cfg["m"], m2=cfg["m"])
    t_plan = time.perf_counter() - t0

    def spent(frac):
        return budget_s is not None and time.perf_counter() - t_start > frac * budget_s

    warm_run = 0
    for _ in range(warmup):
        if warm_run >= 1 and spent(0.25):
            break
        O.trafo(tab, f)
        warm_run += 1
    ts = []
    for _ in range(steps):
        if len(ts) >= 2 and spent(1.0):
            break
        t0 = time.perf_counter()
        O.trafo(tab, f)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    steps, warmup = len(ts), warm_run
    info = cpu_info()
    return {"value": 2 * M / t, "unit": "nodes/s", "cores": 1, "kind": "port",
            "sample": (f"oracle trafo (restatement of the reference's nnfft_trafo, pinned to "
                       f"core {info['affinity']}), N={cfg['N']}, m={cfg['m']}, M1=M2={M} "
                       f"({'clustered' if cfg['clustered'] else 'uniform'}"
                       f"{', the full workload, seed 0' if full else ', a bounded sample'}), "
                       f"median of {steps} after {warmup} warm-up, plan {t_plan:.1f}s untimed"),
            "same_config": full, "plan_s": t_plan, **info,
            "seconds_per_step": t}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # the reference's own CPU path on the same workload as the B200 arm: the
    # full configuration (config 3: ~45 s of plan, ~17 s per trafo on one core)
    # (bounded at ~4 minutes of wall time on a slow host: fewer steps, same workload)
    base = cpu_sample_rate(cfg, steps=args.steps, warmup=args.warmup, sample_nodes=cfg["M1"],
                           budget_s=args.ref_budget_s)
    line = {"metric": METRIC, "value": base["value"], "unit": "nodes/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": base["seconds_per_step"] * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "sample": base["sample"],
                       "same_config": base["same_config"]},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample",
                                                  "nproc", "cpu_model", "affinity")},
            "e2e": {"value": base["value"], "unit": "nodes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_sinc_b200(args, cfg):
    """Config 5: one fast_sinc_transform per step (two NNFFTs), device pointers."""
    import torch
    import paper_2107_02671_b200 as sf
    from paper_2107_02671_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)
    rng = np.random.default_rng(0)
    a_all = rng.uniform(-0.5, 0.5, cfg["M1"])
    b_all = rng.uniform(-0.5, 0.5, cfg["M2"])
    c_all = rng.standard_normal(cfg["M1"])
    # N > 1: sources and targets partitioned by position (quantile ranges);
    # stage 1 is linear in c, so the ranks' partial alphas at the n+1
    # Clenshaw-Curtis nodes are summed with ONE all-reduce of (n+1) complex,
    # then every rank evaluates its own targets (sincfft_sinc_stage1/3)
    si = np.argsort(a_all, kind="stable")[rank * cfg["M1"] // world:(rank + 1) * cfg["M1"] // world]
    ti = np.argsort(b_all, kind="stable")[rank * cfg["M2"] // world:(rank + 1) * cfg["M2"] // world]
    if world == 1:
        si = ti = slice(None)
    a, b, c = a_all[si], b_all[ti], np.ascontiguousarray(c_all[si])
    tp = time.perf_counter()
    plan = sf.sinc_plan(cfg["N"], a, b, m1=cfg["m"], m2=cfg["m"], device=local)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - tp) * 1e3
    d_c = torch.from_numpy(c).to(dev)
    d_out = torch.empty(b.size, dtype=torch.complex128, device=dev)
    d_alpha = torch.empty(plan.n + 1, dtype=torch.complex128, device=dev)
    L = _lib.lib

    def step():
        if world == 1:
            _lib.check(L.sincfft_sinc_execute(plan.handle, d_c.data_ptr(), 1, d_out.data_ptr(),
                                              _lib.PTR_DEVICE, sh))
            return
        _lib.check(L.sincfft_sinc_stage1(plan.handle, d_c.data_ptr(), 1, d_alpha.data_ptr(), sh))
        if args.dist_backend != "nccl":
            torch.cuda.synchronize()
        dist.all_reduce(torch.view_as_real(d_alpha))
        if args.dist_backend != "nccl":
            torch.cuda.synchronize()
        _lib.check(L.sincfft_sinc_stage3(plan.handle, d_alpha.data_ptr(), d_out.data_ptr(), sh))

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    if dist:
        dist.barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    units = cfg["M1"] + cfg["M2"]
    shard_dev = None
    if world > 1 and args.check_shards:
        full = sf.sinc_plan(cfg["N"], a_all, b_all, m1=cfg["m"], m2=cfg["m"], device=local)
        ref = sf.fast_sinc_transform(full, c_all)[ti]
        shard_dev = float(np.max(np.abs(d_out.cpu().numpy() - ref)) / np.abs(c_all).sum())
        del full
    # end to end from pinned host buffers, pipelined like the NNFFT configs:
    # successive steps rotate over --e2e-streams streams (SINCFFT_PTR_HOST_ASYNC)
    # so the H2D of step k+1, the kernels of step k and the D2H of step k-1
    # overlap on the full-duplex PCIe link
    nbuf = args.e2e_streams if world == 1 else 1
    h_c = [torch.from_numpy(c).pin_memory() for _ in range(nbuf)]
    h_out = [torch.empty(b.size, dtype=torch.complex128).pin_memory() for _ in range(nbuf)]
    streams = [torch.cuda.Stream(dev) for _ in range(nbuf)] if world == 1 else [stream]

    def e2e_step(k):
        st = C.c_void_p(streams[k % nbuf].cuda_stream)
        if world == 1:
            _lib.check(L.sincfft_sinc_execute(plan.handle, h_c[k % nbuf].data_ptr(), 1,
                                              h_out[k % nbuf].data_ptr(), _lib.PTR_HOST_ASYNC,
                                              st))
            return
        d_c.copy_(h_c[0], non_blocking=True)  # sharded: H2D, stage 1, all-reduce, stage 3, D2H
        step()
        h_out[0].copy_(d_out, non_blocking=True)

    for k in range(max(3 * nbuf, args.warmup)):
        e2e_step(k)
    torch.cuda.synchronize()
    e2e_reps = []  # median of E2E_REPEATS timed regions, as in the NNFFT leg
    for _ in range(E2E_REPEATS):
        ev0.record(stream)
        for st in streams:
            st.wait_event(ev0)
        for k in range(args.steps):
            e2e_step(k)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            stream.wait_event(e)
        ev1.record(stream)
        ev1.synchronize()
        e2e_reps.append(max_over_ranks(ev0.elapsed_time(ev1) / args.steps))
    e2e_ms = float(np.median(e2e_reps))
    e2e_dev = float(np.max(np.abs(h_out[(args.steps - 1) % nbuf].numpy() - d_out.cpu().numpy()))
                    / np.abs(c).sum())
    if e2e_dev > 1e-13:
        print(f"WARNING: e2e output deviates from the device-resident output by {e2e_dev:.3e}",
              file=sys.stderr)
    g1, g3 = plan.stage_geometry()
    # algorithmic bytes: 16 L1 + 24 L2 + 64 (K + N2) + 56 (n+1)
    alg = 16 * cfg["M1"] + 24 * cfg["M2"] + 64 * (g1["K"] + g1["N2"]) + 56 * (plan.n + 1)
    peak, peak_kind = peaks()
    achieved = alg / (ms * 1e-3) / 1e9
    line = {"metric": "fast sinc transform (L1+L2) nodes/sec fp64", "value": units / (ms * 1e-3),
            "unit": "nodes/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "n_star": plan.n_star, "K": g1["K"],
                       "N2": g1["N2"], "fft_length_L": g1["L"],
                       "parallelism": f"sources+targets sharded x{world} by position"
                                      + ("; one all-reduce of the n+1 stage-1 values"
                                         if world > 1 else "")},
            "roofline": {"bound": "hbm", "kernel": "whole transform", "achieved": achieved,
                         "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "alg_bytes_per_launch": alg},
            "plan_ms": plan_ms,
            "e2e": {"value": units / (e2e_ms * 1e-3), "unit": "nodes/s",
                    "h2d_bytes_per_step": 8 * c.size, "d2h_bytes_per_step": 16 * b.size,
                    "ms_per_step": e2e_ms, "repeats_ms": e2e_reps,
                    "mode": (f"sincfft_sinc_execute(host pinned, PTR_HOST_ASYNC), {nbuf} "
                             "streams round-robin" if world == 1 else
                             "H2D, stage 1, all-reduce, stage 3, D2H on one stream")},
            "e2e_vs_device_rel_err": e2e_dev,
            "gpu_launches": 2 * 5 * args.steps, "clocks": clk.summary()}
    if shard_dev is not None:
        line["shard_check_rel_err"] = shard_dev
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_b200(args, cfg):
    import torch
    import paper_2107_02671_b200 as sf
    from paper_2107_02671_b200 import _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:  # functional test of the multi-rank path on one GPU
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(args.dist_backend)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    sh = C.c_void_p(stream.cuda_stream)

    v, x, f = make_inputs(cfg)
    m = cfg["m"]
    n_star, vs = sf.rescale_frequencies(cfg["N"], v, 2.0, m)
    # shard sources and targets (contiguous index ranges)
    s0, s1 = rank * cfg["M1"] // world, (rank + 1) * cfg["M1"] // world
    t0_, t1_ = rank * cfg["M2"] // world, (rank + 1) * cfg["M2"] // world
    # N > 1: sources and targets are partitioned by POSITION (quantile ranges
    # of v and x): a rank's sources fill 1/P of the K-grid at full density
    # (index shards of clustered nodes cover the whole grid at 1/P density:
    # sparse chunks, and every rank flushes the whole grid)
    src_idx = np.argsort(vs, kind="stable")[s0:s1] if world > 1 else slice(None)
    tgt_idx = np.argsort(x, kind="stable")[t0_:t1_] if world > 1 else slice(None)
    # batched configs shard the independent COLUMNS instead (no
    # communication; every rank plans all nodes and transforms B/P columns)
    col_shard = world > 1 and cfg["batch"] > 0
    c0 = c1 = 0
    if col_shard:
        src_idx = tgt_idx = slice(None)
        s0, s1, t0_, t1_ = 0, cfg["M1"], 0, cfg["M2"]
        c0, c1 = rank * cfg["batch"] // world, (rank + 1) * cfg["batch"] // world
    torch.cuda.synchronize()
    tp = time.perf_counter()
    # N > 1: the FFT is split over the ranks too (sharding.DistributedFftNnfft,
    # plans share one FFT via the geometric h window) unless --replicated-fft
    # or the plan shape is outside the distributed kernels' envelope
    want_dist = world > 1 and not cfg["batch"] and not args.replicated_fft
    plan = sf.nnfft_plan(n_star, vs[src_idx], x[tgt_idx], m1=m, m2=m, device=local,
                         h_window="full" if want_dist else "data")
    dist_fft = None
    if want_dist:
        from paper_2107_02671_b200.sharding import (DistributedFftNnfft,
                                                    SparseDistributedFftNnfft, dist_layout)
        if dist_layout(plan, world) is not None:
            # position partitions: exchange only the grid / h rows each rank
            # touches (sparse) unless --dense-exchange asks for the
            # reduce-scatter / all-gather form
            # default: the two transposes fused into the column / row passes
            # over peer memory (CUDA IPC, NVLink P2P between the node's GPUs)
            # default: NCCL all-to-alls of the rows each rank touches; the
            # kernels-store-into-peer-memory form (CUDA IPC) only on request
            # (--peer-transposes) until it has run across >= 2 GPUs
            if args.dense_exchange:
                dist_fft = DistributedFftNnfft(plan)
            elif args.peer_transposes:
                from paper_2107_02671_b200.sharding import PeerDistributedFftNnfft
                dist_fft = PeerDistributedFftNnfft(plan)
            else:
                dist_fft = SparseDistributedFftNnfft(plan)
    torch.cuda.synchronize()
    plan_ms = (time.perf_counter() - tp) * 1e3
    # the same plan built again (context, allocator pools and window fits warm):
    # what a caller whose nodes change every call pays per transform
    plan_warm_ms = None
    if world == 1:
        tp = time.perf_counter()
        plan2 = sf.nnfft_plan(n_star, vs, x, m1=m, m2=m, device=local)
        torch.cuda.synchronize()
        plan_warm_ms = (time.perf_counter() - tp) * 1e3
        del plan2
    geo = plan.backend_geometry
    B = max(cfg["batch"], 1)
    fshard = np.ascontiguousarray(f[src_idx])
    if col_shard:
        B = c1 - c0
        fshard = np.ascontiguousarray(f[:, c0:c1])
    d_f = torch.from_numpy(fshard).to(dev)
    d_out = torch.empty((t1_ - t0_,) + ((B,) if cfg["batch"] else ()), dtype=torch.complex128,
                        device=dev)
    d_grid = torch.empty((B, geo["K"]), dtype=torch.complex128, device=dev)
    L = _lib.lib
    ph = plan.handle

    def step():
        if world == 1 or col_shard:
            _lib.check(L.sincfft_nnfft_execute(ph, d_f.data_ptr(), d_out.data_ptr(), B,
                                               _lib.PTR_DEVICE, sh))
        elif dist_fft is not None:
            d_out.copy_(dist_fft(d_f))
        else:
            _lib.check(L.sincfft_nnfft_spread(ph, d_f.data_ptr(), d_grid.data_ptr(), B,
                                              _lib.PTR_DEVICE, sh))
            dist.all_reduce(torch.view_as_real(d_grid))
            _lib.check(L.sincfft_nnfft_finish(ph, d_grid.data_ptr(), d_out.data_ptr(), B,
                                              _lib.PTR_DEVICE, sh))

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps)
    total_nodes = (cfg["M1"] + cfg["M2"]) * max(cfg["batch"], 1)  # the whole job
    value = total_nodes / (ms * 1e-3)

    # the device-resident output of the timed steps (the per-stage profiling
    # below reuses d_out and, on a sharded plan, sees only the local sources)
    dev_out = d_out.cpu().numpy()
    shard_dev = None
    if args.check_shards and world > 1:
        # the unsharded transform of the same inputs (one plan over everything)
        full = sf.nnfft_plan(n_star, vs, x, m1=m, m2=m, device=local)
        ref = sf.nnfft_trafo(full, f)[tgt_idx]
        if col_shard:
            ref = ref[:, c0:c1]
        torch.cuda.synchronize()
        shard_dev = float(np.max(np.abs(dev_out - ref)) / np.abs(f).sum())
        del full

    # per-stage device times (spread / fft / gather), live, same stream
    # (sharded runs: the spread of the local sources + replicated FFT + local
    # gather; the all-reduce between them is not included)
    stage = np.zeros(4)
    buf = (C.c_double * 4)()
    nprof = max(3, min(args.steps, 20))
    for _ in range(nprof):
        _lib.check(L.sincfft_nnfft_execute_profiled(ph, d_f.data_ptr(), d_out.data_ptr(), B, sh,
                                                    buf))
        stage += np.array(buf[:])
    stage /= nprof
    names = ["spread", "fft", "gather"]
    K, N2, Ms, Mt = geo["K"], geo["N2"], s1 - s0, t1_ - t0_
    alg = {"spread": 8 * Ms + B * (16 * Ms + 16 * K),
           "fft": B * (16 * K + 16 * N2),
           "gather": 8 * Mt + B * (16 * N2 + 16 * Mt)}
    dom = names[int(np.argmax(stage[:3]))]
    t_dom = stage[names.index(dom)] * 1e-3
    peak, peak_kind = peaks()
    achieved = alg[dom] / t_dom / 1e9
    # FP64 side of the same kernel: the window polynomials + tap MACs are the
    # floor for spread/gather.  Counts per node from the
    # committed ncu capture (profiles/ncu_fp64.json, tools/ncu_pipes.sh:
    # sm__sass_thread_inst_executed_op_dfma / _fp64 per launch; a DFMA is 2
    # flops, any other fp64 instruction 1); without it, the kernel's structure
    # (window.cuh): m pairs x (P + 1) + 2 sqrt (~8 each) + 4m MACs
    P = 16 if m <= 2 else 15 if m <= 3 else 14 if m <= 6 else 13 if m <= 9 else 12
    dfma_node = m * (P + 1) + 16 + 4 * m * B
    fp64_node = {k: (dfma_node, 0, None, "kernel structure (window.cuh)")
                 for k in ("spread", "gather")}
    fj = os.path.join(ROOT, "profiles", "ncu_fp64.json")
    if world == 1 and os.path.exists(fj):
        with open(fj) as fh:
            nc = json.load(fh).get(f"config{args.config}", {})
        for k, d in nc.items():
            units = Ms if k == "spread" else Mt
            if d.get("dfma_thread_inst"):
                fp64_node[k] = (d["dfma_thread_inst"] / units,
                                (d["fp64_thread_inst"] - d["dfma_thread_inst"]) / units,
                                d.get("fp64_pipe_active_pct"), "ncu (profiles/ncu_fp64.json)")
    flops = {k: (2 * v[0] + v[1]) * (Ms if k == "spread" else Mt) for k, v in fp64_node.items()}
    flops["fft"] = None
    # DRAM bytes per launch of that kernel from the committed ncu capture --
    # single-GPU only (a shard's kernels were not captured: null, not the
    # whole-problem figure)
    traffic = None
    tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if world == 1 and os.path.exists(tf):
        with open(tf) as fh:
            traffic = json.load(fh).get(f"config{args.config}", {}).get(dom)

    # end to end through the C ABI with pinned HOST buffers: every step copies
    # its f from pinned host memory and its output back (SINCFFT_PTR_HOST_ASYNC);
    # successive steps rotate over --e2e-streams streams so the H2D of step
    # k+1, the kernels of step k and the D2H of step k-1 overlap (full-duplex
    # PCIe; 4 streams measured 5.95 ms vs 6.42 with 2 at config 3)
    # (N > 1 with a distributed FFT: one stream -- its exchange buffers are
    # shared by every call, so calls could not overlap anyway)
    nbuf = 1 if dist_fft is not None else args.e2e_streams
    h_f = [torch.from_numpy(fshard).pin_memory() for _ in range(nbuf)]
    h_out = [torch.empty(tuple(d_out.shape), dtype=torch.complex128).pin_memory()
             for _ in range(nbuf)]
    streams = [torch.cuda.Stream(dev) for _ in range(nbuf)]
    grids = [d_grid] + [torch.empty_like(d_grid) for _ in range(nbuf - 1)]  # one per stream
    d_fs = [d_f] + [torch.empty_like(d_f) for _ in range(nbuf - 1)]
    h2d = h_f[0].numel() * 16
    d2h = h_out[0].numel() * 16

    def e2e_step(k):
        st = C.c_void_p(streams[k % nbuf].cuda_stream)
        if world == 1 or col_shard:
            _lib.check(L.sincfft_nnfft_execute(ph, h_f[k % nbuf].data_ptr(),
                                               h_out[k % nbuf].data_ptr(), B,
                                               _lib.PTR_HOST_ASYNC, st))
        elif dist_fft is not None:
            with torch.cuda.stream(streams[k % nbuf]):
                fk = d_fs[k % nbuf]
                fk.copy_(h_f[k % nbuf], non_blocking=True)
                if args.dist_backend == "gloo":  # gloo does not order on side streams
                    streams[k % nbuf].synchronize()
                o = dist_fft(fk)
                h_out[k % nbuf].copy_(o, non_blocking=True)
        else:
            g = grids[k % nbuf]
            with torch.cuda.stream(streams[k % nbuf]):
                _lib.check(L.sincfft_nnfft_spread(ph, h_f[k % nbuf].data_ptr(),
                                                  g.data_ptr(), B, _lib.PTR_HOST_ASYNC, st))
                if args.dist_backend == "gloo":  # gloo does not order on side streams
                    streams[k % nbuf].synchronize()
                dist.all_reduce(torch.view_as_real(g))
                if args.dist_backend == "gloo":
                    torch.cuda.synchronize()
                _lib.check(L.sincfft_nnfft_finish(ph, g.data_ptr(),
                                                  h_out[k % nbuf].data_ptr(), B,
                                                  _lib.PTR_HOST_ASYNC, st))

    # warm every stream's buffers and the stream-ordered pool (its first
    # growth costs a few ms of host time per allocation)
    for k in range(max(3 * nbuf, args.warmup)):
        e2e_step(k)
    # drain the warm-up backlog (the host enqueues far ahead of the copies)
    # so the timed region holds exactly the timed steps
    torch.cuda.synchronize()
    # the timed K-step region is repeated E2E_REPEATS times and the median
    # reported (all repeats in the line): one run in ~6 showed a 5x host-side
    # stall of the PCIe pipeline
    e2e_reps = []
    for _ in range(E2E_REPEATS):
        barrier()
        ev0.record(stream)
        for st in streams:
            st.wait_event(ev0)
        for k in range(args.steps):
            e2e_step(k)
        for st in streams:
            e = torch.cuda.Event()
            e.record(st)
            stream.wait_event(e)
        ev1.record(stream)
        ev1.synchronize()
        barrier()
        e2e_reps.append(max_over_ranks(ev0.elapsed_time(ev1) / args.steps))
    e2e_ms = float(np.median(e2e_reps))
    e2e_val = total_nodes / (e2e_ms * 1e-3)
    h_out = h_out[(args.steps - 1) % nbuf]
    # the e2e output must agree with the device-resident one (grid flushes use
    # fp64 atomics, so summation order -- and the last bits -- may differ)
    e2e_dev = float(np.max(np.abs(h_out.numpy() - dev_out)) / np.abs(fshard).sum())
    if e2e_dev > 1e-13:
        print(f"WARNING: e2e output deviates from the device-resident output by {e2e_dev:.3e}",
              file=sys.stderr)

    # the link floor of that pipeline: the same H2D and D2H bytes copied
    # concurrently on two streams with no kernels (PCIe full duplex)
    pcie_ms = None
    if world == 1:
        cs = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
        d_in = torch.empty_like(d_f)

        def copies():
            with torch.cuda.stream(cs[0]):
                d_in.copy_(h_f[0], non_blocking=True)
            with torch.cuda.stream(cs[1]):
                h_out.copy_(d_out, non_blocking=True)  # already checked above

        copies()
        torch.cuda.synchronize()
        ev0.record(stream)
        for c in cs:
            c.wait_event(ev0)
        for _ in range(5):
            copies()
        for c in cs:
            stream.wait_stream(c)
        ev1.record(stream)
        ev1.synchronize()
        pcie_ms = ev0.elapsed_time(ev1) / 5
        del d_in

    # the spread's memory floor: its f reads are a random 16-byte gather over
    # all of f (sources are cell-sorted, f is in caller order).  Time torch's
    # own gather f[perm] of the same M1 complex128 values through a random
    # permutation (random 16-byte reads plus a sequential write; no window
    # math, no grid) -- what the spread's f traffic costs by itself
    gather_floor_ms = None
    if world == 1 and B == 1:
        gen = torch.Generator(device=dev)
        gen.manual_seed(0)
        rp = torch.randperm(d_f.shape[0], device=dev, generator=gen)
        tmp = d_f[rp]
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(5):
            tmp = d_f[rp]
        ev1.record(stream)
        ev1.synchronize()
        gather_floor_ms = ev0.elapsed_time(ev1) / 5
        del rp, tmp

    launches = L.sincfft_nnfft_launches_per_execute(ph, B) * args.steps
    if dist_fft is not None:  # grid memset + spread, pack (+ tail fix), 3 passes
        fix = 1 if geo["L"] < geo["K"] + geo["Kout"] - 1 else 0  # (+ rank-0 fix add), unpack, gather
        if not args.peer_transposes:
            launches = (2 + 1 + fix + 3 + (fix if rank == 0 else 0) + 1 + 1
                        + (0 if args.dense_exchange else 2)) * args.steps
        else:  # memset, spread, pack (+fix) to peers, unpack, 3 passes, unpack h, gather
            launches = (2 + 1 + fix + 1 + 3 + 1 + 1) * args.steps
    fp64_peak, fp64_note = 148 * 64 * 2 * (clk.max_mhz or 1965) * 1e6 / 1e12, \
        "derived: 148 SMs x 64 DFMA/clk x 2 flops x max SM clock"
    pf = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(pf):
        with open(pf) as fh:
            fp64_peak, fp64_note = float(json.load(fh)["fp64_dfma_tflops"]), \
                "measured: tools/fp64_peak.cu (DFMA microbenchmark on this pool's B200)"

    # the same three figures for every stage (the north star asks for each of
    # spread / FFT / interpolate against the HBM roofline): algorithmic bytes
    # over the live stage time, the committed ncu DRAM bytes and FP64 counts
    traffic_all = {}
    if world == 1 and os.path.exists(tf):
        with open(tf) as fh:
            traffic_all = json.load(fh).get(f"config{args.config}", {})
    stages_roof = {}
    for i, n in enumerate(names):
        t_s = stage[i] * 1e-3
        if t_s <= 0:
            continue
        stages_roof[n] = {"launch_ms": float(stage[i]), "alg_bytes_per_launch": alg[n],
                          "achieved": alg[n] / t_s / 1e9, "frac": alg[n] / t_s / 1e9 / peak,
                          "traffic": traffic_all.get(n),
                          "dram_frac": (traffic_all[n] / t_s / 1e9 / peak
                                        if traffic_all.get(n) else None),
                          "fp64_frac": (None if flops.get(n) is None else
                                        flops[n] / t_s / 1e12 / fp64_peak)}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_sample_rate(cfg)
        for k in ("seconds_per_step", "plan_s"):
            cpu.pop(k, None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "N": cfg["N"], "M1": cfg["M1"], "M2": cfg["M2"],
                       "m1": m, "m2": m, "sigma1": 2.0, "sigma2": 2.0, "batch": B,
                       "N_star": n_star, "N1": geo["N1"], "K": K, "N2": N2,
                       "fft_length_L": geo["L"], "fft_L1xL2": [geo["L1"], geo["L2"]], "l2": "inputs larger than L2 "
                       "(f and out 256 MiB each per column vs 126 MB L2)",
                       "parallelism": (f"batch columns sharded x{world} (no communication)"
                                       if col_shard else
                                       f"sources+targets sharded x{world}" +
                                       (" by position (quantiles of v and x)" if world > 1 else "")) +
                       (("; distributed FFT: " + ("reduce-scatter + 2 all-to-all + all-gather"
                                                   if args.dense_exchange else
                                                   "every exchange fused into the kernels as "
                                                   "stores into the owners' buffers over peer "
                                                   "memory (CUDA IPC), 4 barriers"
                                                   if args.peer_transposes else
                                                   "4 NCCL all-to-alls (grid / h rows "
                                                   "exchanged sparsely)")
                         if dist_fft is not None else ", NCCL all-reduce of the K-grid")
                        if world > 1 and not col_shard else "")},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": traffic, "alg_bytes_per_launch": alg[dom],
                         "launch_ms": t_dom * 1e3,
                         "random_gather_floor_ms": gather_floor_ms
                         if dom == "spread" else None,
                         "bound_note": (
                             "single-column spread: f is read through the cell-sort permutation, "
                             "2^24 random 16-byte reads at config 3; HBM serves ~59 G random "
                             "sectors/s whatever the fill size (tools/randread.cu: 0.285 ms alone; "
                             "torch's f[perm] = random_gather_floor_ms), and a timing-only build "
                             "with no window arithmetic and no accumulation still takes 0.351 of "
                             "the kernel's 0.388 ms (DESIGN.md, SFB_SPREAD_ABL), so frac against "
                             "the sequential-copy peak understates how close the kernel is to "
                             "its loads") if dom == "spread" and B == 1 else None,
                         "fp64": None if flops[dom] is None else {
                             "achieved_tflops": flops[dom] / t_dom / 1e12,
                             "peak_tflops": fp64_peak,
                             "frac": flops[dom] / t_dom / 1e12 / fp64_peak,
                             "dfma_per_node": fp64_node[dom][0],
                             "other_fp64_per_node": fp64_node[dom][1],
                             "ncu_fp64_pipe_active_pct": fp64_node[dom][2],
                             "counts_from": fp64_node[dom][3],
                             "peak_note": fp64_note}},
            "stage_ms": {n: float(stage[i]) for i, n in enumerate(names)},
            "roofline_stages": stages_roof,
            "plan_ms": plan_ms,
            "plan_warm_ms": plan_warm_ms,
            "one_shot": None if plan_warm_ms is None else {
                "ms": plan_warm_ms + ms,
                "value": total_nodes / ((plan_warm_ms + ms) * 1e-3), "unit": "nodes/s",
                "note": "plan (host numpy nodes, warm process) + one execute"},
            "e2e": {"value": e2e_val, "unit": "nodes/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                    "repeats_ms": e2e_reps,
                    "pcie_floor_ms": pcie_ms,
                    "mode": f"sincfft_nnfft_execute(host pinned, PTR_HOST_ASYNC), {nbuf} streams "
                            "round-robin: H2D(k+1) || kernels(k) || D2H(k-1)"},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if cpu:
            line["cpu_baseline"] = cpu
        if shard_dev is not None:
            line["shard_check_rel_err"] = shard_dev
        line["e2e_vs_device_rel_err"] = e2e_dev
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def spawn_ranks(n, same_device=False):
    """Re-launch this command under torch.distributed.run with n ranks on this
    node (rendezvous on 127.0.0.1, a free port); returns its exit code."""
    import socket
    import subprocess
    if not same_device:
        import torch
        have = torch.cuda.device_count()
        if have < n:
            print(f"bench.py: --gpus {n} needs {n} visible GPUs, found {have}",
                  file=sys.stderr)
            return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="3")
    ap.add_argument("--m", type=int, default=None,
                    help="window cut-off m1 = m2 (config 2 is BASELINE's sweep over "
                         "m in {2, 4, 6, 8, 10}; default: the config's own m)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--ref-budget-s", type=float, default=240.0,
                    help="--impl reference: wall-time bound (s) after which warm-ups / timed "
                         "steps stop early (never below 1 / 2)")
    ap.add_argument("--e2e-streams", type=int, default=4,
                    help="host-buffer pipeline depth of the e2e leg (streams in flight)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional tests)")
    ap.add_argument("--same-device", action="store_true",
                    help="map every rank to cuda:0 (with gloo: test the sharded path on one "
                         "GPU; kernels of different ranks never wait on each other)")
    ap.add_argument("--replicated-fft", action="store_true",
                    help="N > 1: all-reduce the K-grid and replicate the FFT (the "
                         "north star's baseline partitioning) instead of splitting it")
    ap.add_argument("--dense-exchange", action="store_true",
                    help="N > 1 distributed FFT: reduce-scatter / all-gather the whole "
                         "K-grid and h instead of all-to-alls of the rows each rank touches")
    ap.add_argument("--peer-transposes", action="store_true",
                    help="N > 1 distributed FFT: every exchange fused into the kernels as "
                         "stores into the owners' buffers over peer memory (CUDA IPC) "
                         "instead of NCCL all-to-alls")
    ap.add_argument("--check-shards", action="store_true",
                    help="N > 1: compare this rank's output shard with a single-rank "
                         "transform of the same inputs and report the max deviation")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    cfg = CONFIGS[args.config]
    if args.m is not None:
        cfg = dict(cfg, m=args.m, desc=cfg["desc"].replace(f"m1=m2={cfg['m']}",
                                                           f"m1=m2={args.m}"))
    world = int(os.environ.get("WORLD_SIZE", "0"))
    if args.impl != "reference":
        if args.gpus > 1 and world == 0:
            # `python bench.py --gpus N` without a launcher: start the N ranks
            # ourselves, one process per GPU, exactly as the driver's torchrun
            sys.exit(spawn_ranks(args.gpus, args.same_device))
        if max(world, 1) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world or 1}")
    if args.impl == "reference":
        run_reference(args, cfg)
    elif cfg.get("sinc"):
        run_sinc_b200(args, cfg)
    else:
        run_b200(args, cfg)


if __name__ == "__main__":
    main()
