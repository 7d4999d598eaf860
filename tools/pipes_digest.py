"""dev helper: per-kernel digest of an ncu --metrics CSV (tools/ncu_pipes.sh):
duration, FP64-pipe utilisation, DFMA / fp64 thread instructions, DRAM bytes.
usage: python tools/pipes_digest.py pipes_config3.csv [kernel-substring]"""
import csv
import sys
from collections import OrderedDict, defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hi = next(i for i, r in enumerate(rows) if r[0] == "ID")
h = rows[hi]
ix = {c: i for i, c in enumerate(h)}
filt = sys.argv[2] if len(sys.argv) > 2 else None
launch = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) != len(h):
        continue
    key = (r[ix["ID"]], r[ix["Kernel Name"]])
    launch.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "") or 0)
agg = defaultdict(list)
for (i, k), m in launch.items():
    name = k.split("(")[0].replace("void ", "")
    if filt and filt not in name:
        continue
    agg[name].append(m)
print(f"{'kernel':42s} {'n':>3s} {'us':>8s} {'fp64%act':>8s} {'fp64%el':>8s} {'DFMA/thr M':>10s} "
      f"{'fp64 thr M':>10s} {'fp64 wi%':>8s} {'DRAM MB':>8s} {'warps%':>6s}")
for name, ms in agg.items():
    a = lambda key: sum(m.get(key, 0.0) for m in ms) / len(ms)  # noqa: E731
    print(f"{name[:42]:42s} {len(ms):3d} {a('gpu__time_duration.sum') / 1e3:8.1f} "
          f"{a('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active'):8.1f} "
          f"{a('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed'):8.1f} "
          f"{a('sm__sass_thread_inst_executed_op_dfma_pred_on.sum') / 1e6:10.1f} "
          f"{a('sm__sass_thread_inst_executed_op_fp64_pred_on.sum') / 1e6:10.1f} "
          f"{100 * a('sm__inst_executed_pipe_fp64.sum') / max(a('sm__inst_executed.sum'), 1):8.1f} "
          f"{(a('dram__bytes_read.sum') + a('dram__bytes_write.sum')) / 1e6:8.1f} "
          f"{a('sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f}")


def fp64_json(paths, out):
    """profiles/ncu_fp64.json: per config and hot kernel, the ncu FP64 counts
    per launch (DFMA and all fp64 thread instructions) and the FP64-pipe
    utilisation -- bench.py derives roofline.fp64 from these."""
    import json
    import re
    res = {}
    for cfg, path in paths:
        rows_ = [r for r in csv.reader(open(path)) if r]
        hi_ = next(i for i, r in enumerate(rows_) if r[0] == "ID")
        h_ = rows_[hi_]
        ix_ = {c: i for i, c in enumerate(h_)}
        per = OrderedDict()
        for r in rows_[hi_ + 1:]:
            if len(r) != len(h_):
                continue
            per.setdefault((r[ix_["ID"]], r[ix_["Kernel Name"]]), {})[r[ix_["Metric Name"]]] = \
                float(r[ix_["Metric Value"]].replace(",", "") or 0)
        d = {}
        for (_, k), m in per.items():
            name = re.sub(r"^(void )?(sfb::)?", "", k.split("(")[0]).split("<")[0]
            kind = ("spread" if name in ("k_spread", "k_spread_b", "k_spread_bw", "k_spread_dense") else
                    "gather" if name in ("k_gather", "k_gather2", "k_gather4", "k_gather_b")
                    else None)
            if kind is None or kind in d:
                continue
            d[kind] = {"kernel": k.split("(")[0],
                       "dfma_thread_inst": m.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum"),
                       "fp64_thread_inst": m.get("sm__sass_thread_inst_executed_op_fp64_pred_on.sum"),
                       "fp64_pipe_active_pct": m.get(
                           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                       "duration_us": m.get("gpu__time_duration.sum", 0) / 1e3}
        res[f"config{cfg}"] = d
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    return res
