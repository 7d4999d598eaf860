"""Per-rank DEVICE time of the sharded config-3 NNFFT at P = 1, 2, 4, 8, measured
on ONE B200 by running rank 0's kernels alone (its source/target shards, its
columns/rows of the split FFT), next to the replicated-FFT partitioning, plus
the bytes each rank sends through the collectives.  Collective times are NOT
measured here (one GPU); this is the compute side of the scaling model only.

    python tools/dist_projection.py > profiles/r01g_dist_projection.json
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2107_02671_b200 as sf  # noqa: E402
from paper_2107_02671_b200.sharding import (DistFftRank, SparseDistFftRank,  # noqa: E402
                                            gpu_stages, shard_range, sparse_rows_for)
from tests.inputs import nodes_and_coeffs  # noqa: E402

N, M, m, REPS = 1 << 20, 1 << 24, 8, 20


def timed(fn):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(REPS):
        fn()
    ev[1].record()
    ev[1].synchronize()
    return ev[0].elapsed_time(ev[1]) / REPS


def main():
    v, x, f = nodes_and_coeffs(0, M, M, clustered=True)
    n_star, vs = sf.rescale_frequencies(N, v, 2.0, m)
    rows = []
    order_v, order_x = np.argsort(vs, kind="stable"), np.argsort(x, kind="stable")
    z = lambda n: torch.zeros(int(n), dtype=torch.complex128, device="cuda:0")  # noqa: E731
    cplx = 16
    for world in (1, 2, 4, 8):
        per_rank = []
        # every rank's row ranges (the sparse exchange needs them all)
        sups = []
        for rank in range(world):
            s0, s1 = shard_range(M, world, rank)
            pl = sf.nnfft_plan(n_star, vs[order_v[s0:s1]], x[order_x[s0:s1]], m1=m, m2=m,
                               device=0, h_window="full")
            sups.append(SparseDistFftRank(pl, world, rank).support())
            del pl
        for rank in range(world):
            s0, s1 = shard_range(M, world, rank)
            # a position partition (bench.py N > 1): quantile ranges of v and x
            si, ti = order_v[s0:s1], order_x[s0:s1]
            plan = sf.nnfft_plan(n_star, vs[si], x[ti], m1=m, m2=m, device=0, h_window="full")
            d_f = torch.from_numpy(np.ascontiguousarray(f[si])).to("cuda:0")
            r = DistFftRank(plan, world, rank)
            lay = r.layout
            block, rows_buf, cols2 = z(lay["Sb"]), z(lay["cols"]), z(lay["cols"])
            hall = z(lay["hblk"] * world)
            r.block = block
            t = {"pack(spread)": timed(lambda: r.pack(d_f)),
                 "colfwd": timed(lambda: r.colfwd(block)),
                 "rowmul": timed(lambda: r.rowmul(rows_buf)),
                 "colinv": timed(lambda: r.colinv(cols2)),
                 "gather(unpack)": timed(lambda: r.gather(hall))}
            sr = SparseDistFftRank(plan, world, rank)
            srows = sparse_rows_for(sups, sr)
            sr.set_rows(srows)
            sr.block = block
            rgrid = z(sum(srows.grid_recv_splits(rank)))
            rh = z(sum(srows.h_recv_splits(rank)))
            hb = z(lay["hblk"])
            ts = {"pack_rows(spread)": timed(lambda: sr.pack_rows(d_f)),
                  "unpack_rows": timed(lambda: sr.unpack_rows(rgrid)),
                  "colfwd": t["colfwd"], "rowmul": t["rowmul"], "colinv": t["colinv"],
                  "pack_hrows": timed(lambda: sr.pack_hrows(hb)),
                  "gather_rows(unpack)": timed(lambda: sr.gather_rows(rh))}
            spread, finish = gpu_stages(plan, 1)
            grid = spread(d_f)
            rep = {"spread": timed(lambda: spread(d_f)), "fft+gather": timed(lambda: finish(grid))}
            per_rank.append({"rank": rank,
                             "distributed_ms": {k: round(vv, 4) for k, vv in t.items()},
                             "distributed_compute_ms": round(sum(t.values()), 4),
                             "sparse_ms": {k: round(vv, 4) for k, vv in ts.items()},
                             "sparse_compute_ms": round(sum(ts.values()), 4),
                             "sparse_bytes": {"grid_out": sum(srows.grid_send_splits(rank)) * cplx,
                                              "grid_in": sum(srows.grid_recv_splits(rank)) * cplx,
                                              "h_out": sum(srows.h_send_splits(rank)) * cplx,
                                              "h_in": sum(srows.h_recv_splits(rank)) * cplx},
                             "replicated_compute_ms": round(sum(rep.values()), 4),
                             "replicated_ms": {k: round(vv, 4) for k, vv in rep.items()}})
            bytes_ = {"distributed": {"reduce_scatter_in": world * lay["Sb"] * cplx,
                                      "all_to_all_x2": 2 * lay["cols"] * cplx,
                                      "all_gather_out": world * lay["hblk"] * cplx},
                      "replicated": {"all_reduce": plan.backend_geometry["K"] * cplx}}
            del plan, r, sr, spread, finish, grid
            torch.cuda.empty_cache()
        rows.append({"P": world,
                     "max_rank_distributed_compute_ms": max(q["distributed_compute_ms"] for q in per_rank),
                     "max_rank_sparse_compute_ms": max(q["sparse_compute_ms"] for q in per_rank),
                     "max_rank_sparse_bytes": max(sum(q["sparse_bytes"].values()) for q in per_rank),
                     "max_rank_replicated_compute_ms": max(q["replicated_compute_ms"] for q in per_rank),
                     "bytes_per_rank": bytes_, "ranks": per_rank})
    print(json.dumps({"what": "rank-0 device time per step on one B200 (no collectives), "
                      "config 3 clustered, sources+targets partitioned by position (quantiles); every rank's "
                      "kernels timed alone",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
