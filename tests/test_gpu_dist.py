"""Distributed (column-split) FFT of the sharded NNFFT.

Every rank of a P-way split runs in THIS process on one GPU
(``sharding.run_ranks_in_process``: the reduce-scatter, the two all-to-alls
and the all-gather become tensor sums and slices), so the per-rank layouts and
kernels are checked against the unsharded transform without a process group.
The geometry is config 3's (N = 2^20, m = 8, sigma = 2: FFT 4096 x 1024 with
a Bluestein tail fix of D = 79) with fewer nodes; the clustered nodes put
sources and targets of every rank all over the band.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2107_02671_b200 as sf  # noqa: E402
from paper_2107_02671_b200.sharding import (DistFftRank, dist_layout,  # noqa: E402
                                            run_ranks_in_process, shard_range)
from tests.inputs import nodes_and_coeffs  # noqa: E402

pytestmark = pytest.mark.gpu

N, M, m = 1 << 20, 1 << 18, 8


@pytest.fixture(scope="module")
def problem():
    v, x, f = nodes_and_coeffs(5, M, M, clustered=True)
    n_star, vs = sf.rescale_frequencies(N, v, 2.0, m)
    full = sf.nnfft_plan(n_star, vs, x, m1=m, m2=m, device=0)
    return n_star, vs, x, f, sf.nnfft_trafo(full, f)


def test_full_window_plan_matches_default(problem):
    n_star, vs, x, f, ref = problem
    p = sf.nnfft_plan(n_star, vs, x, m1=m, m2=m, device=0, h_window="full")
    out = sf.nnfft_trafo(p, f)
    assert np.max(np.abs(out - ref)) <= 1e-13 * np.sum(np.abs(f))


def test_layout_rules(problem):
    n_star, vs, x, f, _ = problem
    p = sf.nnfft_plan(n_star, vs[:1000], x[:1000], m1=m, m2=m, device=0, h_window="full")
    geo = p.backend_geometry
    assert (geo["L1"], geo["L2"]) == (4096, 1024)
    for world in (1, 2, 4, 8, 16):
        lay = dist_layout(p, world)
        assert lay is not None and lay["Bc"] * world == 4096 and lay["Br"] * world == 1024
    assert dist_layout(p, 3) is None  # not a power of two
    small = sf.nnfft_plan(256, vs[:64] * 0.9, x[:64], m1=4, m2=4, device=0, h_window="full")
    assert dist_layout(small, 2) is None  # one-CTA FFT: stays replicated


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_in_process_ranks_equal_unsharded(problem, world):
    n_star, vs, x, f, ref = problem
    ranks, shards = [], []
    for r in range(world):
        s0, s1 = shard_range(M, world, r)
        t0, t1 = shard_range(M, world, r)
        plan = sf.nnfft_plan(n_star, vs[s0:s1], x[t0:t1], m1=m, m2=m, device=0, h_window="full")
        ranks.append(DistFftRank(plan, world, r))
        shards.append(torch.from_numpy(f[s0:s1]).to("cuda:0"))
    outs = run_ranks_in_process(ranks, shards)
    got = np.concatenate([o.cpu().numpy() for o in outs])
    err = np.max(np.abs(got - ref)) / np.sum(np.abs(f))
    assert err <= 1e-13, err


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_sparse_exchange_position_partition(problem, world):
    """Position partitions (bench.py N > 1): sources and targets split by
    quantiles, the K-grid / h exchanges move only the rows each rank touches."""
    from paper_2107_02671_b200.sharding import SparseDistFftRank, run_sparse_ranks_in_process

    n_star, vs, x, f, ref = problem
    sv, sx = np.argsort(vs, kind="stable"), np.argsort(x, kind="stable")
    ranks, shards, tidx = [], [], []
    for r in range(world):
        s0, s1 = shard_range(M, world, r)
        si, ti = sv[s0:s1], sx[s0:s1]
        plan = sf.nnfft_plan(n_star, vs[si], x[ti], m1=m, m2=m, device=0, h_window="full")
        ranks.append(SparseDistFftRank(plan, world, r))
        shards.append(torch.from_numpy(np.ascontiguousarray(f[si])).to("cuda:0"))
        tidx.append(ti)
    outs = run_sparse_ranks_in_process(ranks, shards)
    err = max(np.max(np.abs(o.cpu().numpy() - ref[ti])) for o, ti in zip(outs, tidx))
    assert err / np.sum(np.abs(f)) <= 1e-13, err
    if world > 1:  # the exchanged rows are a fraction of the whole grid / h
        rows = ranks[0].rows
        assert max(rows.nrow) < 0.75 * ranks[0].layout["Sb"] / ranks[0].layout["Bc"]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_peer_transposes_in_process(problem, world):
    """The fused transposes (column / row passes storing into the owners'
    receive buffers) reproduce the unsharded transform."""
    from paper_2107_02671_b200.sharding import PeerDistFftRank, run_peer_ranks_in_process

    n_star, vs, x, f, ref = problem
    sv, sx = np.argsort(vs, kind="stable"), np.argsort(x, kind="stable")
    ranks, shards, tidx = [], [], []
    for r in range(world):
        s0, s1 = shard_range(M, world, r)
        si, ti = sv[s0:s1], sx[s0:s1]
        plan = sf.nnfft_plan(n_star, vs[si], x[ti], m1=m, m2=m, device=0, h_window="full")
        ranks.append(PeerDistFftRank(plan, world, r))
        shards.append(torch.from_numpy(np.ascontiguousarray(f[si])).to("cuda:0"))
        tidx.append(ti)
    outs = run_peer_ranks_in_process(ranks, shards)
    err = max(np.max(np.abs(o.cpu().numpy() - ref[ti])) for o, ti in zip(outs, tidx))
    assert err / np.sum(np.abs(f)) <= 1e-13, err
