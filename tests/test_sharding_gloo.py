"""World-size-2 test (gloo, CPU) of the multi-GPU partitioning logic in
paper_2107_02671_b200/sharding.py: sources and targets split over ranks, one
all-reduce of the partial K-grids, replicated FFT, per-rank gather.  The stage
callables are the CPU oracle's (no GPU here); the result must equal the
unsharded transform."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import sincfft_oracle as O
        from paper_2107_02671_b200.sharding import ShardedNnfft, shard_range
        from tests.inputs import nodes_and_coeffs

        N, M1, M2, m = 300, 5000, 3001, 6
        v, x, f = nodes_and_coeffs(21, M1, M2, clustered=True)
        n_star, vs = O.rescale_frequencies(N, v, 2.0, m)
        s0, s1 = shard_range(M1, world, rank)
        t0, t1 = shard_range(M2, world, rank)
        src = O.plan(n_star, vs[s0:s1], x[:1], m1=m, m2=m)
        tgt = O.plan(n_star, vs[:1], x[t0:t1], m1=m, m2=m)

        def spread(fs):
            return torch.from_numpy(O.spread(src, fs)).reshape(1, -1).clone()

        def finish(grid):
            return O.finish(tgt, grid.reshape(-1).numpy())

        out = ShardedNnfft(spread, finish)(f[s0:s1])
        np.save(os.path.join(result_dir, f"out{rank}.npy"), out)
    finally:
        dist.destroy_process_group()


def test_two_rank_source_and_target_sharding(tmp_path):
    from oracle import sincfft_oracle as O
    from tests.inputs import nodes_and_coeffs

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"out{r}.npy") for r in range(world)])
    N, M1, M2, m = 300, 5000, 3001, 6
    v, x, f = nodes_and_coeffs(21, M1, M2, clustered=True)
    n_star, vs = O.rescale_frequencies(N, v, 2.0, m)
    ref = O.trafo(O.plan(n_star, vs, x, m1=m, m2=m), f)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) <= 1e-14 * np.sum(np.abs(f))


def test_shard_range_covers_exactly():
    from paper_2107_02671_b200.sharding import shard_range
    for n in (1, 7, 1 << 24):
        for world in (1, 2, 3, 8):
            pieces = [shard_range(n, world, r) for r in range(world)]
            assert pieces[0][0] == 0 and pieces[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(pieces, pieces[1:]))


def _coll_worker(rank, world, port, result_dir):
    """TorchCollectives over gloo (CPU): the three collectives of the
    distributed FFT must match their definitions (and run_ranks_in_process's
    in-process emulation, which the GPU test checks against the unsharded
    transform)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2107_02671_b200.sharding import TorchCollectives

        c = TorchCollectives()
        n = 5

        def buf(r, salt):  # rank r's send buffer, world blocks of n
            k = torch.arange(world * n, dtype=torch.float64)
            return torch.complex(k + 100 * r + salt, -k * (r + 1) - salt)

        rs = c.reduce_scatter(buf(rank, 0.5))
        want = sum(buf(r, 0.5) for r in range(world))[rank * n:(rank + 1) * n]
        assert torch.equal(rs, want)
        a2a = c.all_to_all(buf(rank, 1.0))
        want = torch.cat([buf(src, 1.0)[rank * n:(rank + 1) * n] for src in range(world)])
        assert torch.equal(a2a, want)
        ag = c.all_gather(buf(rank, 2.0)[:n])
        want = torch.cat([buf(r, 2.0)[:n] for r in range(world)])
        assert torch.equal(ag, want)
        np.save(os.path.join(result_dir, f"ok{rank}.npy"), np.array([1]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_distributed_fft_collectives_gloo(tmp_path, world):
    mp.spawn(_coll_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    assert all((tmp_path / f"ok{r}.npy").exists() for r in range(world))


def _native_worker(rank, world, port, result_dir):
    """The collective layer of the default N > 1 path (sparse distributed FFT)
    on CPU: TorchCollectives' native calls -- the exact reduce_scatter_tensor /
    all_to_all_single / all_gather_into_tensor / uneven all_to_all_single
    calls NCCL executes on the GPUs -- forced on (gloo runs them on CPU
    tensors), against its CPU-staging fallback and against the data movement
    they must perform."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2107_02671_b200.sharding import SparseRows, TorchCollectives, _all_to_all_v
        res = {}
        for native in (True, False):
            c = TorchCollectives()
            c.nccl = native  # the NCCL-path calls (CPU tensors over gloo) or the staging path
            n = 6
            send = torch.complex(torch.arange(world * n, dtype=torch.float64) + 1000 * rank,
                                 -torch.arange(world * n, dtype=torch.float64))
            # (clones: on CPU tensors the staging path's .cpu() aliases its input)
            res[f"rs{native}"] = c.reduce_scatter(send.clone()).numpy()
            res[f"a2a{native}"] = c.all_to_all(send.clone()).numpy()
            res[f"ag{native}"] = c.all_gather(send[:n].clone()).numpy()
            # uneven splits as the sparse exchange produces them: rank q sends
            # (q + 1) * (p + 2) elements to rank p
            ins = [(rank + 1) * (p + 2) for p in range(world)]
            outs = [(q + 1) * (rank + 2) for q in range(world)]
            sv = torch.complex(torch.arange(sum(ins), dtype=torch.float64) + 100 * rank,
                               torch.full((sum(ins),), float(rank), dtype=torch.float64))
            res[f"a2av{native}"] = _all_to_all_v(c, sv, ins, outs).numpy()
        # SparseRows bookkeeping: what a rank sends to q is what q expects from it
        sup = [[1000 * r + 7, 1000 * r + 900, 500 * r, 500 * r + 1300] for r in range(world)]
        rows = SparseRows(sup, 64, 5, 3)
        ok = all(rows.grid_send_splits(a)[b] == rows.grid_recv_splits(b)[a] and
                 rows.h_send_splits(a)[b] == rows.h_recv_splits(b)[a]
                 for a in range(world) for b in range(world))
        res["splits_ok"] = np.array([ok])
        np.savez(os.path.join(result_dir, f"coll{rank}.npz"), **res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_collective_layer_native_calls(tmp_path, world):
    mp.spawn(_native_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    d = [np.load(tmp_path / f"coll{r}.npz") for r in range(world)]
    n = 6
    sends = [np.arange(world * n) + 1000 * r - 1j * np.arange(world * n) for r in range(world)]
    for r in range(world):
        assert bool(d[r]["splits_ok"][0])
        for native in (True, False):
            np.testing.assert_array_equal(d[r][f"rs{native}"],
                                          sum(s[r * n:(r + 1) * n] for s in sends))
            np.testing.assert_array_equal(d[r][f"a2a{native}"],
                                          np.concatenate([s[r * n:(r + 1) * n] for s in sends]))
            np.testing.assert_array_equal(d[r][f"ag{native}"],
                                          np.concatenate([s[:n] for s in sends]))
            exp = []
            for q in range(world):
                ins = [(q + 1) * (p + 2) for p in range(world)]
                off = sum(ins[:r])
                sv = np.arange(sum(ins)) + 100 * q + 1j * q
                exp.append(sv[off:off + ins[r]])
            np.testing.assert_array_equal(d[r][f"a2av{native}"], np.concatenate(exp))
