"""Multi-GPU partitioning of one NNFFT, one process per GPU.

The path shards naturally:
  * targets x_j (and batch columns) -- no communication;
  * sources v_k -- each rank spreads its sources onto a private copy of the
    K = N1 + 2 m1 point grid; the partial grids are summed with ONE all-reduce
    (the path's only exchange step); the deconvolution + FFT that follow are
    replicated on every rank, and each rank gathers its own targets.

``ShardedNnfft`` is written against two small stage callables so the same
host logic runs on the GPU (C ABI ``sincfft_nnfft_spread`` / ``_finish`` over
NCCL) and, in the CPU tests, on the oracle over gloo.
"""

from __future__ import annotations


def shard_range(n: int, world: int, rank: int):
    """Contiguous, balanced [lo, hi) slice of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    return rank * n // world, (rank + 1) * n // world


class ShardedNnfft:
    """One NNFFT split over the ranks of a torch.distributed process group.

    spread(f_shard) -> grid tensor (complex128, shape (B, K)) for this rank's
    sources; finish(grid) -> output for this rank's targets.  With world == 1
    the all-reduce is skipped.
    """

    def __init__(self, spread, finish, group=None):
        self.spread = spread
        self.finish = finish
        self.group = group

    def __call__(self, f_shard):
        import torch
        import torch.distributed as dist

        grid = self.spread(f_shard)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(self.group) > 1:
            dist.all_reduce(torch.view_as_real(grid), op=dist.ReduceOp.SUM, group=self.group)
        return self.finish(grid)


def gpu_stages(plan, batch: int, stream=None):
    """Stage callables over the C ABI for a plan built on this rank's shards
    (device tensors in, device tensors out)."""
    import ctypes as C

    import torch

    from . import _lib

    geo = plan.backend_geometry
    dev = torch.device("cuda", plan.device)

    def _stream():
        return C.c_void_p((stream or torch.cuda.current_stream(dev)).cuda_stream)

    def spread(f):
        grid = torch.empty((batch, geo["K"]), dtype=torch.complex128, device=dev)
        _lib.check(_lib.lib.sincfft_nnfft_spread(plan.handle, f.data_ptr(), grid.data_ptr(),
                                                 batch, _lib.PTR_DEVICE, _stream()))
        return grid

    def finish(grid):
        shape = (geo["M2"], batch) if batch > 1 else (geo["M2"],)
        out = torch.empty(shape, dtype=torch.complex128, device=dev)
        _lib.check(_lib.lib.sincfft_nnfft_finish(plan.handle, grid.data_ptr(), out.data_ptr(),
                                                 batch, _lib.PTR_DEVICE, _stream()))
        return out

    return spread, finish


# ------------------------------------------------------------ distributed FFT
def dist_layout(plan, world: int):
    """Buffer sizes of the distributed FFT for `world` ranks, or None when the
    plan shape / world size is not supported (then use ShardedNnfft)."""
    import ctypes as C

    from . import _lib

    sizes = (C.c_int64 * 6)()
    _lib.check(_lib.lib.sincfft_nnfft_dist_layout(plan.handle, int(world), sizes))
    if not sizes[0]:
        return None
    return {"Sb": sizes[1], "cols": sizes[2], "hblk": sizes[3], "Bc": sizes[4], "Br": sizes[5]}


class DistFftRank:
    """The per-rank steps of the distributed FFT (C ABI ``sincfft_nnfft_dist_*``),
    with the collectives left to the caller:

        send = pack(f)            reduce-scatter(sum) -> block
        cols = colfwd(block)      all-to-all          -> rows
        rowmul(rows)              all-to-all          -> cols2
        hblk = colinv(cols2)      all-gather          -> hall
        out  = gather(hall)

    ``plan`` covers this rank's source and target shards and must be built
    with ``h_window="full"`` (identical FFT on every rank).  Device tensors,
    complex128, single column, on the current torch stream."""

    def __init__(self, plan, world: int, rank: int):
        import torch

        self.plan, self.world, self.rank = plan, int(world), int(rank)
        self.layout = dist_layout(plan, world)
        if self.layout is None:
            raise ValueError("distributed FFT not supported for this plan / world size")
        self.dev = torch.device("cuda", plan.device)
        self.geo = plan.backend_geometry
        self.block = None

    def _s(self):
        import ctypes as C

        import torch
        return C.c_void_p(torch.cuda.current_stream(self.dev).cuda_stream)

    def _empty(self, n):
        import torch
        return torch.empty(int(n), dtype=torch.complex128, device=self.dev)

    def pack(self, f):
        from . import _lib
        grid = self._empty(self.geo["K"])
        _lib.check(_lib.lib.sincfft_nnfft_spread(self.plan.handle, f.data_ptr(), grid.data_ptr(),
                                                 1, _lib.PTR_DEVICE, self._s()))
        send = self._empty(self.world * self.layout["Sb"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_pack(self.plan.handle, self.world, grid.data_ptr(),
                                                    send.data_ptr(), self._s()))
        return send

    def colfwd(self, block):
        from . import _lib
        self.block = block  # colinv reads the reduced tail fix from it (rank 0)
        cols = self._empty(self.layout["cols"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_colfwd(self.plan.handle, self.world, self.rank,
                                                      block.data_ptr(), cols.data_ptr(),
                                                      self._s()))
        return cols

    def rowmul(self, rows):
        from . import _lib
        _lib.check(_lib.lib.sincfft_nnfft_dist_rowmul(self.plan.handle, self.world, self.rank,
                                                      rows.data_ptr(), self._s()))
        return rows

    def colinv(self, cols2):
        from . import _lib
        hblk = self._empty(self.layout["hblk"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_colinv(self.plan.handle, self.world, self.rank,
                                                      cols2.data_ptr(), self.block.data_ptr(),
                                                      hblk.data_ptr(), self._s()))
        return hblk

    def gather(self, hall):
        from . import _lib
        out = self._empty(self.geo["M2"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_gather(self.plan.handle, self.world,
                                                      hall.data_ptr(), out.data_ptr(), self._s()))
        return out


class TorchCollectives:
    """The four collectives over a torch.distributed group: NCCL natively
    (reduce_scatter_tensor / all_to_all_single / all_gather_into_tensor on
    the fp64 view), other backends (gloo, CPU tests and one-GPU validation)
    through CPU staging and all_gather."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"

    def reduce_scatter(self, send):
        import torch
        import torch.distributed as dist
        n = send.numel() // self.world
        if self.nccl:
            out = torch.empty(n, dtype=send.dtype, device=send.device)
            dist.reduce_scatter_tensor(torch.view_as_real(out), torch.view_as_real(send),
                                       group=self.group)
            return out
        buf = torch.view_as_real(send).cpu()
        dist.all_reduce(buf, group=self.group)
        return torch.view_as_complex(buf)[self.rank * n:(self.rank + 1) * n].to(send.device)

    def all_to_all(self, send):
        import torch
        import torch.distributed as dist
        if self.nccl:
            out = torch.empty_like(send)
            dist.all_to_all_single(torch.view_as_real(out), torch.view_as_real(send),
                                   group=self.group)
            return out
        n = send.numel() // self.world
        full = [torch.empty_like(torch.view_as_real(send).cpu()) for _ in range(self.world)]
        dist.all_gather(full, torch.view_as_real(send).cpu(), group=self.group)
        parts = [torch.view_as_complex(b)[self.rank * n:(self.rank + 1) * n] for b in full]
        return torch.cat(parts).to(send.device)

    def all_gather(self, blk):
        import torch
        import torch.distributed as dist
        if self.nccl:
            out = torch.empty(blk.numel() * self.world, dtype=blk.dtype, device=blk.device)
            dist.all_gather_into_tensor(torch.view_as_real(out), torch.view_as_real(blk),
                                        group=self.group)
            return out
        full = [torch.empty_like(torch.view_as_real(blk).cpu()) for _ in range(self.world)]
        dist.all_gather(full, torch.view_as_real(blk).cpu(), group=self.group)
        return torch.view_as_complex(torch.cat(full)).to(blk.device)


class DistributedFftNnfft:
    """One NNFFT over the ranks of a torch.distributed group with the FFT
    split too (no replicated stage): four collectives per transform, sized
    ~(K + 2 L / P + Kout)/P complex per rank instead of an all-reduce of the
    whole K-grid followed by the full FFT on every rank."""

    def __init__(self, plan, group=None):
        self.coll = TorchCollectives(group)
        self.r = DistFftRank(plan, self.coll.world, self.coll.rank)

    def __call__(self, f_shard):
        r, c = self.r, self.coll
        block = c.reduce_scatter(r.pack(f_shard))
        rows = c.all_to_all(r.colfwd(block))
        cols2 = c.all_to_all(r.rowmul(rows))
        return r.gather(c.all_gather(r.colinv(cols2)))


def run_ranks_in_process(ranks, f_shards):
    """All ranks of the distributed FFT in ONE process (e.g. on one GPU): the
    collectives become tensor sums and slices.  Used to validate the layouts
    and kernels of every rank against the unsharded transform without a
    process group; nothing here waits on another rank inside a kernel."""
    import torch

    world = len(ranks)
    sends = [r.pack(f) for r, f in zip(ranks, f_shards)]
    n = sends[0].numel() // world
    total = torch.stack(sends).sum(dim=0)
    blocks = [total[q * n:(q + 1) * n].clone() for q in range(world)]
    cols = [r.colfwd(b) for r, b in zip(ranks, blocks)]

    def a2a(bufs):
        m = bufs[0].numel() // world
        return [torch.cat([bufs[src][dst * m:(dst + 1) * m] for src in range(world)])
                for dst in range(world)]

    rows = a2a(cols)
    rows = [r.rowmul(x) for r, x in zip(ranks, rows)]
    cols2 = a2a(rows)
    hblks = [r.colinv(x) for r, x in zip(ranks, cols2)]
    hall = torch.cat(hblks)
    return [r.gather(hall) for r in ranks]


# ------------------------------------------- sparse exchange (position partitions)
def _i64(vals):
    import ctypes as C
    return (C.c_int64 * len(vals))(*[int(v) for v in vals])


class SparseRows:
    """Row ranges of every rank for the sparse exchange: grid rows
    [ilo, ilo + nrow) a rank's spread touches and h rows [k2lo, k2lo + cnt)
    its gather reads (row = L1 consecutive indices), from each rank's
    ``sincfft_nnfft_dist_support``."""

    def __init__(self, supports, L1, Dpad, Bc):
        self.ilo = [s[0] // L1 for s in supports]
        self.nrow = [s[1] // L1 - s[0] // L1 + 1 for s in supports]
        self.k2lo = [s[2] // L1 for s in supports]
        self.cnt = [s[3] // L1 - s[2] // L1 + 1 for s in supports]
        self.Dpad, self.Bc, self.world = Dpad, Bc, len(supports)

    def grid_send_splits(self, rank):
        return [self.nrow[rank] * self.Bc + (self.Dpad if q == 0 else 0)
                for q in range(self.world)]

    def grid_recv_splits(self, rank):
        return [self.nrow[s] * self.Bc + (self.Dpad if rank == 0 else 0)
                for s in range(self.world)]

    def h_send_splits(self, rank):
        return [self.cnt[r] * self.Bc for r in range(self.world)]

    def h_recv_splits(self, rank):
        return [self.cnt[rank] * self.Bc for _ in range(self.world)]


class SparseDistFftRank(DistFftRank):
    """DistFftRank with the sparse first and last exchanges
    (``sincfft_nnfft_dist_pack_rows`` / ``_unpack_rows`` / ``_pack_hrows`` /
    ``_gather_rows``); the middle two all-to-alls are unchanged."""

    def support(self):
        import ctypes as C

        from . import _lib
        out = (C.c_int64 * 4)()
        _lib.check(_lib.lib.sincfft_nnfft_dist_support(self.plan.handle, out, self._s()))
        return [int(v) for v in out]

    def set_rows(self, rows: SparseRows):
        self.rows = rows

    def pack_rows(self, f):
        from . import _lib
        grid = self._empty(self.geo["K"])
        _lib.check(_lib.lib.sincfft_nnfft_spread(self.plan.handle, f.data_ptr(), grid.data_ptr(),
                                                 1, _lib.PTR_DEVICE, self._s()))
        rw, r = self.rows, self.rank
        send = self._empty(sum(rw.grid_send_splits(r)))
        _lib.check(_lib.lib.sincfft_nnfft_dist_pack_rows(self.plan.handle, self.world,
                                                         grid.data_ptr(), rw.ilo[r], rw.nrow[r],
                                                         send.data_ptr(), self._s()))
        return send

    def unpack_rows(self, recv):
        from . import _lib
        rw = self.rows
        block = self._empty(self.layout["Sb"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_unpack_rows(
            self.plan.handle, self.world, self.rank, recv.data_ptr(), _i64(rw.ilo),
            _i64(rw.nrow), block.data_ptr(), self._s()))
        return block

    def pack_hrows(self, hblk):
        from . import _lib
        rw = self.rows
        send = self._empty(sum(rw.h_send_splits(self.rank)))
        _lib.check(_lib.lib.sincfft_nnfft_dist_pack_hrows(
            self.plan.handle, self.world, hblk.data_ptr(), _i64(rw.k2lo), _i64(rw.cnt),
            send.data_ptr(), self._s()))
        return send

    def gather_rows(self, recv):
        from . import _lib
        rw, r = self.rows, self.rank
        out = self._empty(self.geo["M2"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_gather_rows(
            self.plan.handle, self.world, recv.data_ptr(), rw.k2lo[r], rw.cnt[r],
            out.data_ptr(), self._s()))
        return out


def sparse_rows_for(ranks_supports, rank0: DistFftRank):
    geo = rank0.geo
    L1 = geo["L1"]
    I = -(-geo["K"] // L1)
    return SparseRows(ranks_supports, L1, rank0.layout["Sb"] - I * rank0.layout["Bc"],
                      rank0.layout["Bc"])


def _all_to_all_v(coll, send, in_splits, out_splits):
    import torch
    import torch.distributed as dist
    if coll.nccl:
        out = torch.empty(sum(out_splits), dtype=send.dtype, device=send.device)
        dist.all_to_all_single(torch.view_as_real(out), torch.view_as_real(send),
                               output_split_sizes=out_splits, input_split_sizes=in_splits,
                               group=coll.group)
        return out
    # other backends: pad to the longest send buffer, all-gather, pick chunks
    n = torch.tensor([send.numel()], dtype=torch.int64)
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(coll.world)]
    dist.all_gather(sizes, n, group=coll.group)
    width = int(max(s.item() for s in sizes))
    splits = torch.tensor(in_splits, dtype=torch.int64)
    all_splits = [torch.zeros_like(splits) for _ in range(coll.world)]
    dist.all_gather(all_splits, splits, group=coll.group)
    buf = torch.zeros((width, 2), dtype=torch.float64)
    buf[:send.numel()] = torch.view_as_real(send).cpu()
    full = [torch.empty_like(buf) for _ in range(coll.world)]
    dist.all_gather(full, buf, group=coll.group)
    parts = []
    for s in range(coll.world):
        off = int(all_splits[s][:coll.rank].sum())
        parts.append(torch.view_as_complex(full[s][off:off + out_splits[s]].contiguous()))
    return torch.cat(parts).to(send.device)


class SparseDistributedFftNnfft:
    """DistributedFftNnfft for position partitions: the K-grid and h exchanges
    move only the rows each rank touches (per rank ~(K + Kout)/P complex
    instead of K + Kout); plans built with ``h_window="full"``."""

    def __init__(self, plan, group=None):
        import torch
        import torch.distributed as dist

        self.coll = TorchCollectives(group)
        self.r = SparseDistFftRank(plan, self.coll.world, self.coll.rank)
        mine = torch.tensor(self.r.support(), dtype=torch.int64,
                            device=self.r.dev if self.coll.nccl else "cpu")
        allsup = [torch.zeros_like(mine) for _ in range(self.coll.world)]
        dist.all_gather(allsup, mine, group=group)
        self.r.set_rows(sparse_rows_for([a.tolist() for a in allsup], self.r))

    def __call__(self, f_shard):
        r, c, rw, k = self.r, self.coll, self.r.rows, self.coll.rank
        recv = _all_to_all_v(c, r.pack_rows(f_shard), rw.grid_send_splits(k),
                             rw.grid_recv_splits(k))
        rows = c.all_to_all(r.colfwd(r.unpack_rows(recv)))
        hblk = r.colinv(c.all_to_all(r.rowmul(rows)))
        recv2 = _all_to_all_v(c, r.pack_hrows(hblk), rw.h_send_splits(k), rw.h_recv_splits(k))
        return r.gather_rows(recv2)


def run_sparse_ranks_in_process(ranks, f_shards):
    """run_ranks_in_process for SparseDistFftRank (one process, one GPU)."""
    import torch

    world = len(ranks)
    rows = sparse_rows_for([r.support() for r in ranks], ranks[0])
    for r in ranks:
        r.set_rows(rows)

    def a2av(sends, send_splits):
        chunks = [list(torch.split(s, send_splits(i))) for i, s in enumerate(sends)]
        return [torch.cat([chunks[src][dst] for src in range(world)]) for dst in range(world)]

    recv = a2av([r.pack_rows(f) for r, f in zip(ranks, f_shards)], rows.grid_send_splits)
    blocks = [r.unpack_rows(x) for r, x in zip(ranks, recv)]
    cols = [r.colfwd(b) for r, b in zip(ranks, blocks)]

    def a2a(bufs):
        m = bufs[0].numel() // world
        return [torch.cat([bufs[src][dst * m:(dst + 1) * m] for src in range(world)])
                for dst in range(world)]

    rws = [r.rowmul(x) for r, x in zip(ranks, a2a(cols))]
    hblks = [r.colinv(x) for r, x in zip(ranks, a2a(rws))]
    recv2 = a2av([r.pack_hrows(h) for r, h in zip(ranks, hblks)], rows.h_send_splits)
    return [r.gather_rows(x) for r, x in zip(ranks, recv2)]


# --------------------------------------- fused transposes over peer memory
def _u64(ptrs):
    import ctypes as C
    return (C.c_uint64 * len(ptrs))(*[int(p) for p in ptrs])


class PeerDistFftRank(SparseDistFftRank):
    """SparseDistFftRank whose two middle all-to-alls are fused into the passes:
    the column pass stores each element into the row-owner's receive buffer,
    the row pass into the column-owner's (``sincfft_nnfft_dist_colfwd_peer`` /
    ``_rowmul_peer``; the buffers are mapped over NVLink with CUDA IPC)."""

    def colfwd_peer(self, block, rows_ptrs):
        from . import _lib
        self.block = block
        _lib.check(_lib.lib.sincfft_nnfft_dist_colfwd_peer(
            self.plan.handle, self.world, self.rank, block.data_ptr(), _u64(rows_ptrs),
            self._s()))

    def rowmul_peer(self, rows_ptr, cols2_ptrs):
        from . import _lib
        _lib.check(_lib.lib.sincfft_nnfft_dist_rowmul_peer(
            self.plan.handle, self.world, self.rank, rows_ptr, _u64(cols2_ptrs), self._s()))

    def grid_offsets(self):
        """poff[q]: this rank's chunk offset in receiver q's grid-row buffer."""
        rw, out = self.rows, []
        for q in range(self.world):
            extra = rw.Dpad if q == 0 else 0
            out.append(sum(rw.nrow[s] * rw.Bc + extra for s in range(self.rank)))
        return out

    def grid_recv_elems(self):
        return sum(self.rows.grid_recv_splits(self.rank))

    def h_recv_elems(self):
        return sum(self.rows.h_recv_splits(self.rank))

    def pack_rows_peer(self, f, grid_ptrs):
        from . import _lib
        grid = self._empty(self.geo["K"])
        _lib.check(_lib.lib.sincfft_nnfft_spread(self.plan.handle, f.data_ptr(), grid.data_ptr(),
                                                 1, _lib.PTR_DEVICE, self._s()))
        rw, r = self.rows, self.rank
        _lib.check(_lib.lib.sincfft_nnfft_dist_pack_rows_peer(
            self.plan.handle, self.world, r, grid.data_ptr(), rw.ilo[r], rw.nrow[r],
            _u64(grid_ptrs), _i64(self.grid_offsets()), self._s()))
        self._grid_keep = grid  # alive until the stream passes the barrier

    def unpack_rows_ptr(self, recv_ptr):
        from . import _lib
        rw = self.rows
        block = self._empty(self.layout["Sb"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_unpack_rows(
            self.plan.handle, self.world, self.rank, recv_ptr, _i64(rw.ilo), _i64(rw.nrow),
            block.data_ptr(), self._s()))
        return block

    def colinv_peer(self, cols2_ptr, h_ptrs):
        from . import _lib
        rw = self.rows
        _lib.check(_lib.lib.sincfft_nnfft_dist_colinv_peer(
            self.plan.handle, self.world, self.rank, cols2_ptr, self.block.data_ptr(),
            _u64(h_ptrs), _i64(rw.k2lo), _i64(rw.cnt), self._s()))

    def gather_rows_ptr(self, recv_ptr):
        from . import _lib
        rw, r = self.rows, self.rank
        out = self._empty(self.geo["M2"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_gather_rows(
            self.plan.handle, self.world, recv_ptr, rw.k2lo[r], rw.cnt[r], out.data_ptr(),
            self._s()))
        return out

    def colinv_ptr(self, cols2_ptr):
        from . import _lib
        hblk = self._empty(self.layout["hblk"])
        _lib.check(_lib.lib.sincfft_nnfft_dist_colinv(self.plan.handle, self.world, self.rank,
                                                      cols2_ptr, self.block.data_ptr(),
                                                      hblk.data_ptr(), self._s()))
        return hblk


class IpcBuffer:
    """A device buffer of this rank mapped into every other rank (CUDA IPC):
    ``ptrs[q]`` is rank q's buffer as seen from this process."""

    def __init__(self, device, nbytes, coll):
        import ctypes as C

        import torch
        import torch.distributed as dist

        from . import _lib
        self.device = device
        p = C.c_void_p()
        _lib.check(_lib.lib.sincfft_ipc_alloc(device, int(nbytes), C.byref(p)))
        self.own = p.value
        h = (C.c_uint8 * 64)()
        _lib.check(_lib.lib.sincfft_ipc_handle(C.c_void_p(self.own), h))
        mine = torch.tensor(list(bytes(h)), dtype=torch.uint8,
                            device=torch.device("cuda", device) if coll.nccl else "cpu")
        allh = [torch.zeros_like(mine) for _ in range(coll.world)]
        dist.all_gather(allh, mine, group=coll.group)
        self.ptrs, self._opened = [], []
        for q, t in enumerate(allh):
            if q == coll.rank:
                self.ptrs.append(self.own)
                continue
            hq = (C.c_uint8 * 64)(*t.cpu().tolist())
            pq = C.c_void_p()
            _lib.check(_lib.lib.sincfft_ipc_open(device, hq, C.byref(pq)))
            self.ptrs.append(pq.value)
            self._opened.append(pq.value)

    def close(self):
        import ctypes as C

        from . import _lib
        for p in self._opened:
            _lib.lib.sincfft_ipc_close(C.c_void_p(p))
        self._opened = []
        if self.own:
            _lib.lib.sincfft_ipc_free(C.c_void_p(self.own))
            self.own = None


class PeerDistributedFftNnfft:
    """The distributed FFT with every exchange fused into a kernel over peer
    memory: the grid rows are packed straight into their owners' buffers, the
    two transposes are the column / row passes' stores, and the inverse column
    pass stores each h row into every rank whose targets read it.  Per
    transform: four stream-ordered barriers and no data collective.

    The peer receive buffers are persistent and shared by every call, so calls
    are serialised: each call's stream first waits on an event recorded at the
    end of the previous call (whatever stream that was on).  Within one call
    the barriers order every peer store before its reader."""

    def __init__(self, plan, group=None):
        import torch
        import torch.distributed as dist

        self.coll = TorchCollectives(group)
        self.r = PeerDistFftRank(plan, self.coll.world, self.coll.rank)
        mine = torch.tensor(self.r.support(), dtype=torch.int64,
                            device=self.r.dev if self.coll.nccl else "cpu")
        allsup = [torch.zeros_like(mine) for _ in range(self.coll.world)]
        dist.all_gather(allsup, mine, group=group)
        self.r.set_rows(sparse_rows_for([a.tolist() for a in allsup], self.r))
        cols = 16 * self.r.layout["cols"]
        self.gridrecv = IpcBuffer(plan.device, 16 * self.r.grid_recv_elems(), self.coll)
        self.rows = IpcBuffer(plan.device, cols, self.coll)
        self.cols2 = IpcBuffer(plan.device, cols, self.coll)
        self.hrecv = IpcBuffer(plan.device, 16 * self.r.h_recv_elems(), self.coll)
        self._flag = torch.zeros(1, dtype=torch.float64, device=self.r.dev)
        self._done = None  # event recorded at the end of the previous call

    def _barrier(self):
        """Every rank's peer stores have landed: a stream-ordered all-reduce
        (NCCL) or a host barrier (other backends)."""
        import torch
        import torch.distributed as dist
        if self.coll.nccl:
            dist.all_reduce(self._flag, group=self.coll.group)
        else:
            torch.cuda.synchronize(self.r.dev)
            dist.barrier(group=self.coll.group)

    def __call__(self, f_shard):
        import torch
        r = self.r
        cur = torch.cuda.current_stream(r.dev)
        if self._done is not None:  # the previous call (any stream) has released the buffers
            cur.wait_event(self._done)
        r.pack_rows_peer(f_shard, self.gridrecv.ptrs)
        self._barrier()
        r.colfwd_peer(r.unpack_rows_ptr(self.gridrecv.own), self.rows.ptrs)
        self._barrier()
        r.rowmul_peer(self.rows.own, self.cols2.ptrs)
        self._barrier()
        r.colinv_peer(self.cols2.own, self.hrecv.ptrs)
        self._barrier()
        out = r.gather_rows_ptr(self.hrecv.own)
        self._done = torch.cuda.Event()
        self._done.record(cur)
        return out

    def close(self):
        for b in (self.gridrecv, self.rows, self.cols2, self.hrecv):
            b.close()


def run_peer_ranks_in_process(ranks, f_shards):
    """PeerDistributedFftNnfft with all ranks in one process (one GPU): a
    rank's 'peer' buffers are simply the other ranks' tensors."""
    world = len(ranks)
    rows = sparse_rows_for([r.support() for r in ranks], ranks[0])
    for r in ranks:
        r.set_rows(rows)
    gbuf = [r._empty(r.grid_recv_elems()) for r in ranks]
    rbuf = [r._empty(r.layout["cols"]) for r in ranks]
    cbuf = [r._empty(r.layout["cols"]) for r in ranks]
    hbuf = [r._empty(r.h_recv_elems()) for r in ranks]
    ptrs = lambda bufs: [x.data_ptr() for x in bufs]  # noqa: E731
    for r, f in zip(ranks, f_shards):
        r.pack_rows_peer(f, ptrs(gbuf))
    for r, g in zip(ranks, gbuf):
        r.colfwd_peer(r.unpack_rows_ptr(g.data_ptr()), ptrs(rbuf))
    for r, x in zip(ranks, rbuf):
        r.rowmul_peer(x.data_ptr(), ptrs(cbuf))
    for r, y in zip(ranks, cbuf):
        r.colinv_peer(y.data_ptr(), ptrs(hbuf))
    assert world == len(hbuf)
    return [r.gather_rows_ptr(h.data_ptr()) for r, h in zip(ranks, hbuf)]
