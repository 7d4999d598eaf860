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
