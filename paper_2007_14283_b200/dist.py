"""Seed sharding and pixel sharding (8(e)3) over torch.distributed: in-library NCCL
(the unique id shared through torch.distributed) or the exchange / all-gather callbacks for
Context.set_exchange / set_allgather / set_pixel_shard.

The library calls the exchange at its two collective points (per lockstep step: per-frame counts;
per round: the owners' converged seeds) with an int32 device buffer and its stream; this module
sums it over the process group in place.  With the NCCL backend the all-reduce is enqueued on the
library's stream (no host round trip); with gloo (tests on one GPU, CPU transport) the buffer goes
through host memory.  Plumbing only -- no step of the method runs here.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


class _DevBuf:
    """Zero-copy view of a raw int32 device buffer (CUDA array interface)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": "<i4", "data": (int(ptr), False),
                                         "version": 3, "strides": None}


def make_exchange(group=None):
    backend = dist.get_backend(group)

    def exchange(ptr: int, count: int, stream: int) -> int:
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            t = torch.as_tensor(_DevBuf(ptr, count), device="cuda")
            if backend == "nccl":
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
            else:
                h = t.cpu()  # synchronous on s
                dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
                t.copy_(h)
                s.synchronize()
        return 0

    return exchange


def make_allgather(group=None):
    """The all-gather of seed sharding's round exchange: rank r's `count` int32 values land at
    recv[r * count, (r + 1) * count)."""
    backend = dist.get_backend(group)
    world = dist.get_world_size(group)

    def allgather(send_ptr: int, recv_ptr: int, count: int, stream: int) -> int:
        s = torch.cuda.ExternalStream(stream) if stream else torch.cuda.current_stream()
        with torch.cuda.stream(s):
            snd = torch.as_tensor(_DevBuf(send_ptr, count), device="cuda")
            rcv = torch.as_tensor(_DevBuf(recv_ptr, count * world), device="cuda")
            if backend == "nccl":
                dist.all_gather_into_tensor(rcv, snd, group=group)
            else:
                h = snd.cpu()  # synchronous on s
                parts = [torch.empty_like(h) for _ in range(world)]
                dist.all_gather(parts, h, group=group)
                rcv.copy_(torch.cat(parts))
                s.synchronize()
        return 0

    return allgather


def _share_unique_id(group=None) -> bytes:
    import paper_2007_14283_b200 as fms
    obj = [fms.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def enable_seed_sharding(ctx, group=None, in_library=None):
    """Make `ctx` iterate only this rank's share of every round's seeds (all ranks must call the
    clustering entry points with identical inputs; each returns the full result).  With the NCCL
    backend the collectives run as NCCL calls inside the library (include/fms.h fms_set_nccl: no
    Python callback per lockstep step); otherwise (gloo: tests with several ranks on one GPU) through
    the callbacks above, the round exchange as an all-gather of owned rows."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        ctx.set_exchange(None, 0, 1)
        return ctx
    if in_library is None:
        in_library = dist.get_backend(group) == "nccl"
    if in_library:
        import paper_2007_14283_b200 as fms
        ctx.set_nccl(_share_unique_id(group), rank, world, fms.SHARD_SEEDS)
    else:
        ctx.set_exchange(make_exchange(group), rank, world)
        ctx.set_allgather(make_allgather(group))
    return ctx


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous pixel range [lo, hi) of `rank` when n pixels are split over `world` ranks (sizes
    differ by at most one; the first n % world ranks take one more)."""
    if not (0 <= rank < world) or n < world:
        raise ValueError("need 0 <= rank < world <= n")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def enable_pixel_sharding(ctx, n_global: int, group=None, in_library=None):
    """Make `ctx` cluster frames of n_global pixels of which this rank holds shard_range(n_global, rank,
    world): pass this rank's rows to the clustering calls; every rank returns the same centres and K,
    and labels for its own rows.  Returns (lo, hi)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        ctx.set_pixel_shard(None, 0, 1, n_global, 0)
        return 0, n_global
    lo, hi = shard_range(n_global, rank, world)
    if in_library is None:
        in_library = dist.get_backend(group) == "nccl"
    if in_library:
        import paper_2007_14283_b200 as fms
        ctx.set_nccl(_share_unique_id(group), rank, world, fms.SHARD_PIXELS, n_global, lo)
    else:
        ctx.set_pixel_shard(make_exchange(group), rank, world, n_global, lo)
    return lo, hi
