"""Seed sharding over torch.distributed: the exchange callback for
Context.set_exchange.

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


def enable_seed_sharding(ctx, group=None):
    """Make `ctx` iterate only this rank's share of every round's seeds (all ranks must call the
    clustering entry points with identical inputs; each returns the full result)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if world == 1:
        ctx.set_exchange(None, 0, 1)
    else:
        ctx.set_exchange(make_exchange(group), rank, world)
    return ctx
