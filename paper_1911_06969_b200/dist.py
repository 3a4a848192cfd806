"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box; gloo in CPU tests) behind the C ABI's
``gpm_exchange_fn`` hook.

The engine partitions root units (level-1 entries) by a degree-weighted static
split computed identically on every rank (no communication), so the only
exchanges are:
  * op 0  sum of u64 per-pattern counters / per-level size vectors (C1)
  * op 1  bitwise OR of u32 domain bitmaps (FSM, C2) — NCCL has no bitwise
          reduction, so it is an all-gather of the packed words followed by an
          OR-reduction on the device
  * op 2  all-gather (FSM pattern-key union)
"""
from __future__ import annotations

import ctypes as C

from ._lib import EXCHANGE_FN

_TYPESTR = {1: "|u1", 4: "<u4", 8: "<u8"}


class _DevArray:
    def __init__(self, ptr: int, count: int, elem_bytes: int):
        self.__cuda_array_interface__ = {
            "shape": (count,), "typestr": _TYPESTR[elem_bytes], "data": (ptr, False), "version": 3,
            "strides": None, "stream": None,
        }


def exchange_op(t, op: int, group=None):
    """Performs exchange `op` in place on tensor t (any device torch.distributed supports)."""
    import torch
    import torch.distributed as dist
    if op == 0:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    elif op == 1:
        world = dist.get_world_size(group)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        acc = parts[0].clone()
        for p in parts[1:]:
            acc.bitwise_or_(p)
        t.copy_(acc)
    elif op == 2:
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        n = t.numel() // world
        mine = t[rank * n:(rank + 1) * n].clone()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        t.copy_(torch.cat(parts))
    else:
        raise ValueError(f"unknown exchange op {op}")


def make_exchange(group=None):
    """Returns a ctypes gpm_exchange_fn bound to torch.distributed."""
    import torch

    def _cb(ctx, dev_buf, count, elem_bytes, op, stream):
        try:
            t = torch.as_tensor(_DevArray(dev_buf, count, elem_bytes), device="cuda")
            if elem_bytes == 8 and op == 0:
                t = t.view(torch.int64)  # NCCL sums int64 == uint64 modulo 2^64
            elif elem_bytes == 4:
                t = t.view(torch.int32)
            exchange_op(t, op, group)
            torch.cuda.current_stream().synchronize()
            return 0
        except Exception as e:  # never let an exception cross the C boundary
            print(f"[gpm exchange] {e!r}")
            return 1

    return EXCHANGE_FN(_cb)
