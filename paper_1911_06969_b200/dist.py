"""Multi-GPU plumbing: one process per GPU, torch.distributed (NCCL over
NVLink/NVSwitch on the GPU box; gloo in CPU tests) behind the C ABI's
``gpm_exchange_fn`` hook.

The engine partitions root units (level-1 entries) by a degree-weighted static
split computed identically on every rank (no communication), so the only
exchanges are:
  * op 0  sum of u64 per-pattern counters / per-level size vectors (C1)
  * op 1  bitwise OR of u32 domain bitmaps (FSM, C2) — NCCL has no bitwise
          reduction, so it is owner-based: an all-to-all hands every rank the
          N copies of its 1/N slice of the words, the rank ORs them on the
          device, and an all-gather returns the ORed slices (2(N-1)/N of the
          bitmap bytes per GPU, vs (N-1)x for all-gather + local OR)
  * op 2  all-gather (FSM pattern-key union)

Load balance beyond the static split: ``StealCounters`` creates the shared
work-stealing counters of gpm_config.steal_ctrs (one uint64 per rank on rank
0's GPU, exported by CUDA IPC and peer-mapped over NVLink by the other ranks);
the engine claims chunks of every rank's tail with device-side system-scope
atomics once its own head is done.
"""
from __future__ import annotations

import ctypes as C

from ._lib import EXCHANGE_FN, check, lib

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
        owner_or_(t, group)
    elif op == 2:  # t holds world * n elements, this rank's slot filled
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        n = t.numel() // world
        mine = t[rank * n:(rank + 1) * n].clone()
        parts = [torch.empty_like(mine) for _ in range(world)]
        dist.all_gather(parts, mine, group=group)
        t.copy_(torch.cat(parts))
    else:
        raise ValueError(f"unknown exchange op {op}")


def owner_or_(t, group=None):
    """In-place bitwise OR over ranks, owner-based (the algorithm of the
    in-library NCCL hook, csrc/nccl_exchange.cu): pad to world * per words,
    all-to-all the slices to their owners, OR, all-gather."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if world == 1:
        return t
    n = t.numel()
    per = (n + world - 1) // world
    src = t
    if per * world != n:
        src = torch.zeros(per * world, dtype=t.dtype, device=t.device)
        src[:n] = t
    parts = torch.empty_like(src)
    dist.all_to_all_single(parts, src, group=group)
    own = parts.view(world, per)[0].clone()
    for q in range(1, world):
        own.bitwise_or_(parts.view(world, per)[q])
    out = torch.empty_like(src)
    dist.all_gather_into_tensor(out, own, group=group)
    t.copy_(out[:n])
    return t


def dist_world(group=None) -> int:
    import torch.distributed as dist
    return dist.get_world_size(group)


def make_exchange(group=None):
    """Returns a ctypes gpm_exchange_fn bound to torch.distributed."""
    import torch

    def _cb(ctx, dev_buf, count, elem_bytes, op, stream):
        try:
            # op 2 (all-gather): `count` is per rank, the buffer holds world * count
            n = count * (dist_world(group) if op == 2 else 1)
            t = torch.as_tensor(_DevArray(dev_buf, n, elem_bytes), device="cuda")
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


class NativeExchange:
    """The in-library NCCL exchange (gpm_exchange_nccl_*; no Python callback on
    the exchange path).  Rank 0 draws the NCCL unique id, torch.distributed
    broadcasts its 128 bytes, every rank creates its communicator on its GPU.
    Pass ``exchange=ex.fn, exchange_ctx=ex.ctx`` to mine()."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        L = lib()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_char * 128)()
        if rank == 0:
            check(L.gpm_nccl_unique_id(uid))
        on_cuda = dist.get_backend(group) == "nccl"
        h = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device="cuda" if on_cuda else "cpu")
        dist.broadcast(h, 0, group=group)
        raw = bytes(h.cpu().tolist())
        ctx = C.c_void_p()
        check(L.gpm_exchange_nccl_create(raw, rank, world, torch.cuda.current_device(), C.byref(ctx)))
        self.ctx = ctx.value
        self.fn = L.gpm_exchange_nccl_fn()

    def close(self):
        if self.ctx:
            check(lib().gpm_exchange_nccl_destroy(self.ctx))
            self.ctx = None


class StealCounters:
    """Shared steal counters for one process per GPU (gpm_steal_* in gpm.h).

    Rank 0 allocates ``world`` counters on its device and broadcasts the CUDA
    IPC handle; every other rank opens it (peer mapping).  Call ``reset()``
    (collective) before each mine; pass ``ptr`` as ``steal_ctrs``."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        dev = torch.cuda.current_device()
        L = lib()
        handle = (C.c_char * 64)()
        ptr = C.c_void_p()
        if self.rank == 0:
            check(L.gpm_steal_create(dev, self.world, C.byref(ptr), handle))
        on_cuda = dist.get_backend(group) == "nccl"
        h = torch.tensor(list(bytes(handle)), dtype=torch.uint8, device="cuda" if on_cuda else "cpu")
        dist.broadcast(h, 0, group=group)
        if self.rank != 0:
            raw = bytes(h.cpu().tolist())
            check(L.gpm_steal_open(dev, raw, C.byref(ptr)))
        self._opened = int(self.rank != 0)
        self.ptr = ptr.value

    def reset(self):
        import torch.distributed as dist
        dist.barrier(group=self.group)
        if self.rank == 0:
            check(lib().gpm_steal_reset(self.ptr, self.world, None))
        dist.barrier(group=self.group)

    def close(self):
        import torch.distributed as dist
        dist.barrier(group=self.group)   # peers unmap before the owner frees
        if self._opened and self.ptr:
            check(lib().gpm_steal_release(self.ptr, 1))
        dist.barrier(group=self.group)
        if not self._opened and self.ptr:
            check(lib().gpm_steal_release(self.ptr, 0))
        self.ptr = None
