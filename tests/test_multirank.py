"""Multi-rank (N>1) coverage.

* CPU, world_size 2 over gloo: the exchange ops the engine's hook performs
  (sum / bitwise OR / all-gather; paper_1911_06969_b200/dist.py) and
  partition invariance of root-unit sharding with a count all-reduce.
* GPU: two ranks as two threads on one device with an in-process exchange,
  driving the real engine's multi-rank code paths (degree-weighted root split,
  count exchange, FSM pattern-key union + domain-bitmap OR) and checking the
  result equals the single-rank run.
"""
import os
import socket
import threading

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bruteforce as BF

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1911_06969_b200.dist import exchange_op
        out = {}
        t = torch.tensor([rank + 1, 10 * (rank + 1)], dtype=torch.int64)
        exchange_op(t, 0)
        out["sum"] = t.tolist()
        b = torch.tensor([1 << rank, 0x100 << rank], dtype=torch.int32)
        exchange_op(b, 1)
        out["or"] = b.tolist()
        # owner-based OR (the algorithm of csrc/nccl_exchange.cu): word counts
        # that do and do not divide by the world size, against a plain OR
        from paper_1911_06969_b200.dist import owner_or_
        ok = []
        for n in (1, 2, 7, 64, 1001):
            arrs = [torch.from_numpy(np.random.default_rng(100 * q + n).integers(0, 2**31, n).astype(np.int32))
                    for q in range(world)]
            want = arrs[0].clone()
            for a in arrs[1:]:
                want |= a
            mine = arrs[rank].clone()
            owner_or_(mine)
            ok.append(bool(torch.equal(mine, want)))
        out["owner_or"] = ok
        g = torch.zeros(2 * world, dtype=torch.int64)
        g[2 * rank:2 * rank + 2] = torch.tensor([rank, rank + 100])
        exchange_op(g, 2)
        out["gather"] = g.tolist()
        # partition invariance with the oracle: each rank mines its root slice
        import pyoracle
        E = BF.gnp(160, 0.1, 9)
        c = pyoracle.csr_from_edges(E, 160)
        full_n1 = pyoracle.mine(c, "cf", 4)["level_sizes"][0]
        lo, hi = rank * full_n1 // world, (rank + 1) * full_n1 // world
        r = pyoracle.mine(c, "cf", 4, root_lo=lo, root_hi=hi)
        cnt = torch.tensor([r["total"], r["n_explored"]], dtype=torch.int64)
        exchange_op(cnt, 0)
        out["cf4"] = cnt.tolist()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_exchange_and_partition(oracle, world):
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["sum"] == [sum(range(1, world + 1)), 10 * sum(range(1, world + 1))]
        assert res[r]["or"] == [(1 << world) - 1, ((1 << world) - 1) << 8]
        assert res[r]["gather"] == sum(([q, q + 100] for q in range(world)), [])
        assert all(res[r]["owner_or"])
    full = oracle.mine(oracle.csr_from_edges(BF.gnp(160, 0.1, 9), 160), "cf", 4)
    assert res[0]["cf4"] == [full["total"], full["n_explored"]] == res[1]["cf4"]


# ------------------------------------------------------------------ GPU, threaded ranks
class ThreadedExchange:
    """In-process stand-in for torch.distributed: ranks are threads."""

    def __init__(self, world):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.result = None
        self.lock = threading.Lock()

    def fn(self, rank):
        from paper_1911_06969_b200._lib import EXCHANGE_FN
        from paper_1911_06969_b200.dist import _DevArray

        def cb(ctx, ptr, count, eb, op, stream):
            try:
                n = count * (self.world if op == 2 else 1)  # op 2: per-rank count, world slots
                t = torch.as_tensor(_DevArray(ptr, n, eb), device="cuda")
                t = t.view(torch.int64) if eb == 8 else t.view(torch.int32)
                self.slots[rank] = t.cpu()
                self.barrier.wait()
                if rank == 0:
                    acc = self.slots[0].clone()
                    for s in self.slots[1:]:
                        if op == 0:
                            acc += s
                        elif op == 1:
                            acc |= s
                        elif op == 2:  # disjoint slots: sum == all-gather
                            acc += s
                        else:
                            raise ValueError(op)
                    self.result = acc
                self.barrier.wait()
                t.copy_(self.result.to("cuda"))
                torch.cuda.synchronize()
                self.barrier.wait()
                return 0
            except Exception as e:  # pragma: no cover
                print("exchange failed", e)
                self.barrier.abort()
                return 1

        return EXCHANGE_FN(cb)


def _run_ranks(P, hg, app, k, sigma, world, steal=None, steal_chunk=0):
    ex = ThreadedExchange(world)
    out = [None] * world
    errs = []
    fns = [ex.fn(r) for r in range(world)]

    def run(r):
        try:
            g = P.Graph(hg)
            kw = dict(steal_ctrs=steal.data_ptr(), steal_chunk=steal_chunk) if steal is not None else {}
            out[r] = P.mine(g, app, k, sigma, rank=r, world=world, exchange=fns[r], **kw)
        except Exception as e:
            errs.append(e)
            ex.barrier.abort()

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    assert not errs, errs
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_threaded_ranks_match_single(world):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    hg = P.generate_rmat(12, 8, 0.45, 0.15, 0.15, seed=5, n_labels=6, label_seed=101)
    for app, k, sigma in (("tc", 3, 0), ("cf", 4, 0), ("mc", 3, 0), ("mc", 4, 0), ("fsm", 4, 30), ("fsm", 3, 5)):
        base = P.mine(P.Graph(hg), app, k, sigma)
        outs = _run_ranks(P, hg, app, k, sigma, world)
        for r in outs:
            assert r.total == base.total, (app, k)
            assert r.patterns == base.patterns, (app, k)
            assert r.stats["n_explored"] == base.stats["n_explored"], (app, k)
            assert r.stats["level_sizes"] == base.stats["level_sizes"], (app, k)


@pytest.mark.gpu
@pytest.mark.parametrize("world,chunk", [(2, 0), (3, 97), (4, 1024)])
def test_threaded_work_stealing_tail(world, chunk):
    """Device-side stealing over shared counters (gpm_config.steal_ctrs): every
    level-1 root unit is mined exactly once whatever the interleaving, so the
    reduced result equals the single-rank one."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    hg = P.generate_rmat(13, 8, 0.57, 0.19, 0.19, seed=6)
    for app, k in (("tc", 3), ("cf", 4), ("cf", 5), ("mc", 3), ("mc", 4)):
        base = P.mine(P.Graph(hg), app, k)
        ctrs = torch.zeros(world, dtype=torch.int64, device="cuda")
        outs = _run_ranks(P, hg, app, k, 0, world, steal=ctrs, steal_chunk=chunk)
        for r in outs:
            assert r.total == base.total, (app, k)
            assert r.patterns == base.patterns, (app, k)
            assert r.stats["n_explored"] == base.stats["n_explored"], (app, k)
            assert r.stats["level_sizes"] == base.stats["level_sizes"], (app, k)
            assert r.stats["candidates"] == base.stats["candidates"], (app, k)
        # every tail was drained: counters >= the tail lengths
        assert int(ctrs.min().item()) > 0


def _ipc_worker(rank, world, port, q):
    """One process per rank on the same GPU: the steal counters live on rank
    0's allocation and are opened by the other ranks through CUDA IPC (the
    multi-GPU path peer-maps them over NVLink the same way)."""
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1911_06969_b200 as P
        from paper_1911_06969_b200._lib import EXCHANGE_FN
        from paper_1911_06969_b200.dist import StealCounters, _DevArray, exchange_op

        def cb(ctx, ptr, count, eb, op, stream):  # device buffer -> host gloo collective -> device
            n = count * (world if op == 2 else 1)  # op 2: per-rank count, world slots
            t = torch.as_tensor(_DevArray(ptr, n, eb), device="cuda")
            t = t.view(torch.int64) if eb == 8 else t.view(torch.int32)
            h = t.cpu()
            exchange_op(h, op)
            t.copy_(h.to("cuda"))
            torch.cuda.synchronize()
            return 0

        fn = EXCHANGE_FN(cb)
        steal = StealCounters()
        hg = P.generate_rmat(13, 8, 0.57, 0.19, 0.19, seed=8)
        out = {}
        for app, k in (("tc", 3), ("cf", 4), ("mc", 3)):
            steal.reset()
            r = P.mine(P.Graph(hg), app, k, rank=rank, world=world, exchange=fn, steal_ctrs=steal.ptr, steal_chunk=64)
            out[f"{app}{k}"] = (r.total, r.stats["n_explored"], sorted(r.patterns))
        steal.close()
        q.put((rank, out))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_ipc_steal_counters_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1911_06969_b200 as P
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    hg = P.generate_rmat(13, 8, 0.57, 0.19, 0.19, seed=8)
    for r in range(world):
        assert isinstance(res[r], dict), res[r]
        for app, k in (("tc", 3), ("cf", 4), ("mc", 3)):
            base = P.mine(P.Graph(hg), app, k)
            assert res[r][f"{app}{k}"] == (base.total, base.stats["n_explored"], sorted(base.patterns)), (app, k)


@pytest.mark.gpu
def test_native_nccl_exchange_single_rank():
    """The in-library NCCL hook (gpm_exchange_nccl_*): communicator creation
    from a unique id, and ops 0/1/2 on device buffers at world 1 (the box has
    one GPU; the owner-based OR algorithm is covered at world 2/3 on gloo)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import ctypes as C
    import paper_1911_06969_b200 as P
    from paper_1911_06969_b200._lib import check, lib
    L = lib()
    uid = (C.c_char * 128)()
    check(L.gpm_nccl_unique_id(uid))
    ctx = C.c_void_p()
    check(L.gpm_exchange_nccl_create(bytes(uid), 0, 1, torch.cuda.current_device(), C.byref(ctx)))
    fn = L.gpm_exchange_nccl_fn()
    s = torch.cuda.current_stream()
    a = torch.arange(5, dtype=torch.int64, device="cuda")
    assert fn(ctx, a.data_ptr(), 5, 8, 0, s.cuda_stream) == 0
    b = torch.tensor([3, 5, 9], dtype=torch.int32, device="cuda")
    assert fn(ctx, b.data_ptr(), 3, 4, 1, s.cuda_stream) == 0
    c = torch.tensor([7, 8], dtype=torch.int64, device="cuda")
    assert fn(ctx, c.data_ptr(), 2, 8, 2, s.cuda_stream) == 0
    torch.cuda.synchronize()
    assert a.tolist() == list(range(5)) and b.tolist() == [3, 5, 9] and c.tolist() == [7, 8]
    assert fn(ctx, a.data_ptr(), 5, 8, 9, s.cuda_stream) != 0   # unknown op -> error code, no exception
    # mine() with the native hook bound (world 1)
    hg = P.generate_rmat(10, 8, 0.45, 0.15, 0.15, seed=3, n_labels=4, label_seed=7)
    g = P.Graph(hg)
    base = P.mine(g, "fsm", 3, 20)
    r = P.mine(g, "fsm", 3, 20, exchange=fn, exchange_ctx=ctx.value)
    assert r.patterns == base.patterns
    check(L.gpm_exchange_nccl_destroy(ctx))
