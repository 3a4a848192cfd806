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


def test_gloo_exchange_and_partition(oracle):
    world = 2
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
        assert res[r]["sum"] == [3, 30]
        assert res[r]["or"] == [3, 0x300]
        assert res[r]["gather"] == [0, 100, 1, 101]
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
                t = torch.as_tensor(_DevArray(ptr, count, eb), device="cuda")
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


def _run_ranks(P, hg, app, k, sigma, world):
    ex = ThreadedExchange(world)
    out = [None] * world
    errs = []
    fns = [ex.fn(r) for r in range(world)]

    def run(r):
        try:
            g = P.Graph(hg)
            out[r] = P.mine(g, app, k, sigma, rank=r, world=world, exchange=fns[r])
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
