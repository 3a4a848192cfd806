#!/usr/bin/env python
"""bench.py — embeddings explored/s for the Pangolin E-R-F hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--app cf4|tc|mc3|mc4|fsm] [--impl ours|reference]

Headline workload (BASELINE.json configs[1]): 4-clique listing on the
Patent-like synthetic RMAT (scale 22, edge factor 3.35, (a,b,c)=(.50,.20,.20),
seed 1), degree-ordered DAG.  A step = one complete mine() of that workload.

* value  = N_explored (summed over ranks) / device time per step, the DAG CSR
           resident in HBM, L2 flushed between steps (256 MiB write).
* e2e    = the same metric through the public C ABI from pinned HOST buffers:
           every step uploads the undirected CSR, orients it on the device,
           mines, and reads the result back.
* roofline = bytes the dominant extend kernel reads (SURVEY §8d B_alg, or the
           streamed + staged bytes of the staged MC kernels) / its
           CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
* cpu_baseline = the C++/OpenMP oracle (oracle/liboracle.so) on this host,
           engine time only, on the oracle's own generator restatement.
* workloads = sub-records (value, e2e, roofline, parity vs the full-size
           goldens) of the other BASELINE configs: tc, mc3, mc4, fsm.
* --impl reference = the oracle port on every host thread (never imports
           paper_1911_06969_b200); same config keys as this arm.
Multi-GPU (torchrun): root units split by degree weight, counts all-reduced
over NCCL; time is the max over ranks.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (app, k, sigma, rmat args, description)
    "cf4": ("cf", 4, 0, dict(scale=22, edge_factor=3.35, a=0.50, b=0.20, c=0.20, seed=1),
            "4-CL on Patent-like RMAT-22 ef3.35 (.50,.20,.20) seed 1, degree-ordered DAG"),
    "tc": ("tc", 3, 0, dict(scale=16, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1),
           "TC on RMAT-16 ef16 (.57,.19,.19) seed 1, degree-ordered DAG"),
    "mc3": ("mc", 3, 0, dict(scale=22, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1),
            "3-MC on LiveJournal-sized RMAT-22 ef16 (.57,.19,.19) seed 1"),
    "mc4": ("mc", 4, 0, dict(scale=22, edge_factor=8.6, a=0.45, b=0.15, c=0.15, seed=1),
            "4-MC on power-law RMAT-22 ef8.6 (.45,.15,.15) seed 1"),
    "fsm": ("fsm", 4, 300, dict(scale=17, edge_factor=11, a=0.45, b=0.15, c=0.15, seed=1, n_labels=32,
                                 label_seed=101),
            "3-edge FSM on Mico-like RMAT-17 ef11 (.45,.15,.15) 32 labels"),
}
METRIC = "embeddings explored/sec (N_explored = |L1| + accepted per extend level)"
UNIT = "embeddings/s"


L2_RESIDENT = ("cf4", "tc", "fsm")
_L2_PEAK = []


def l2_read_peak():
    """L2 read GB/s, measured once per process on cuda:0 (64 MiB working set)."""
    if not _L2_PEAK:
        import torch
        import paper_1911_06969_b200 as P
        _L2_PEAK.append(P.probe_read_bandwidth(64 << 20, torch.cuda.current_device(), 10))
    return _L2_PEAK[0]


def load_peaks():
    for p in (os.path.join(ROOT, "MEASURED_PEAKS.json"),):
        if os.path.exists(p):
            with open(p) as f:
                d = json.load(f)
            return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons DURING the timed region (B200_PROFILING.md)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index, period_ms="100"):
        self.index = index
        self.period_ms = str(period_ms)
        self.proc = None
        self.lines = []

    # No reader thread: a Python thread waking for every sample competes for
    # the GIL with the host side of the timed steps (ctypes calls reacquire it
    # on return).  Samples queue in the pipe (~100 B each, 64 KiB buffer ≈ a
    # minute of samples) and are drained here, outside the timed steps.
    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", self.period_ms],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def drain(self, block_s=0.0):
        """Reads the samples already queued (waits up to block_s for one)."""
        if not self.proc:
            return
        import select
        t_end = time.time() + block_s
        while True:
            r, _, _ = select.select([self.proc.stdout], [], [], max(0.0, t_end - time.time()))
            if not r:
                return
            line = self.proc.stdout.readline()
            if not line:
                return
            self.lines.append(line.strip())
            t_end = time.time()  # got one: only take what is already queued

    def wait_samples(self, n, timeout=5.0):
        """Blocks until n samples have arrived (the sampler's first lines lag
        its start; short timed regions would otherwise see none)."""
        t = time.time()
        while self.proc and len(self.lines) < n and time.time() - t < timeout:
            self.drain(0.2)

    def stop(self, first=0):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.drain()
        self.proc.terminate()
        try:
            rest, _ = self.proc.communicate(timeout=5)
            self.lines += [ln.strip() for ln in (rest or "").splitlines() if ln.strip()]
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines[first:]:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def _oracle():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    return pyoracle


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_graph(name):
    """The workload's graph from the oracle's own generator restatement (the
    reference arm and the CPU baseline never load libgpm.so); TC/CF graphs
    are oriented here, outside every timed region, as on the GPU path."""
    O = _oracle()
    app, k, sigma, rmat, _ = WORKLOADS[name]
    g = O.generate_rmat(rmat["scale"], rmat["edge_factor"], rmat["a"], rmat["b"], rmat["c"], rmat["seed"],
                        rmat.get("n_labels", 0), rmat.get("label_seed", 101))
    gin = O.orient_dag(g) if app in ("tc", "cf") else g
    return g, gin


def cpu_sample(gin, app, k, sigma, budget_s, threads):
    """Chooses a bounded sample of the workload for the CPU oracle: a contiguous
    prefix of level-1 root units grown x4 until it costs >= budget_s/4 (or is
    the whole workload).  Returns (root_hi or None for all, description)."""
    O = _oracle()
    probe = 1 << 14
    while True:
        r = O.mine(gin, app, k, sigma, threads=threads, root_lo=0, root_hi=probe)
        if r["level_sizes"][0] < probe:
            return None, "full workload"
        if r["ms"] / 1e3 >= budget_s / 4:
            return probe, f"first {probe} level-1 root units (contiguous prefix)"
        probe *= 4


def cpu_run(gin, app, k, sigma, root_hi, threads):
    """One oracle mine; its "ms" covers the engine only (CSR copy and, for
    TC/CF, orientation excluded, like the GPU value)."""
    O = _oracle()
    return O.mine(gin, app, k, sigma, threads=threads, root_lo=0, root_hi=root_hi if root_hi else 2**64 - 1)


def workload_config(name, n, m, sigma):
    """`config` of a bench line: identical in both arms for the same workload."""
    app, k, _, _, desc = WORKLOADS[name]
    cfg = {"workload": desc, "app": app, "k": k, "n": n, "m_half_edges": m,
           "generator": "SURVEY §8d RMAT (splitmix64 quadrant draws, seeded permutation, load_edge_list cleaning)",
           "l2": "flushed between timed steps (256 MiB device write, outside the step events)"}
    if app == "fsm":
        cfg["min_support"] = sigma
    return cfg


def golden_parity(name, sigma, result):
    """Compares a run with tests/golden/configs.json (oracle numbers at full
    size, tests/golden/make_config_goldens.py); None when no golden exists."""
    gp = os.path.join(ROOT, "tests", "golden", "configs.json")
    key = {"cf4": "pat_cf4", "tc": "tc16", "mc3": "lj22_mc3", "mc4": "mc4_mc4"}.get(name)
    if name == "fsm":
        key = f"fsm17_s{sigma}"
    if not key or not os.path.exists(gp):
        return None
    with open(gp) as f:
        gold = json.load(f).get(key)
    if not gold:
        return None
    out = {"golden": f"tests/golden/configs.json[{key}]", "source": gold.get("source")}
    checks = {"n_explored": result["n_explored"] == gold["n_explored"],
              "level_sizes": list(result["level_sizes"]) == list(gold["level_sizes"])}
    if "total" in gold:
        checks["total"] = result["total"] == gold["total"]
        out["oracle_total"] = gold["total"]
    if "patterns_digest" in gold:
        checks["patterns_sha256"] = result.get("patterns_sha256") == gold["patterns_digest"]["sha256"]
    elif "patterns" in gold:
        checks["patterns"] = sorted((int(a), str(b), int(c)) for a, b, c in result["patterns"]) == \
            sorted((int(a), str(b), int(c)) for a, b, c in gold["patterns"])
    out["checks"] = checks
    out["match"] = all(checks.values())
    return out


def reference_arm(args, names):
    """`--impl reference`: the reference's CPU path = the oracle port
    (oracle/liboracle.so) on every host thread; the reference itself has no
    engine code.  Never imports paper_1911_06969_b200."""
    threads = os.cpu_count() or 1
    line = None
    subs = {}
    for i, name in enumerate(names):
        app, k, sigma, _, _ = WORKLOADS[name]
        if i == 0 and args.sigma is not None:
            sigma = args.sigma
        g, gin = oracle_graph(name)
        budget = args.cpu_budget if i == 0 else args.cpu_budget / 4
        steps, warm = (args.steps, args.warmup) if i == 0 else (2, 1)
        root_hi, sample = cpu_sample(gin, app, k, sigma, budget, threads)
        times, r = [], None
        for j in range(warm + steps):
            r = cpu_run(gin, app, k, sigma, root_hi, threads)
            if j >= warm:
                times.append(r["ms"])
        ms = sum(times) / len(times)
        v = r["n_explored"] / (ms / 1e3)
        cb = {"value": v, "unit": UNIT, "cores": threads, "cpu": cpu_model(), "kind": "port",
              "sample": sample + "; oracle/liboracle.so (C++/OpenMP restatement of SPEC.md engine), "
                                 "engine time only (graph orientation outside, as in the GPU value)"}
        rec = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
               "steps": steps, "warmup": warm, "ms_per_step": ms, "higher_is_better": True,
               "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
               "config": workload_config(name, g.n, g.m, sigma), "cpu_baseline": cb,
               "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
               "result": {"total": r.get("total"), "n_explored": r["n_explored"]}}
        if i == 0:
            line = rec
        else:
            subs[name] = {k_: rec[k_] for k_ in ("value", "ms_per_step", "config", "cpu_baseline", "result")}
    if subs:
        line["workloads"] = subs
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--app", default="cf4", choices=sorted(WORKLOADS))
    ap.add_argument("--sigma", type=int, default=None)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU oracle work for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true",
                    help="headline workload only (default: the cf4 line also carries tc/mc3/mc4/fsm sub-records)")
    ap.add_argument("--no-steal", action="store_true", help="N>1: static split only (no work-stealing tail)")
    args = ap.parse_args()
    rank, world, local = dist_env()
    names = [args.app]
    if args.app == "cf4" and not args.no_sub and args.sigma is None:
        names += ["tc", "mc3", "mc4", "fsm"]

    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, names)
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_1911_06969_b200 as P
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    # N > 1: the in-library NCCL exchange (no Python on the exchange path);
    # the torch.distributed callback only if the native one cannot start
    exchange, exchange_ctx, native_ex, exchange_kind = None, 0, None, "none (single rank)"
    if world > 1:
        try:
            from paper_1911_06969_b200.dist import NativeExchange
            native_ex = NativeExchange()
            exchange, exchange_ctx, exchange_kind = native_ex.fn, native_ex.ctx, "libgpm NCCL (owner-based OR)"
        except Exception as e:
            print(f"[bench] native NCCL exchange unavailable ({e!r}); torch.distributed callback", file=sys.stderr)
            from paper_1911_06969_b200.dist import make_exchange
            exchange, exchange_kind = make_exchange(), "torch.distributed callback"
    # a dedicated (non-default) stream: the engine launches every kernel on it
    # and the step events are recorded on it, so they bracket the device work
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # N > 1: degree-weighted static split + device-side work-stealing tail
    # over counters peer-mapped from rank 0's GPU (FSM levels exchange anyway)
    steal = None
    if world > 1 and not args.no_steal:
        try:
            from paper_1911_06969_b200.dist import StealCounters
            steal = StealCounters()
        except Exception as e:  # static split only
            print(f"[bench] work stealing disabled: {e!r}", file=sys.stderr)
            steal = None

    def run_workload(name, steps, warmup, cpu_budget, headline):
        app, k, sigma, rmat, desc = WORKLOADS[name]
        if headline and args.sigma is not None:
            sigma = args.sigma
        use_steal = steal if app != "fsm" else None
        t0 = time.time()
        hg = P.generate_rmat(rmat["scale"], rmat["edge_factor"], rmat["a"], rmat["b"], rmat["c"], rmat["seed"],
                             rmat.get("n_labels", 0), rmat.get("label_seed", 101))
        gen_s = time.time() - t0
        config = workload_config(name, hg.n, hg.m, sigma)
        partition = ("degree-weighted static split" + (" + device work-stealing tail" if use_steal else "")
                     if world > 1 else "single rank")

        # ---------------- device-resident path (value)
        g_und = P.Graph(hg, device=local)
        g_in = g_und.orient_dag() if app in ("tc", "cf") else g_und   # preprocessing
        kw = dict(rank=rank, world=world, stream=sp, exchange=exchange, exchange_ctx=exchange_ctx)

        def mine_step():
            skw = {}
            if use_steal is not None:
                use_steal.reset()
                skw = dict(steal_ctrs=use_steal.ptr)
            return P.mine(g_in, app, k, sigma, **kw, **skw)

        res = None
        # the sampler starts (and delivers its first line) BEFORE the warm-up, so
        # the GPU goes straight from the warm-up steps into the timed ones instead
        # of idling (and dropping clocks) while nvidia-smi comes up
        clocks = ClockSampler(local, os.environ.get("GPM_BENCH_CLOCK_MS", "100"))
        clocks.start()
        clocks.wait_samples(1)
        # collect before the warm-up, not between it and the timed steps (an
        # idle GPU during a collection made the first timed step the slowest)
        gc.collect()
        gc.disable()  # no collector pauses inside the timed host calls (re-enabled after the e2e steps)
        for _ in range(warmup):  # the same as a timed step (L2 flush + step), untimed
            flush.zero_()
            res = mine_step()
        barrier()
        clocks.drain()
        n_before = len(clocks.lines)
        step_ms = []
        dom_ms, dom_b, dom_mv, launches = [], [], [], 0
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        barrier()
        for _ in range(steps):
            flush.zero_()
            if use_steal is not None:
                use_steal.reset()
            ev0.record(stream)
            res = P.mine(g_in, app, k, sigma, **kw, **({"steal_ctrs": use_steal.ptr} if use_steal else {}))
            ev1.record(stream)
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            dom_ms.append(res.stats["ms_dominant"])
            dom_b.append(res.stats["b_dominant"])
            dom_mv.append(res.stats["b_moved_dominant"])
            launches += res.stats["launches"]
        barrier()
        # a short timed region may fall between two 100 ms samples: keep the GPU
        # busy with further (untimed) steps until one sample lands after it began
        t_extra = time.time()
        clocks.drain()
        while len(clocks.lines) <= n_before + 1 and time.time() - t_extra < 3.0:
            mine_step()
            torch.cuda.synchronize()
            clocks.drain()
        clock_rec = clocks.stop(first=n_before)
        tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        ms_per_step = tot.item() / steps
        n_explored = res.stats["n_explored"]   # already summed over ranks by the engine's exchange
        value = n_explored / (ms_per_step / 1e3)

        # ---------------- end-to-end through the public C ABI from pinned host buffers
        off_p = torch.from_numpy(np.ascontiguousarray(hg.off, dtype=np.uint64).view(np.int64)).pin_memory()
        col_p = torch.from_numpy(np.ascontiguousarray(hg.col, dtype=np.uint32).view(np.int32)).pin_memory()
        lab_p = (torch.from_numpy(np.ascontiguousarray(hg.labels, dtype=np.uint32).view(np.int32)).pin_memory()
                 if hg.labels is not None else None)
        pinned = P.HostGraph(off_p.numpy().view(np.uint64), col_p.numpy().view(np.uint32),
                             None if lab_p is None else lab_p.numpy().view(np.uint32))
        h2d = pinned.off.nbytes + pinned.col.nbytes + (0 if lab_p is None else pinned.labels.nbytes)
        e2e_ms = []
        er = None
        ew = max(1, warmup)  # untimed e2e warm-up calls (first-touch of pinned pages, caches)
        for i in range(ew + steps):
            if use_steal is not None:
                use_steal.reset()
            barrier()
            t = time.perf_counter()
            # TC/CF need the degree-ordered DAG: fused pipelined upload + orientation
            g = P.Graph(pinned, device=local, orient=app in ("tc", "cf"))
            er = P.mine(g, app, k, sigma, rank=rank, world=world, exchange=exchange, exchange_ctx=exchange_ctx,
                        **({"steal_ctrs": use_steal.ptr} if use_steal else {}))
            del g
            torch.cuda.synchronize()
            if i >= ew:
                e2e_ms.append(1e3 * (time.perf_counter() - t))
        gc.enable()
        et = torch.tensor([sum(e2e_ms)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_ms_step = et.item() / steps
        assert er.stats["n_explored"] == n_explored and er.total == res.total, "e2e result differs from device path"
        d2h = 8 + 8 * len(er.patterns) + 8 * 16 * 3

        peak, peak_kind = load_peaks()
        dms = statistics.median(dom_ms)
        b_alg = statistics.median(dom_b)
        b_mv = statistics.median(dom_mv)
        achieved = (b_mv / (dms / 1e3) / 1e9) if dms > 0 else 0.0
        traffic = l2_bytes = None
        tp = os.path.join(ROOT, "profiles", f"traffic_{name}.json")
        # the ncu capture is of the workload's default configuration only
        if os.path.exists(tp) and sigma == WORKLOADS[name][2]:
            with open(tp) as f:
                tj = json.load(f)
            traffic = tj.get("dram_bytes_per_launch")
            l2_bytes = tj.get("l2_bytes_per_launch") or None
        # measured traffic of one ncu-captured launch over this run's live kernel time:
        # the DRAM rate, and the L2 rate SURVEY §8d asks for on the L2-resident configs
        mem_rates = {}
        if dms > 0:
            mem_rates["b_alg_survey"] = b_alg
            mem_rates["b_alg_survey_gbs"] = b_alg / (dms / 1e3) / 1e9
            if traffic:
                mem_rates["dram_gbs"] = traffic / (dms / 1e3) / 1e9
                mem_rates["dram_frac"] = mem_rates["dram_gbs"] / peak
            if l2_bytes:
                mem_rates["l2_bytes_per_launch"] = l2_bytes
                mem_rates["l2_gbs"] = l2_bytes / (dms / 1e3) / 1e9
        # L2-resident CSRs (the PAT DAG is 76 MB, TC16 / FSM17 smaller; L2 is
        # 126 MB): their kernels stream the CSR from L2, so the L2 read rate is
        # the roofline that bounds them (measured, stated)
        if name in L2_RESIDENT and dms > 0:
            l2_peak = l2_read_peak()
            mem_rates["l2"] = {"achieved_gbs": achieved, "peak_gbs": l2_peak, "frac": achieved / l2_peak,
                               "peak_kind": ("builder-measured in this run: gpm_probe_read_bandwidth over a 64 MiB "
                                             "device buffer (16-byte __ldcg loads, persistent grid, best of 10)")}
        pats = res.patterns
        result = {"total": res.total, "n_explored": n_explored, "level_sizes": res.stats["level_sizes"],
                  "candidates": res.stats["candidates"], "patterns": len(pats),
                  "n_counted": res.stats["n_counted"]}
        pres = dict(result, patterns=pats)
        if app == "fsm":
            import hashlib
            rows = sorted((int(l), str(t), int(s_)) for l, t, s_ in pats)
            pres["patterns_sha256"] = hashlib.sha256(
                "".join(f"{l}\t{t}\t{s_}\n" for l, t, s_ in rows).encode()).hexdigest()
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": config, "partition": partition, "exchange": exchange_kind,
            "e2e": {"value": n_explored / (e2e_ms_step / 1e3), "unit": UNIT, "ms_per_step": e2e_ms_step,
                    "step_ms": [round(x, 3) for x in e2e_ms],
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": res.stats["dominant"],
                         "kernel_ms": dms, "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs)",
                         "bytes": ("bytes the dominant kernel reads per launch (b_moved): SURVEY §8d B_alg "
                                   "(8*l per parent + (16 + 4*deg) per extended position) except for the "
                                   "staged MC kernels, whose reads are the streamed suffixes + staged sets "
                                   "(DESIGN.md §5); b_alg_survey keeps the per-candidate figure"),
                         "note": ("traffic = ncu dram bytes of one captured launch "
                                  "(profiles/traffic_<app>.json); L2-resident CSRs (cf4, tc, fsm) are "
                                  "re-read from L2, so their b_moved/t can exceed the HBM rate"),
                         **mem_rates},
            "step_ms": [round(x, 4) for x in step_ms],
            # SURVEY §8d asks for best and median as well as the mean (`ms_per_step`)
            "step_stats": {"best_ms": min(step_ms), "median_ms": statistics.median(step_ms),
                           "e2e_best_ms": min(e2e_ms), "e2e_median_ms": statistics.median(e2e_ms)},
            "gpu_launches": launches,
            "clocks": clock_rec,
            "result": result,
            "parity": golden_parity(name, sigma, pres),
            "gen_s": round(gen_s, 2),
        }
        del g_in, g_und
        if rank == 0 and world == 1 and not args.no_cpu_baseline:
            threads = os.cpu_count() or 1
            _, gin = oracle_graph(name)
            root_hi, sample = cpu_sample(gin, app, k, sigma, cpu_budget, threads)
            r = cpu_run(gin, app, k, sigma, root_hi, threads)
            out["cpu_baseline"] = {"value": r["n_explored"] / (r["ms"] / 1e3), "unit": UNIT, "cores": threads,
                                   "cpu": cpu_model(), "kind": "port",
                                   "sample": sample + " (oracle/liboracle.so, OpenMP; engine time only)"}
        return out

    line = run_workload(names[0], args.steps, args.warmup, args.cpu_budget, True)
    subs = {}
    for name in names[1:]:
        sub = run_workload(name, args.steps, args.warmup, args.cpu_budget / 4, False)
        subs[name] = {k_: sub[k_] for k_ in ("value", "ms_per_step", "config", "e2e", "roofline", "step_stats",
                                              "gpu_launches", "clocks", "result", "parity", "cpu_baseline")
                      if k_ in sub}
        line["gpu_launches"] += sub["gpu_launches"]
    if subs:
        line["workloads"] = subs
        line["gpu_launches_note"] = "gpu_launches sums the headline and the sub-record workloads"
    if rank == 0:
        print(json.dumps(line))
    if steal is not None:
        steal.close()
    if native_ex is not None:
        native_ex.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
