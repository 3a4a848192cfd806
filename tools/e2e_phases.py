"""Times the e2e path of bench.py (pinned host CSR -> fused upload + orient ->
mine -> free) phase by phase over many iterations, to locate outliers:
    python tools/e2e_phases.py [cf4|tc] [iters]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import gc
import numpy as np, torch
import paper_1911_06969_b200 as P
app = sys.argv[1] if len(sys.argv) > 1 else "cf4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 20
W = {"cf4": ("cf", 4, (22, 3.35, .50, .20, .20)), "tc": ("tc", 3, (16, 16, .57, .19, .19))}
a, k, (sc, ef, pa, pb, pc) = W[app]
hg = P.generate_rmat(sc, ef, pa, pb, pc, 1)
off = torch.from_numpy(hg.off.view(np.int64)).pin_memory(); col = torch.from_numpy(hg.col.view(np.int32)).pin_memory()
ph = P.HostGraph(off.numpy().view(np.uint64), col.numpy().view(np.uint32))
keep = []
if "--keep" in sys.argv:  # as bench.py: the device-resident graphs stay alive during the e2e steps
    gu = P.Graph(hg)
    gd = gu.orient_dag()
    for _ in range(8):
        P.mine(gd, a, k)
    keep = [gu, gd]
    torch.cuda.synchronize()
gc.disable()
for it in range(iters):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    g = P.Graph(ph, orient=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    r = P.mine(g, a, k)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    del g
    torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"create_dag {1e3*(t1-t0):7.2f}  mine {1e3*(t2-t1):7.2f} (dev {r.stats['ms_total']:.2f})  free {1e3*(t3-t2):6.2f}  total {1e3*(t3-t0):7.2f}", flush=True)
