"""Times the phases of the e2e path (pinned host CSR -> device -> orient -> mine)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1911_06969_b200 as P
app = sys.argv[1] if len(sys.argv) > 1 else "cf4"
W = {"cf4": ("cf", 4, (22, 3.35, .50, .20, .20)), "tc": ("tc", 3, (16, 16, .57, .19, .19))}
a, k, (sc, ef, pa, pb, pc) = W[app]
hg = P.generate_rmat(sc, ef, pa, pb, pc, 1)
off = torch.from_numpy(hg.off.view(np.int64)).pin_memory(); col = torch.from_numpy(hg.col.view(np.int32)).pin_memory()
ph = P.HostGraph(off.numpy().view(np.uint64), col.numpy().view(np.uint32))
def t(f):
    torch.cuda.synchronize(); s = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, 1e3 * (time.perf_counter() - s)
for it in range(4):
    g, t1 = t(lambda: P.Graph(ph))
    d, t2 = t(lambda: g.orient_dag())
    r, t3 = t(lambda: P.mine(d, a, k))
    _, t4 = t(lambda: (g.__del__(), d.__del__()))
    r2, t5 = t(lambda: P.mine(P.Graph(ph), a, k))
    gd, t6 = t(lambda: P.Graph(ph, orient=True))
    r3, t7 = t(lambda: P.mine(gd, a, k))
    del gd
    print(f"create {t1:.2f}  orient {t2:.2f}  mine {t3:.2f} (dev {r.stats['ms_total']:.2f})  free {t4:.2f} | e2e-one-call {t5:.2f} (dev {r2.stats['ms_total']:.2f}) | create_dag {t6:.2f} + mine {t7:.2f}")
