import sys, time, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import paper_1911_06969_b200 as P
for sc, s in ((14, 100), (15, 100), (16, 100), (17, 1000), (17, 300)):
    hg = P.generate_rmat(sc, 11, .45, .15, .15, seed=1, n_labels=32, label_seed=101)
    g = P.Graph(hg)
    t = time.time()
    r = P.mine(g, 'fsm', 4, s)
    print(sc, s, time.time() - t, r.stats['level_sizes'], r.stats['survivors'], len(r.patterns), r.stats['dominant'], r.stats['ms_dominant'], flush=True)
