import sys, os
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import numpy as np, torch, datagen, oracle
from gpu_util import Pair, t_i64, t_i32, t_f32, ids_np
cfg = datagen.CONFIGS["c3s"]
P = Pair(cfg)
for s in range(0, cfg.N, cfg.insert_batch):
    c = min(cfg.insert_batch, cfg.N - s)
    ip, ix, v = datagen.docs(cfg, s, c)
    P.insert(ip, ix, v, np.arange(s, s + c, dtype=np.uint32))
qp, qi, qv = datagen.queries(cfg, 0, cfg.nq)
ci, cs = P.gpu.search_stage1(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.kprime)
ci, cs = ids_np(ci), cs.cpu().numpy()
for q in range(qp.size - 1):
    g = ci[q][ci[q] != oracle.NO_ID]
    u, cnt = np.unique(g, return_counts=True)
    bad = g[g >= cfg.N]
    if u.size != g.size or bad.size:
        print("q", q, "n", g.size, "unique", u.size, "dups", u[cnt > 1][:5], "bad", bad[:5], "scores", cs[q][:3], cs[q][g.size-3:g.size])
print("done")
