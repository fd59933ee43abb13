import numpy as np, torch, os, sys
sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
os.environ['SINN_HEAD'] = '0'
import datagen, oracle
import paper_2301_10622_b200 as sinn
from gpu_util import Pair, t_i64, t_i32, t_f32
cfg = datagen.CONFIGS["tiny"]
table = datagen.hash_table(cfg)
P = Pair(cfg, table)
N = 70_000
ip = np.arange(N + 1, dtype=np.int64); ix = np.zeros(N, np.int32); v = np.ones(N, np.float32); v[::1000] = 2.0
P.insert(ip, ix, v, np.arange(N, dtype=np.uint32))
qp = np.array([0, 1, 3], np.int64); qi = np.array([0, 0, 5], np.int32); qv = np.array([1.0, 1.0, -1.0], np.float32)
print("stage1...", flush=True)
ci, cs = P.gpu.search_stage1(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 200)
torch.cuda.synchronize(); print("stage1 ok", flush=True)
oi, os_ = P.gpu.search(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 10, 200, True)
torch.cuda.synchronize(); print("search ok", flush=True)
