"""The document-sharded search protocol (paper_2301_10622_b200/sharded.py) over a real
process group on CPU: gloo, world_size 2.  The device ends of the exchange (stage 1, merge, owner
re-rank) are CUDA kernels, so here each rank's shard is backed by the ORACLE and the merges by numpy —
what is under test is the plumbing: row routing by id, the all-gather layout [W, nq, k], the
local <-> global id maps handed to the merge and the re-rank, and that every rank ends with the result
of one oracle holding all the documents."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

NO_ID = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _i32(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.uint32).view(np.int32)))


class OracleShard:
    """The Index methods ShardedIndex calls, answered by the oracle (CPU tensors, uint32 ids as int32)."""

    def __init__(self, cfg, table):
        import oracle
        self.o = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, cfg.upper_only)

    def insert_host(self, ip, ix, v, ids):
        assert self.o.insert(ip, ix, v, ids) == 0

    def delete_host(self, ids):
        assert self.o.delete(ids) == 0

    def search_stage1(self, qp, qi, qv, kprime):
        qp, qi, qv = qp.numpy(), qi.numpy(), qv.numpy()
        nq = qp.size - 1
        ci = np.full((nq, kprime), NO_ID, np.uint32)
        cs = np.full((nq, kprime), -np.inf, np.float32)
        for q in range(nq):
            s, _ = self.o.scores(qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]])
            live = np.nonzero(np.isfinite(s))[0]
            order = live[np.lexsort((live, -s[live]))][:kprime]
            ci[q, :order.size] = order
            cs[q, :order.size] = s[order]
        return _i32(ci), torch.from_numpy(cs)

    def rerank(self, qp, qi, qv, cand, k, mul, add):
        qp, qi, qv = qp.numpy(), qi.numpy(), qv.numpy()
        cand = cand.numpy().view(np.uint32)
        nq = qp.size - 1
        oi = np.full((nq, k), NO_ID, np.uint32)
        os_ = np.full((nq, k), -np.inf, np.float32)
        for q in range(nq):
            own = np.array([g for g in cand[q] if g != NO_ID and g % mul == add and self.o.is_live(int(g) // mul)],
                           np.int64)
            ex = np.array([self.o.exact_dot(int(g) // mul, qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]]) for g in own])
            order = np.lexsort((own, -ex))[:k]
            oi[q, :order.size] = own[order]
            os_[q, :order.size] = ex[order]
        return _i32(oi), torch.from_numpy(os_)


class NumpyOps:
    @staticmethod
    def merge_topk(ids, scores, kout, id_mul=1, id_add=None):
        ids, scores = ids.numpy().view(np.uint32), scores.numpy()
        parts, nq, kin = ids.shape
        add = np.zeros(parts, np.int64) if id_add is None else np.asarray(id_add, np.int64)
        oi = np.full((nq, kout), NO_ID, np.uint32)
        os_ = np.full((nq, kout), -np.inf, np.float32)
        for q in range(nq):
            keep = ids[:, q, :] != NO_ID
            g = (ids[:, q, :].astype(np.int64) * id_mul + add[:, None])[keep]
            s = scores[:, q, :][keep]
            order = np.lexsort((g, -s.astype(np.float64)))[:kout]
            oi[q, :order.size] = g[order]
            os_[q, :order.size] = s[order]
        return _i32(oi), torch.from_numpy(os_)


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import datagen
    from paper_2301_10622_b200.sharded import ShardedIndex
    cfg = datagen.CONFIGS["tiny"]
    table = datagen.hash_table(cfg)
    sh = ShardedIndex(OracleShard(cfg, table), ops=NumpyOps())   # rank / world from the process group
    assert (sh.rank, sh.world) == (rank, ws)
    N = 1201
    ip, ix, v = datagen.docs(cfg, 0, N)
    ids = np.arange(N, dtype=np.uint32)[::-1].copy()              # global ids in descending row order
    took = sh.insert_host(ip, ix, v, ids)
    dead = np.array([5, 6, 7, 1200], np.uint32)
    took -= sh.delete_host(dead)
    qp, qi, qv = datagen.queries(cfg, 0, 12)
    q = (torch.from_numpy(qp), torch.from_numpy(qi), torch.from_numpy(qv))
    fi, fs = sh.search(*q, 10, 100, rerank=True)
    ai, as_ = sh.search(*q, 10, 100, rerank=False)
    out[rank] = (took, fi.numpy().view(np.uint32).copy(), fs.numpy().copy(), ai.numpy().view(np.uint32).copy(),
                 as_.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_search_equals_one_oracle_index():
    import datagen
    import oracle
    ws, port = 2, _free_port()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    cfg = datagen.CONFIGS["tiny"]
    N = 1201
    O = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, datagen.hash_table(cfg), cfg.upper_only)
    ip, ix, v = datagen.docs(cfg, 0, N)
    assert O.insert(ip, ix, v, np.arange(N, dtype=np.uint32)[::-1].copy()) == 0
    assert O.delete(np.array([5, 6, 7, 1200], np.uint32)) == 0
    qp, qi, qv = datagen.queries(cfg, 0, 12)
    wi, wsc = O.search(qp, qi, qv, 10, 100, True)
    ai, asc = O.search(qp, qi, qv, 10, 100, False)
    assert out[0][0] + out[1][0] == N - 4                         # every live row on exactly one shard
    assert abs(out[0][0] - out[1][0]) <= 4                        # id % W balances the shards
    for r in range(ws):
        _, fi, fs, gi, gs = out[r]
        np.testing.assert_array_equal(fi, wi)                     # same ids, same order, on every rank
        np.testing.assert_allclose(fs, wsc, rtol=1e-6, atol=0)
        np.testing.assert_array_equal(gi, ai)
        np.testing.assert_allclose(gs, asc, rtol=1e-6, atol=0)


def test_route_rows_host_partitions_a_batch():
    from paper_2301_10622_b200.sharded import owner, route_rows_host
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 9, 50)
    ip = np.concatenate([[7], 7 + np.cumsum(lens)]).astype(np.int64)      # an indptr that does not start at 0
    ix = rng.integers(0, 100, ip[-1]).astype(np.int32)
    v = rng.standard_normal(ip[-1]).astype(np.float32)
    ids = rng.choice(1000, 50, replace=False).astype(np.uint32)
    seen = 0
    for r in range(3):
        p, jx, w, lid = route_rows_host(ip, ix, v, ids, 3, r)
        rows = np.nonzero(owner(ids, 3) == r)[0]
        assert p[0] == 0 and lid.size == rows.size and p.size == rows.size + 1
        np.testing.assert_array_equal(lid, ids[rows] // 3)
        for t, row in enumerate(rows):
            np.testing.assert_array_equal(jx[p[t]:p[t + 1]], ix[ip[row]:ip[row + 1]])
            np.testing.assert_array_equal(w[p[t]:p[t + 1]], v[ip[row]:ip[row + 1]])
        seen += rows.size
    assert seen == 50
