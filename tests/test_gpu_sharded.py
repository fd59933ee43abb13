"""Document sharding on ONE GPU: W shard indexes of one process are driven
through the protocol phase by phase (`sharded.search_lockstep`: a stack of the per-shard outputs stands
in for the all-gather, so no rank ever waits on another) and compared with the oracle holding ALL the
documents under their global ids — the sharded search must reproduce the single-index search.
Plus unit parity of the two device ends of the exchange: sinn_merge_topk vs a numpy FindLargest, and
sinn_rerank vs the oracle's exact dots."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device (no fallback path exists)"
    import paper_2301_10622_b200 as sinn
    sinn.lib()


from gpu_util import Pair, check_final, check_stage1, ids_np, t_f32, t_i32, t_i64  # noqa: E402


class ShardedFacade:
    """W shards behind the Index methods the parity checks call (global ids in and out)."""

    def __init__(self, cfg, table, W, peer=False):
        import paper_2301_10622_b200 as sinn
        from paper_2301_10622_b200.sharded import ShardedIndex
        self.W = W
        self.peer = peer   # stage-1 rows stored by the select kernels into every shard's buffer
        self._peers = {}
        self.shards = [ShardedIndex(sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only), rank=r, world=W)
                       for r in range(W)]

    def _set_peers(self, nq, kprime):
        if not self.peer:
            return
        from paper_2301_10622_b200.sharded import PeerGather
        key = (nq, kprime)
        if key not in self._peers:
            self._peers[key] = PeerGather.local(self.W, nq, kprime, "cuda")
        for s, pg in zip(self.shards, self._peers[key]):
            s.peer = pg

    def insert_host(self, ip, ix, v, ids):
        took = [s.insert_host(ip, ix, v, ids) for s in self.shards]
        assert sum(took) == len(ids)

    def delete_host(self, ids):
        assert sum(s.delete_host(ids) for s in self.shards) == len(ids)

    def _agree(self, outs):
        for oi, os_ in outs[1:]:
            assert torch.equal(oi, outs[0][0]) and torch.equal(os_, outs[0][1]), "shards disagree"
        return outs[0]

    def search_stage1(self, qp, qi, qv, kprime):
        q = (qp, qi, qv)
        self._set_peers(qp.numel() - 1, kprime)
        if self.peer:
            own = [s.phase_stage1_gather(q, kprime) for s in self.shards]
            for gi, gs in own[1:]:      # every shard's buffer holds the same gathered lists
                assert torch.equal(gi, own[0][0]) and torch.equal(gs, own[0][1])
            gi, gs = own[0]
        else:
            s1 = [s.phase_stage1(q, kprime) for s in self.shards]
            gi, gs = torch.stack([a for a, _ in s1]), torch.stack([b for _, b in s1])
        return self._agree([s.phase_select(gi, gs, kprime) for s in self.shards])

    def search(self, qp, qi, qv, k, kprime, rerank=True):
        from paper_2301_10622_b200.sharded import search_lockstep
        self._set_peers(qp.numel() - 1, kprime)
        return self._agree(search_lockstep(self.shards, (qp, qi, qv), k, kprime, rerank))

    def live(self):
        return sum(s.index.stats()["live"] for s in self.shards)


def sharded_pair(name, N, W, batch, peer=False):
    """A Pair whose .gpu is the W-shard facade and whose oracle holds every document (global ids)."""
    cfg = datagen.CONFIGS[name]
    P = Pair(cfg)
    P.single = P.gpu
    P.gpu = ShardedFacade(cfg, P.table, W, peer)
    for s in range(0, N, batch):
        c = min(batch, N - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        ids = np.arange(s, s + c, dtype=np.uint32)
        assert P.orc.insert(ip, ix, v, ids) == oracle.OK
        P.gpu.insert_host(ip, ix, v, ids)
        P.single.insert_host(ip, ix, v, ids)
        for r, i in enumerate(ids):
            P.rows[int(i)] = (ix[ip[r]:ip[r + 1]].copy(), v[ip[r]:ip[r + 1]].copy())
    return P


@pytest.mark.parametrize("name,N,W,batch", [("tiny", 5000, 3, 1700), ("c2s", 6000, 2, 2500), ("c5s", 5000, 4, 5000)])
def test_sharded_search_matches_the_single_index_oracle(name, N, W, batch):
    cfg = datagen.CONFIGS[name]
    P = sharded_pair(name, N, W, batch)
    assert P.gpu.live() == N
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 48))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=False)
    # and against the unsharded GPU index: the exact re-rank scores of common ids are bit-identical
    # (the same k_rerank on the same stored rows), the id sets differ at most at tolerance ties
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    si, ss = P.single.search(*tq, cfg.k, cfg.kprime, True)
    gi, gs = P.gpu.search(*tq, cfg.k, cfg.kprime, True)
    si, ss, gi, gs = ids_np(si), ss.cpu().numpy(), ids_np(gi), gs.cpu().numpy()
    same = 0
    for q in range(qp.size - 1):
        a = dict(zip(si[q].tolist(), ss[q].tolist()))
        b = dict(zip(gi[q].tolist(), gs[q].tolist()))
        for i in set(a) & set(b):
            assert a[i] == b[i]
        same += len(set(a) & set(b))
    assert same >= 0.98 * si.size


@pytest.mark.parametrize("dense", [False, True])
def test_select_kernels_store_the_gather_buffers(dense, monkeypatch):
    """sinn_search_stage1_gather: every shard's select kernel (k_cand_select, and k_sel_sort on the dense
    path) stores its rows into slot r of ALL W gather buffers — the all-gather by peer stores; the buffers
    must equal the stack of the plain stage-1 outputs, and the sharded search through them the oracle."""
    cfg = datagen.CONFIGS["c2s"]
    P = sharded_pair("c2s", 5000, 3, 5000, peer=True)
    if dense:
        monkeypatch.setenv("SINN_FORCE_DENSE", "1")
    qp, qi, qv = datagen.queries(cfg, 0, 24)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    P.gpu._set_peers(24, cfg.kprime)
    own = [s.phase_stage1_gather(tq, cfg.kprime) for s in P.gpu.shards]
    plain = [s.phase_stage1(tq, cfg.kprime) for s in P.gpu.shards]
    for gi, gs in own[1:]:        # one run, W destinations: identical buffers
        assert torch.equal(gi, own[0][0]) and torch.equal(gs, own[0][1])
    # against a second, plain run (fp32 summation order may differ between runs: DESIGN.md R7)
    pi, ps = torch.stack([a for a, _ in plain]), torch.stack([b for _, b in plain])
    assert (own[0][0] == pi).float().mean().item() > 0.99
    fin = torch.isfinite(ps)
    assert torch.equal(fin, torch.isfinite(own[0][1]))
    torch.testing.assert_close(own[0][1][fin], ps[fin], rtol=1e-4, atol=1e-4)
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=False)
    # both buffer sets were used in turn; a second batch does not disturb the first's result
    a = P.gpu.search(*tq, cfg.k, cfg.kprime)
    b = P.gpu.search(*tq, cfg.k, cfg.kprime)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])
    import paper_2301_10622_b200 as sinn
    G = P.gpu.shards[0].index
    bad = [torch.zeros((2, 24, cfg.kprime), dtype=torch.int32, device="cuda")] * 3
    with pytest.raises(ValueError):
        G.search_stage1_gather(*tq, cfg.kprime, 0, bad, bad)
    nine = [torch.zeros((9, 24, 8), dtype=torch.int32, device="cuda")] * 9
    ninef = [torch.zeros((9, 24, 8), dtype=torch.float32, device="cuda")] * 9
    with pytest.raises(sinn.SinnError) as e:
        G.search_stage1_gather(*tq, 8, 0, nine, ninef)       # more than 8 destinations
    assert e.value.status == sinn.EINVAL


def test_sharded_deletes_and_small_shards():
    """Deletes routed to their owners; k' larger than a shard's (and the whole index's) live count."""
    cfg = datagen.CONFIGS["tiny"]
    P = sharded_pair("tiny", 150, 4, 150)
    dead = np.array([0, 1, 2, 3, 8, 21, 149], dtype=np.uint32)
    assert P.orc.delete(dead) == oracle.OK
    P.gpu.delete_host(dead)
    for i in dead:
        del P.rows[int(i)]
    qp, qi, qv = datagen.queries(cfg, 0, 20)
    ci, _ = check_stage1(P, qp, qi, qv, 100)          # 100 > ~36 live per shard
    assert not set(ci.ravel().tolist()) & set(dead.tolist())
    check_final(P, qp, qi, qv, 10, 100)
    ci, _ = check_stage1(P, qp, qi, qv, 200)          # 200 > 143 live in total: V = every live id
    assert all(np.count_nonzero(ci[q] != oracle.NO_ID) == 143 for q in range(20))
    check_final(P, qp, qi, qv, 10, 200)


def np_merge(ids, scores, kout, mul, add):
    parts, nq, kin = ids.shape
    oi = np.full((nq, kout), oracle.NO_ID, np.uint32)
    os_ = np.full((nq, kout), -np.inf, np.float32)
    for q in range(nq):
        g, s = [], []
        for p in range(parts):
            for r in range(kin):
                if ids[p, q, r] != oracle.NO_ID:
                    gid = int(ids[p, q, r]) * mul + int(add[p])
                    if gid < oracle.NO_ID:
                        g.append(gid)
                        s.append(scores[p, q, r])
        g, s = np.array(g, np.int64), np.array(s, np.float32)
        order = np.lexsort((g, -s.astype(np.float64)))[:kout]
        oi[q, :order.size] = g[order]
        os_[q, :order.size] = s[order]
    return oi, os_


@pytest.mark.parametrize("parts,nq,kin,kout,mul", [(1, 5, 7, 7, 1), (3, 33, 100, 100, 3), (8, 17, 2000, 2000, 8),
                                                    (64, 4, 256, 300, 64), (2, 9, 10, 10, 1), (5, 3, 40, 500, 5)])
def test_merge_topk_matches_findlargest(parts, nq, kin, kout, mul):
    """sinn_merge_topk vs FindLargest over the union (Alg. 3): ties by ascending global id, padding,
    skipped SINN_NO_ID entries, the local -> global id map, more outputs than inputs."""
    import paper_2301_10622_b200 as sinn
    rng = np.random.default_rng(parts * 1000 + kin)
    ids = rng.integers(0, 50000, size=(parts, nq, kin)).astype(np.uint32)
    for p in range(parts):      # distinct local ids inside a list, as a shard returns them
        for q in range(nq):
            ids[p, q] = rng.choice(60000, kin, replace=False)
    scores = rng.choice(np.array([-2.5, -0.0, 0.0, 1.0, 1.0, 3.25, 7.0], np.float32), size=ids.shape)  # heavy ties
    scores += (rng.random(ids.shape) < 0.3) * rng.standard_normal(ids.shape).astype(np.float32)
    scores = scores.astype(np.float32)
    ids[rng.random(ids.shape) < 0.1] = oracle.NO_ID
    add = np.arange(parts, dtype=np.uint32) if mul > 1 else np.zeros(parts, np.uint32)
    if mul == 1 and parts > 1:  # global ids already: make the parts disjoint
        ids = np.where(ids == oracle.NO_ID, ids, ids * parts + np.arange(parts, dtype=np.uint32)[:, None, None])
    oi, os_ = sinn.merge_topk(t_i32(ids), t_f32(scores), kout, mul, add if mul > 1 else None)
    wi, ws = np_merge(ids, scores, kout, mul, add)
    np.testing.assert_array_equal(ids_np(oi), wi)
    np.testing.assert_array_equal(os_.cpu().numpy(), ws)


def test_merge_topk_rejects_bad_arguments():
    import paper_2301_10622_b200 as sinn
    ids = torch.zeros((2, 3, 9000), dtype=torch.int32, device="cuda")          # 18,000 > 16,384 items
    sc = torch.zeros((2, 3, 9000), dtype=torch.float32, device="cuda")
    with pytest.raises(sinn.SinnError) as e:
        sinn.merge_topk(ids, sc, 10)
    assert e.value.status == sinn.EINVAL
    with pytest.raises(sinn.SinnError):
        sinn.merge_topk(ids[:, :, :10].contiguous(), sc[:, :, :10].contiguous(), 0)
    ids65 = torch.zeros((65, 1, 4), dtype=torch.int32, device="cuda")
    with pytest.raises(sinn.SinnError):
        sinn.merge_topk(ids65, torch.zeros((65, 1, 4), dtype=torch.float32, device="cuda"), 4)
    oi, _ = sinn.merge_topk(torch.zeros((2, 0, 5), dtype=torch.int32, device="cuda"),
                            torch.zeros((2, 0, 5), dtype=torch.float32, device="cuda"), 5)
    assert oi.shape == (0, 5)


def test_rerank_of_given_candidates_matches_oracle_dots():
    """sinn_rerank on an unsharded index (id map 1, 0): exact scores and order of caller-chosen candidates,
    with SINN_NO_ID, vacant and out-of-range ids skipped; with a shard map only owned ids are scored."""
    cfg = datagen.CONFIGS["tiny"]
    P = Pair(cfg)
    ip, ix, v = datagen.docs(cfg, 0, 3000)
    P.insert(ip, ix, v, np.arange(3000, dtype=np.uint32))
    P.delete(np.arange(100, 200, dtype=np.uint32))
    qp, qi, qv = datagen.queries(cfg, 0, 25)
    rng = np.random.default_rng(3)
    kc, k = 300, 20
    cand = np.stack([rng.choice(3200, kc, replace=False) for _ in range(25)]).astype(np.uint32)  # some vacant / beyond
    cand[:, ::17] = oracle.NO_ID
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    for mul, add in ((1, 0), (3, 1)):
        oi, os_ = P.gpu.rerank(*tq, t_i32(cand), k, mul, add)
        oi, os_ = ids_np(oi), os_.cpu().numpy()
        for q in range(25):
            a, b = qp[q], qp[q + 1]
            own = [int(g) for g in cand[q] if g != oracle.NO_ID and g % mul == add and P.orc.is_live(int(g) // mul)]
            ex = np.array([P.orc.exact_dot(g // mul, qi[a:b], qv[a:b]) for g in own])
            mass = P.exact_mass([g // mul for g in own], qi[a:b], qv[a:b])
            order = np.lexsort((np.array(own), -ex))[:k]
            take = order.size
            got = oi[q][:take]
            assert np.all(oi[q][take:] == oracle.NO_ID) and np.all(np.isneginf(os_[q][take:]))
            pos = {g: t for t, g in enumerate(own)}
            assert all(int(g) in pos for g in got) and np.unique(got).size == take
            gi = np.array([pos[int(g)] for g in got], np.int64)
            np.testing.assert_array_less(np.abs(os_[q][:take] - ex[gi]), 1e-5 * mass[gi] + 1e-30)
            kth = ex[order[-1]] if take else 0.0
            for g in set(got.tolist()) ^ set(np.array(own)[order].tolist()):
                assert abs(ex[pos[int(g)]] - kth) <= 1e-5 * (mass[pos[int(g)]] + mass[order[-1]]) + 1e-30
    st = P.gpu.status_of(P.gpu._lib.sinn_rerank, 1, tq[0].data_ptr(), tq[1].data_ptr(), tq[2].data_ptr(), 10,
                         t_i32(cand).data_ptr(), 2, 2, 5, None, None, None)
    import paper_2301_10622_b200 as sinn
    assert st == sinn.EINVAL                                            # id_add >= id_mul


def test_gather_stores_beyond_one_query_pass():
    """Batches beyond 1,024 queries are scored in passes; the select kernels' gather stores must land at
    row (pass offset + query) of slot r in every buffer."""
    cfg = datagen.CONFIGS["tiny"]
    P = sharded_pair("tiny", 3000, 2, 3000, peer=True)
    nq, kp = 1500, 64
    qp, qi, qv = datagen.queries(cfg, 0, nq)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    P.gpu._set_peers(nq, kp)
    own = [s.phase_stage1_gather(tq, kp) for s in P.gpu.shards]
    assert torch.equal(own[0][0], own[1][0]) and torch.equal(own[0][1], own[1][1])
    plain = [s.phase_stage1(tq, kp) for s in P.gpu.shards]
    pi, ps = torch.stack([a for a, _ in plain]), torch.stack([b for _, b in plain])
    assert (own[0][0] == pi).float().mean().item() > 0.995
    fin = torch.isfinite(ps)
    assert torch.equal(fin, torch.isfinite(own[0][1]))
    torch.testing.assert_close(own[0][1][fin], ps[fin], rtol=1e-4, atol=1e-4)
    sub = np.r_[0:8, 1020:1030, 1492:1500]                       # queries on both sides of the pass boundary
    sp = np.concatenate([[0], np.cumsum([qp[q + 1] - qp[q] for q in sub])]).astype(np.int64)
    si = np.concatenate([qi[qp[q]:qp[q + 1]] for q in sub]).astype(np.int32)
    sv = np.concatenate([qv[qp[q]:qp[q + 1]] for q in sub]).astype(np.float32)
    vi, vs = P.gpu.shards[0].phase_select(own[0][0], own[0][1], kp)
    ci, _ = check_stage1(P, sp, si, sv, kp)                      # the facade's own run of the sub-batch
    got = ids_np(vi)[sub]
    assert np.mean([len(set(got[t].tolist()) & set(ci[t].tolist())) / kp for t in range(len(sub))]) > 0.97
