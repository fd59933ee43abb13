"""GPU (libsinn.so, sm_100a) vs oracle parity — run on a B200 with `pytest -m gpu`.

Sizes span several tiles and ragged tails; config-level parity at the scaled sizes of each
BASELINE.json config law, plus the full-size config-2 index in the bench launch configuration
(sampled queries).  Protocol: tests/gpu_util.py.
"""
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
    sinn.lib()  # loud failure if libsinn.so is missing


from gpu_util import Pair, check_final, check_postings, check_sketches, check_stage1, ids_np, t_i32, t_i64, t_f32  # noqa: E402


def build_pair(name, N=None, batch=None, host=False, bf16=False):
    cfg = datagen.CONFIGS[name]
    N = cfg.N if N is None else N
    batch = cfg.insert_batch if batch is None else batch
    P = Pair(cfg, bf16=bf16)
    for s in range(0, N, batch):
        c = min(batch, N - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        P.insert(ip, ix, v, np.arange(s, s + c, dtype=np.uint32), host=host)
    return P


@pytest.mark.parametrize("name", ["tiny", "c2s", "c3s", "c5s"])
def test_config_parity(name):
    cfg = datagen.CONFIGS[name]
    P = build_pair(name)
    N = cfg.N
    rng = np.random.default_rng(1)
    check_sketches(P, np.arange(N, dtype=np.uint32) if N <= 20000 else rng.choice(N, 5000, replace=False))
    terms = np.arange(cfg.n) if cfg.n <= 2000 else np.concatenate([np.arange(64), rng.choice(cfg.n, 400, replace=False)])
    check_postings(P, terms)
    qp, qi, qv = datagen.queries(cfg, 0, cfg.nq)
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=False)
    st = P.gpu.stats()
    assert st["live"] == N and st["postings"] == int(sum(len(r[0]) for r in P.rows.values()))


def test_decode_bit_exact():
    cfg = datagen.CONFIGS["c5s"]
    P = build_pair("c5s", N=6000)
    ids, terms, pos = [], [], []
    for i in range(0, 6000, 5):
        cols, _ = P.rows[i]
        for j in cols[::7]:
            for p in (0, 1):
                ids.append(i); terms.append(int(j)); pos.append(p)
    ids = np.array(ids, np.uint32)
    terms = np.array(terms, np.int32)
    pos = np.array(pos, np.uint8)
    got = P.gpu.decode(t_i32(ids), t_i32(terms.view(np.uint32)), torch.from_numpy(pos).cuda()).cpu().numpy()
    want = np.array([P.orc.decode(int(i), int(j), bool(p)) for i, j, p in zip(ids, terms, pos)], np.float32)
    np.testing.assert_array_equal(got, want)


def test_host_entry_points_match_device():
    cfg = datagen.CONFIGS["tiny"]
    P = build_pair("tiny", N=4000, batch=1500, host=True)
    check_sketches(P, np.arange(4000, dtype=np.uint32))
    qp, qi, qv = datagen.queries(cfg, 0, 50)
    a = check_final(P, qp, qi, qv, 10, 100, host=True)
    b = check_final(P, qp, qi, qv, 10, 100, host=False)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("poison", ["0", "1"])
def test_streaming_delete_recycle_parity(poison, monkeypatch):
    """Config-4 law at small scale: insert rounds (recycled ids first, LIFO), delete 1% of live, search.
    poison=1 fills every fresh index/workspace allocation with 0xA5 bytes (SINN_POISON): the path must
    not depend on freshly allocated (pool-recycled) memory being zero."""
    if poison == "1":
        monkeypatch.setenv("SINN_POISON", "1")
    cfg = datagen.CONFIGS["c4s"]
    P = Pair(cfg)
    free, next_id, gen = [], 0, 0
    for rnd in range(6):
        B = cfg.insert_batch
        ip, ix, v = datagen.docs(cfg, gen, B)
        gen += B
        ids = []
        for _ in range(B):
            if free:
                ids.append(free.pop())
            else:
                ids.append(next_id); next_id += 1
        P.insert(ip, ix, v, np.array(ids, np.uint32))
        live = np.array(sorted(P.rows), np.uint32)
        dele = datagen.choose(live, max(1, live.size // 100) * 5, cfg.seed, rnd)
        P.delete(dele)
        free.extend(int(i) for i in dele)
        qp, qi, qv = datagen.queries(cfg, rnd * cfg.nq, cfg.nq)
        check_stage1(P, qp, qi, qv, cfg.kprime)
        oi, _ = check_final(P, qp, qi, qv, cfg.k, cfg.kprime)
        assert not np.isin(oi, dele).any()
    rng = np.random.default_rng(0)
    check_postings(P, rng.choice(cfg.n, 300, replace=False))
    check_sketches(P, np.array(sorted(P.rows), np.uint32)[::7])


def test_kprime_all_gives_exact_topk():
    """O10 on the GPU: k' = live count -> exact top-k (the oracle's exact brute force)."""
    cfg = datagen.CONFIGS["tiny"]
    P = build_pair("tiny", N=3000)
    qp, qi, qv = datagen.queries(cfg, 0, 40)
    oi, os_ = check_final(P, qp, qi, qv, 10, 3000)
    eids, esc = P.orc.exact(qp, qi, qv, 10)
    for q in range(40):
        # equal ids except exact ties (fp32 re-rank vs fp64)
        diff = set(oi[q].tolist()) ^ set(eids[q].tolist())
        assert all(abs(P.orc.exact_dot(int(i), qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]]) - esc[q][-1]) < 1e-4
                   for i in diff)


def test_edge_cases_and_errors():
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    table = datagen.hash_table(cfg)
    G = sinn.Index(cfg.n, cfg.m, cfg.h, table)
    # empty index: padded results
    qp, qi, qv = datagen.queries(cfg, 0, 3)
    oi, os_ = G.search_host(qp, qi, qv, 5, 10)
    assert np.all(oi == oracle.NO_ID) and np.all(np.isneginf(os_))
    # empty query rows and zero-valued entries
    P = build_pair("tiny", N=500)
    qp2 = np.array([0, 0, 3, 3], np.int64)
    qi2 = np.array([5, 9, 17], np.int32)
    qv2 = np.array([0.0, 1.5, -2.0], np.float32)
    check_final(P, qp2, qi2, qv2, 10, 50)
    check_stage1(P, qp2, qi2, qv2, 50)
    # k' > live count: every live document is a candidate
    check_stage1(P, qp, qi, qv, 800)
    check_final(P, qp, qi, qv, 600, 800)
    # errors are all-or-nothing
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.insert_host([0, 1], [3], [1.0], [7])            # live id
    assert e.value.status == sinn.EEXIST
    for bad in (([0, 2], [4, 4], [1.0, 2.0], [600]),            # not strictly increasing
                ([0, 1], [cfg.n], [1.0], [600]),                 # index out of range
                ([0, 1], [1], [np.inf], [600]),                  # non-finite
                ([0, 1, 2], [1, 2], [1.0, 1.0], [600, 600]),     # duplicate ids
                ([0, 1], [1], [1.0], [0xFFFFFFFF])):             # reserved id
        with pytest.raises(sinn.SinnError) as e:
            P.gpu.insert_host(*bad)
        assert e.value.status == sinn.EINVAL
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.delete_host([600])
    assert e.value.status == sinn.ENOTFOUND
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.delete_host([3, 3])
    assert e.value.status == sinn.EINVAL
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.search_host([0, 2], [4, 3], [1.0, 1.0], 1, 1)
    assert e.value.status == sinn.EINVAL
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.search_host(qp, qi, qv, 11, 10)                  # k > k'
    assert e.value.status == sinn.EINVAL
    assert P.gpu.stats()["live"] == 500
    check_sketches(P, np.arange(500, dtype=np.uint32))
    check_postings(P, np.arange(cfg.n))
    check_final(P, qp, qi, qv, 10, 100)
    # Sinnamon+: negative values rejected, negative query entries contribute 0
    c3 = datagen.CONFIGS["c3s"]
    Q = build_pair("c3s", N=2000)
    with pytest.raises(sinn.SinnError):
        Q.gpu.insert_host([0, 1], [1], [-1.0], [5000])
    qp3, qi3, qv3 = datagen.queries(c3, 0, 10)
    qv3 = qv3.copy()
    qv3[::3] *= -1
    check_stage1(Q, qp3, qi3, qv3, 200)
    check_final(Q, qp3, qi3, qv3, 10, 200)


def test_unsorted_ids_and_sparse_id_space():
    """Ids in arbitrary order with gaps (capacity growth, unsorted-batch radix path)."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["c2s"]
    P = Pair(cfg)
    P.gpu.reserve(150_000, 1_000_000)  # part of the id space and entries reserved up front, the rest grows
    with pytest.raises(sinn.SinnError) as e:
        P.gpu.reserve(-1, 10)
    assert e.value.status == sinn.EINVAL
    rng = np.random.default_rng(9)
    pool = rng.choice(200_000, 12_000, replace=False).astype(np.uint32)
    for s in range(0, 12_000, 5000):
        c = min(5000, 12_000 - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        P.insert(ip, ix, v, pool[s:s + c])
    check_postings(P, rng.choice(cfg.n, 500, replace=False))
    check_sketches(P, pool[::11])
    qp, qi, qv = datagen.queries(cfg, 0, 30)
    check_stage1(P, qp, qi, qv, 500)
    check_final(P, qp, qi, qv, 10, 500)


@pytest.mark.slow
def test_full_config2_sampled_queries():
    """configs[1] at full size (1M docs, the bench workload) — sampled queries vs the oracle."""
    cfg = datagen.CONFIGS["c2"]
    P = build_pair("c2")
    qp, qi, qv = datagen.queries(cfg, 0, 16)
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)
    rng = np.random.default_rng(2)
    check_sketches(P, rng.choice(cfg.N, 2000, replace=False).astype(np.uint32))
    check_postings(P, rng.choice(cfg.n, 50, replace=False))


@pytest.mark.parametrize("name", ["tiny", "c2s", "c5s"])
def test_dense_path_parity(name, monkeypatch):
    """The dense fallback path (score rows in HBM), forced for every query, against the oracle."""
    monkeypatch.setenv("SINN_FORCE_DENSE", "1")
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 20000))
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 32))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)


def test_candidate_overflow_falls_back_to_dense(monkeypatch):
    """70,000 tied documents exceed the per-query candidate buffer (forced to 65,536 here; the
    default is larger): the synchronous search completes the query on the dense path; a
    SINN_SEARCH_NOSYNC search reports SINN_EAGAIN at sinn_sync."""
    import paper_2301_10622_b200 as sinn
    monkeypatch.setenv("SINN_HEAD", "0")
    monkeypatch.setenv("SINN_CAND_CAP", "65536")
    monkeypatch.setenv("SINN_POISON", "1")  # the overflowed query's row must not be read before it is written
    cfg = datagen.CONFIGS["tiny"]
    table = datagen.hash_table(cfg)
    P = Pair(cfg, table)
    N = 70_000
    ip = np.arange(N + 1, dtype=np.int64)
    ix = np.zeros(N, np.int32)
    v = np.ones(N, np.float32)
    v[::1000] = 2.0  # a few strictly better documents
    P.insert(ip, ix, v, np.arange(N, dtype=np.uint32))
    qp = np.array([0, 1, 3], np.int64)
    qi = np.array([0, 0, 5], np.int32)
    qv = np.array([1.0, 1.0, -1.0], np.float32)
    check_stage1(P, qp, qi, qv, 200)
    check_final(P, qp, qi, qv, 10, 200)
    G = P.gpu
    oi, os_ = G.search(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 10, 200, True, sync=False)
    with pytest.raises(sinn.SinnError) as e:
        G.sync()
    assert e.value.status == sinn.EAGAIN
    G.sync()  # the deferred status is cleared


def test_nosync_matches_sync():
    cfg = datagen.CONFIGS["c2s"]
    P = build_pair("c2s", N=30000)
    qp, qi, qv = datagen.queries(cfg, 0, 64)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    a = P.gpu.search(*tq, 10, 500, True)
    b = P.gpu.search(*tq, 10, 500, True, sync=False)
    P.gpu.sync()
    np.testing.assert_array_equal(ids_np(a[0]), ids_np(b[0]))


@pytest.mark.parametrize("name,head", [("c3s", "1"), ("c3s", "0"), ("c3s", "d"), ("c5s", "1"), ("c5s", "0"),
                                       ("c5s", "d"), ("c2s", "1"), ("c2s", "d"), ("tiny", "1"), ("tiny", "d")])
def test_head_split_parity(name, head, monkeypatch):
    """The head-term splits against the oracle: SINN_HEAD=1 the tile kernel (k_head.cu: head terms as an
    FFMA product per tile, tail entries sparse, sampled theta cascade); d the per-document dense product
    inside k_doc_score; 0 the plain sparse walk — including batches with no head term."""
    monkeypatch.setenv("SINN_HEAD", head)
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 30000))
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 40))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=False)


def _sampled_oracle(cfg, table, ids, bf16=False):
    """An oracle index of the given documents only (compact ids 0..len-1), rebuilt from their seeded
    rows: a document's Alg. 6 score and exact dot depend only on its own row, so these are the
    full index's values for those documents."""
    O = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, datagen.hash_table(cfg), cfg.upper_only, bf16=bf16)
    rows = [datagen.docs(cfg, int(i), 1) for i in ids]
    ip = np.zeros(len(rows) + 1, np.int64)
    ip[1:] = np.cumsum([r[0][1] for r in rows])
    ix = np.concatenate([r[1] for r in rows]) if rows else np.zeros(0, np.int32)
    v = np.concatenate([r[2] for r in rows]) if rows else np.zeros(0, np.float32)
    assert O.insert(ip, ix, v, np.arange(len(rows), dtype=np.uint32)) == oracle.OK
    return O


@pytest.mark.slow
@pytest.mark.parametrize("name,bf16", [("c3", False), ("c5", False), ("c5", True)])
def test_full_size_sampled_parity(name, bf16):
    """configs[2] / configs[4] at full size in the bench's launch configuration (1,024-query batch):
    for sampled queries, every stage-1 candidate's approximate score and every returned exact score
    are recomputed one by one by the oracle; random other documents must not beat the k'-th
    candidate (V is the top-k'), and the final top-k is the exact re-rank of V."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS[name]
    table = datagen.hash_table(cfg)
    G = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only, bf16=bf16)
    for s in range(0, cfg.N, cfg.insert_batch):
        c = min(cfg.insert_batch, cfg.N - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        G.insert(t_i64(ip), t_i32(ix.view(np.uint32)), t_f32(v), t_i32(np.arange(s, s + c, dtype=np.uint32)))
    qp, qi, qv = datagen.queries(cfg, 0, cfg.batch)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    ci, cs = G.search_stage1(*tq, cfg.kprime)
    oi, os_ = G.search(*tq, cfg.k, cfg.kprime, True)
    ci, cs, oi, os_ = ids_np(ci), cs.cpu().numpy(), ids_np(oi), os_.cpu().numpy()
    rng = np.random.default_rng(7)
    for q in (0, 511, 1023):
        a, b = qp[q], qp[q + 1]
        V = ci[q][ci[q] != oracle.NO_ID]
        assert V.size == cfg.kprime and np.unique(V).size == V.size
        others = np.setdiff1d(rng.choice(cfg.N, 1500, replace=False).astype(np.uint32), V)
        ids = np.concatenate([V, others, oi[q]]).astype(np.uint32)
        O = _sampled_oracle(cfg, table, ids, bf16)
        s, mass = O.scores(qi[a:b], qv[a:b])
        tol = 1e-5 * mass + 1e-30
        nv = V.size
        np.testing.assert_array_less(np.abs(cs[q][:nv] - s[:nv]), tol[:nv] + 1e-30)  # stage-1 scores
        kth = cs[q][nv - 1]
        no = others.size
        assert np.all(s[nv:nv + no] <= kth + tol[nv:nv + no] + 1e-5 * mass[:nv].max()), "a non-candidate beats V"
        ex = np.array([O.exact_dot(t, qi[a:b], qv[a:b]) for t in range(nv)])
        order = np.lexsort((V, -ex))[: cfg.k]
        got = oi[q]
        exg = np.array([O.exact_dot(nv + no + t, qi[a:b], qv[a:b]) for t in range(got.size)])
        np.testing.assert_allclose(os_[q], exg, rtol=1e-5, atol=1e-5)
        kex = ex[order[-1]]
        for i in set(got.tolist()) ^ set(V[order].tolist()):
            t = int(np.flatnonzero(V == i)[0]) if i in V else None
            val = ex[t] if t is not None else exg[list(got).index(i)]
            assert abs(val - kex) <= 1e-5 * (abs(kex) + 1), (q, i, val, kex)
    G.close()


@pytest.mark.slow
def test_full_streaming_sampled_parity():
    """configs[3] at full size: 0 -> 4M documents in 100K inserts, 1% of live deleted after each
    (LIFO id recycling), as bench.py runs it; then, for sampled queries, the candidates' scores and the
    final top-k are recomputed one by one from each live id's current row, deleted ids never appear,
    and random live documents do not beat the k'-th candidate."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["c4"]
    table = datagen.hash_table(cfg)
    G = sinn.Index(cfg.n, cfg.m, cfg.h, table, cfg.upper_only)
    row_of = np.full(cfg.N + cfg.insert_batch, -1, np.int64)  # id -> generator row of its current document
    free, next_id, gen, rnd = [], 0, 0, 0
    while (row_of >= 0).sum() < cfg.N:
        B = cfg.insert_batch
        ip, ix, v = datagen.docs(cfg, gen, B)
        take = min(len(free), B)
        ids = np.empty(B, np.uint32)
        for r in range(take):
            ids[r] = free.pop()
        ids[take:] = np.arange(next_id, next_id + B - take, dtype=np.uint32)
        next_id += B - take
        G.insert(t_i64(ip), t_i32(ix.view(np.uint32)), t_f32(v), t_i32(ids))
        row_of[ids] = np.arange(gen, gen + B)
        gen += B
        pool = np.flatnonzero(row_of >= 0).astype(np.uint32)
        dele = datagen.choose(pool, pool.size // 100, cfg.seed, rnd)
        G.delete(t_i32(dele))
        row_of[dele] = -1
        free.extend(int(i) for i in dele)
        rnd += 1
    live = np.flatnonzero(row_of >= 0)
    assert G.stats()["live"] == live.size
    qp, qi, qv = datagen.queries(cfg, 0, cfg.batch)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    ci, cs = G.search_stage1(*tq, cfg.kprime)
    oi, os_ = G.search(*tq, cfg.k, cfg.kprime, True)
    ci, cs, oi, os_ = ids_np(ci), cs.cpu().numpy(), ids_np(oi), os_.cpu().numpy()
    rng = np.random.default_rng(11)
    for q in (0, 700):
        a, b = qp[q], qp[q + 1]
        V = ci[q][ci[q] != oracle.NO_ID]
        assert V.size == cfg.kprime and np.all(row_of[V] >= 0) and np.all(row_of[oi[q]] >= 0)
        others = np.setdiff1d(rng.choice(live, 1500, replace=False), V).astype(np.uint32)
        ids = np.concatenate([V, others, oi[q]]).astype(np.uint32)
        O = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, cfg.upper_only)
        rows = [datagen.docs(cfg, int(row_of[i]), 1) for i in ids]
        rip = np.zeros(len(rows) + 1, np.int64)
        rip[1:] = np.cumsum([r[0][1] for r in rows])
        assert O.insert(rip, np.concatenate([r[1] for r in rows]), np.concatenate([r[2] for r in rows]),
                        np.arange(len(rows), dtype=np.uint32)) == oracle.OK
        s, mass = O.scores(qi[a:b], qv[a:b])
        tol = 1e-5 * mass + 1e-30
        nv, no = V.size, others.size
        np.testing.assert_array_less(np.abs(cs[q][:nv] - s[:nv]), tol[:nv] + 1e-30)
        assert np.all(s[nv:nv + no] <= cs[q][nv - 1] + tol[nv:nv + no] + 1e-5 * mass[:nv].max())
        exg = np.array([O.exact_dot(nv + no + t, qi[a:b], qv[a:b]) for t in range(cfg.k)])
        np.testing.assert_allclose(os_[q], exg, rtol=1e-5, atol=1e-5)
        ex = np.array([O.exact_dot(t, qi[a:b], qv[a:b]) for t in range(nv)])
        want = V[np.lexsort((V, -ex))][: cfg.k]
        kex = np.sort(ex)[::-1][cfg.k - 1]
        for i in set(oi[q].tolist()) ^ set(want.tolist()):
            val = ex[int(np.flatnonzero(V == i)[0])] if i in V else exg[list(oi[q]).index(i)]
            assert abs(val - kex) <= 1e-5 * (abs(kex) + 1)
    G.close()


@pytest.mark.parametrize("name", ["tiny", "c2s", "c3s", "c5s"])
def test_exact_search_matches_oracle_exact(name):
    """sinn_search_exact (LinScan, Alg. 2, on the GPU) vs the oracle's exact MIPS: scores of the returned
    ids equal their exact dots within the fp32 tolerance; id sets equal up to ties at the k-th score.
    Config-3 queries get some negative values (exact MIPS counts them even under Sinnamon+)."""
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 30000))
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 40))
    if cfg.upper_only:
        qv = qv.copy()
        qv[::4] *= -1
    gi, gs = P.gpu.search_exact(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.k)
    gi, gs = ids_np(gi), gs.cpu().numpy()
    eids, esc = P.orc.exact(qp, qi, qv, cfg.k)
    for q in range(qp.size - 1):
        a, b = qp[q], qp[q + 1]
        ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in gi[q]])
        mass = P.exact_mass(gi[q], qi[a:b], qv[a:b])
        np.testing.assert_array_less(np.abs(gs[q] - ex), 1e-5 * mass + 1e-30)
        assert np.all(np.diff(gs[q]) <= 0)
        kth = esc[q][-1]
        for i in set(gi[q].tolist()) ^ set(eids[q].tolist()):
            v = P.orc.exact_dot(int(i), qi[a:b], qv[a:b])
            assert abs(v - kth) <= 1e-5 * (abs(kth) + P.exact_mass([i], qi[a:b], qv[a:b])[0]) + 1e-30, (q, i, v, kth)


@pytest.mark.parametrize("name,budget", [("c2s", 1), ("c2s", 7), ("c5s", 12), ("c3s", 5), ("tiny", 3)])
def test_anytime_budget_parity(name, budget):
    """sinn_search_anytime (R20): stage 1 scores each query's `budget` largest-|q_j| terms,
    the re-rank uses the whole query.  Every returned id is a top-k' document of the oracle's budgeted
    scores (up to ties at the k'-th) with its exact score, and the GPU's top-k equals the oracle's
    except for ties at the k-th exact score or the k'-th budgeted score."""
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 20000))
    qp, qi, qv = datagen.queries(cfg, 0, 24)
    oi, os_ = P.gpu.search_anytime(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.k, cfg.kprime, budget)
    oi, os_ = ids_np(oi), os_.cpu().numpy()
    oids, osc = P.orc.search(qp, qi, qv, cfg.k, cfg.kprime, True, max_terms=budget)
    for q in range(qp.size - 1):
        a, b = qp[q], qp[q + 1]
        s, smass = P.orc.scores(qi[a:b], qv[a:b], max_terms=budget)
        live = np.isfinite(s)
        order = np.lexsort((np.arange(s.size), -s))
        take = min(cfg.kprime, int(live.sum()))
        kp_th = s[order[take - 1]]
        got = oi[q][oi[q] != oracle.NO_ID]
        ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in got])
        emass = P.exact_mass(got, qi[a:b], qv[a:b])
        np.testing.assert_array_less(np.abs(os_[q][:got.size] - ex), 1e-5 * emass + 1e-30)
        assert np.all(s[got] >= kp_th - 1e-5 * (smass[got] + smass[order[take - 1]]) - 1e-30)
        kex = ex.min() if ex.size else 0.0
        for i in set(oids[q][oids[q] != oracle.NO_ID].tolist()) - set(got.tolist()):
            v = P.orc.exact_dot(int(i), qi[a:b], qv[a:b])
            tie_k = v <= kex + 1e-5 * (abs(kex) + P.exact_mass([i], qi[a:b], qv[a:b])[0])
            tie_kp = abs(s[i] - kp_th) <= 1e-5 * (smass[i] + smass[order[take - 1]]) + 1e-30
            assert tie_k or tie_kp, (q, i, v, kex)


@pytest.mark.parametrize("name", ["tiny", "c2s", "c5s", "c3s"])
def test_constrained_search_parity(name):
    """sinn_search_filtered (Eq. 3) against the oracle's filtered search: only allowed documents
    come back, with their exact scores, and the top-k equals the oracle's up to ties at the k-th exact or
    the k'-th approximate score; an all-zeros mask returns nothing; an all-ones mask equals sinn_search."""
    cfg = datagen.CONFIGS[name]
    N = min(cfg.N, 20000)
    P = build_pair(name, N=N)
    rng = np.random.default_rng(3)
    allowed = rng.random(N) < 0.4
    words = np.zeros((N + 31) // 32, np.uint32)
    for i in np.flatnonzero(allowed):
        words[i >> 5] |= np.uint32(1 << (i & 31))
    qp, qi, qv = datagen.queries(cfg, 0, 24)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    oi, os_ = P.gpu.search_filtered(*tq, cfg.k, cfg.kprime, t_i32(words))
    oi, os_ = ids_np(oi), os_.cpu().numpy()
    fid, _ = P.orc.search_filtered(qp, qi, qv, cfg.k, cfg.kprime, words)
    for q in range(qp.size - 1):
        a, b = qp[q], qp[q + 1]
        got = oi[q][oi[q] != oracle.NO_ID]
        assert got.size == min(cfg.k, int(allowed.sum())) and np.all(allowed[got])
        ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in got])
        np.testing.assert_array_less(np.abs(os_[q][:got.size] - ex), 1e-5 * P.exact_mass(got, qi[a:b], qv[a:b]) + 1e-30)
        s, smass = P.orc.scores(qi[a:b], qv[a:b])
        s = np.where(np.arange(s.size) < N, s, -np.inf)
        s[:N][~allowed] = -np.inf
        order = np.lexsort((np.arange(s.size), -s))
        take = min(cfg.kprime, int(np.isfinite(s).sum()))
        kp_th = s[order[take - 1]]
        kex = ex.min()
        for i in set(fid[q][fid[q] != oracle.NO_ID].tolist()) - set(got.tolist()):
            v = P.orc.exact_dot(int(i), qi[a:b], qv[a:b])
            tie_k = v <= kex + 1e-5 * (abs(kex) + P.exact_mass([i], qi[a:b], qv[a:b])[0])
            tie_kp = abs(s[i] - kp_th) <= 1e-5 * (smass[i] + smass[order[take - 1]]) + 1e-30
            assert tie_k or tie_kp, (q, i, v, kex)
    zi, _ = P.gpu.search_filtered(*tq, cfg.k, cfg.kprime, t_i32(np.zeros_like(words)))
    assert np.all(ids_np(zi) == oracle.NO_ID)
    ai, a_s = P.gpu.search_filtered(*tq, cfg.k, cfg.kprime, t_i32(np.full_like(words, 0xFFFFFFFF)))
    ui, u_s = P.gpu.search(*tq, cfg.k, cfg.kprime, True)
    ai, ui, a_s = ids_np(ai), ids_np(ui), a_s.cpu().numpy()
    # equal up to exact-score ties at the k-th (fp32 sums may differ in the last place between two
    # calls when updates land in a run-dependent order: R7)
    for q in range(qp.size - 1):
        a, b = qp[q], qp[q + 1]
        kex = a_s[q][cfg.k - 1]
        for i in set(ai[q].tolist()) ^ set(ui[q].tolist()):
            v = P.orc.exact_dot(int(i), qi[a:b], qv[a:b])
            assert abs(v - kex) <= 1e-5 * (P.exact_mass([i], qi[a:b], qv[a:b])[0] + abs(kex)) + 1e-30, (q, i)


def test_batches_beyond_1024_queries():
    """One call with 2,500 queries (three 1,024-query passes, the last ragged): sampled queries from every
    pass match the oracle (stage 1 and final), as in a single-pass batch."""
    cfg = datagen.CONFIGS["c2s"]
    P = build_pair("c2s", N=25000)
    qp, qi, qv = datagen.queries(cfg, 0, 2500)
    tq = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    ci, cs = P.gpu.search_stage1(*tq, cfg.kprime)
    oi, os_ = P.gpu.search(*tq, cfg.k, cfg.kprime, True)
    ci, cs, oi, os_ = ids_np(ci), cs.cpu().numpy(), ids_np(oi), os_.cpu().numpy()
    for q in (0, 1023, 1024, 2047, 2048, 2499):
        a, b = qp[q], qp[q + 1]
        sub = np.array([0, b - a], np.int64)
        # the big batch's rows for query q, checked against the oracle (summation order within a document
        # may differ from a one-query batch, so the comparison is the oracle's tolerance, not equality)
        s, mass = P.orc.scores(qi[a:b], qv[a:b])
        take = min(cfg.kprime, int(np.isfinite(s).sum()))
        g = ci[q][:take]
        np.testing.assert_array_less(np.abs(cs[q][:take] - s[g]), 1e-5 * mass[g] + 1e-30)
        kth = np.sort(s[np.isfinite(s)])[::-1][take - 1]
        assert np.all(s[g] >= kth - 1e-5 * (mass[g] + mass.max()))
        ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in oi[q]])
        np.testing.assert_array_less(np.abs(os_[q] - ex), 1e-5 * P.exact_mass(oi[q], qi[a:b], qv[a:b]) + 1e-30)
        check_final(P, sub, qi[a:b], qv[a:b], cfg.k, cfg.kprime)


# ---------------------------------------------------------------- F3: bfloat16 sketch cells (R21)
@pytest.mark.parametrize("name", ["tiny", "c2s", "c3s", "c5s"])
def test_bf16_sketch_parity(name):
    """SINN_SKETCH_BF16: the bfloat16 cells (U rounded up, L rounded down) are bit-exact against the
    oracle's, decodes bit-exact, scores/candidates/final top-k within the parity protocol."""
    cfg = datagen.CONFIGS[name]
    N = min(cfg.N, 20000)
    P = build_pair(name, N=N, bf16=True)
    check_sketches(P, np.arange(N, dtype=np.uint32))
    ids, terms, pos = [], [], []
    for i in range(0, N, 7):
        cols, _ = P.rows[i]
        for j in cols[::5]:
            for p in ((1,) if cfg.upper_only else (0, 1)):
                ids.append(i); terms.append(int(j)); pos.append(p)
    ids = np.array(ids, np.uint32)
    terms = np.array(terms, np.int32)
    pos = np.array(pos, np.uint8)
    got = P.gpu.decode(t_i32(ids), t_i32(terms.view(np.uint32)), torch.from_numpy(pos).cuda()).cpu().numpy()
    want = np.array([P.orc.decode(int(i), int(j), bool(p)) for i, j, p in zip(ids, terms, pos)], np.float32)
    np.testing.assert_array_equal(got, want)
    assert np.all((got.view(np.uint32) & 0xFFFF) == 0)  # bfloat16 values
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 48))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    st = P.gpu.stats()
    assert st["bytes_sketch"] == (1 if cfg.upper_only else 2) * st["capacity"] * cfg.m * 2


def test_bf16_dense_path_and_streaming(monkeypatch):
    """bfloat16 index on the dense fallback path (SINN_FORCE_DENSE) and under delete + id recycling."""
    cfg = datagen.CONFIGS["c2s"]
    P = build_pair("c2s", N=20000, bf16=True)
    rng = np.random.default_rng(5)
    dels = rng.choice(20000, 500, replace=False).astype(np.uint32)
    P.delete(dels)
    ip, ix, v = datagen.docs(cfg, 30000, 300)
    P.insert(ip, ix, v, dels[:300])
    check_sketches(P, dels[:300])
    qp, qi, qv = datagen.queries(cfg, 0, 32)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    monkeypatch.setenv("SINN_FORCE_DENSE", "1")
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


def test_bf16_rejects_m_not_multiple_of_8():
    import paper_2301_10622_b200 as sinn
    with pytest.raises(sinn.SinnError):
        sinn.Index(100, 60, 2, np.zeros(200, np.int32), bf16=True)


def test_raw_store_compaction_under_recycling():
    """The raw store (vector storage S) reclaims deleted rows: when it must grow while a
    quarter or more of it is dead, live rows are compacted first; re-rank (Alg. 7) and exact search
    still read the right rows afterwards."""
    cfg = datagen.CONFIGS["tiny"]
    P = build_pair("tiny", N=4000, batch=4000)
    before = P.gpu.stats()
    rng = np.random.default_rng(11)
    dels = rng.choice(4000, 2000, replace=False).astype(np.uint32)
    P.delete(dels)
    ip, ix, v = datagen.docs(cfg, 10_000, 2400)
    P.insert(ip, ix, v, np.concatenate([dels, np.arange(4000, 4400, dtype=np.uint32)]))
    after = P.gpu.stats()
    assert after["raw_entries"] == after["postings"]          # compacted: no dead entries left
    assert after["raw_entries"] < before["raw_entries"] + int(np.diff(ip).sum())
    check_sketches(P, np.concatenate([dels[:200], np.arange(4000, 4400, dtype=np.uint32)]))
    qp, qi, qv = datagen.queries(cfg, 0, 60)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    ei, es = P.gpu.search_exact(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.k)
    ei, es = ids_np(ei), es.cpu().numpy()
    for q in range(60):
        a, b = qp[q], qp[q + 1]
        for t in range(cfg.k):
            if ei[q][t] != oracle.NO_ID:
                ex = P.orc.exact_dot(int(ei[q][t]), qi[a:b], qv[a:b])
                assert abs(es[q][t] - ex) <= 1e-5 * max(1.0, abs(ex))


@pytest.mark.parametrize("name,single", [("tiny", "1"), ("c2s", "0"), ("c5s", "0"), ("c3s", "1")])
def test_column_buffering_modes(name, single, monkeypatch):
    """k_doc_score with one sketch-column buffer per warp (staged after the previous document's last
    decode) and with two (staged a document ahead): both match the oracle."""
    monkeypatch.setenv("SINN_SINGLE_BUF", single)
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 20000))
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 32))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


def test_insert_append_and_merge_paths_interleaved():
    """Bulk loads of fresh ids past every occupied tile are appended in place; anything else is
    merged tile by tile.  Interleave both (with gaps, a non-aligned boundary, deletes) and check
    the postings of every term and the search results against the oracle (O12)."""
    cfg = datagen.CONFIGS["tiny"]
    P = Pair(cfg)
    def ins(lo, hi, src):
        ip, ix, v = datagen.docs(cfg, src, hi - lo)
        P.insert(ip, ix, v, np.arange(lo, hi, dtype=np.uint32))
    ins(0, 5000, 0)          # append (empty index)
    ins(10000, 12010, 5000)  # append past a gap (ends inside tile 375)
    ins(6000, 7013, 7000)    # below id_end: merge
    ins(12020, 12500, 9000)  # shares tile 375 with the live ids 12000..12009: merge
    P.delete(np.arange(100, 400, dtype=np.uint32))
    ins(12512, 13000, 9600)  # past every occupied tile: append
    ins(100, 300, 9900)      # recycled ids: merge
    check_postings(P, np.arange(cfg.n))
    qp, qi, qv = datagen.queries(cfg, 0, 40)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


@pytest.mark.parametrize("name", ["c3s", "c5s", "c2s"])
def test_nested_sample_threshold(name, monkeypatch):
    """The nested sample (a 1/8 sample's bound floors the full sample's histogram) forced on at test
    size: the threshold stays a provable bound, so candidates and final results match the oracle."""
    monkeypatch.setenv("SINN_CASCADE", "1")
    cfg = datagen.CONFIGS[name]
    P = build_pair(name, N=min(cfg.N, 40000))
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 32))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
