"""GPU vs oracle parity on the configurations and edge cases the ABI accepts beyond the BASELINE
configs (round-2 VERDICT "parity holes"): h = 4 (the directory's high map half), h = 6 and 8 (the
generic pi-table path), fp32 m % 4 != 0 (4-byte column copies), large m (few warps per CTA / the
dense path), exact ties at the k'-th score (selected by ascending id, R10), the candidate
shortfall guard, batches beyond 65,535 queries with re-rank, and null CSR arrays.

Protocol: tests/gpu_util.py (sketches bit-exact, scores within 1e-5 of the term mass, V and the final
top-k against the oracle).  Rules followed: Alg. 5, Alg. 6,
Alg. 7, Alg. 3's FindLargest.
"""
import ctypes
import dataclasses

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


from gpu_util import Pair, check_final, check_postings, check_sketches, check_stage1, ids_np, t_f32, t_i32, t_i64  # noqa: E402


def _pair(cfg, N, batch):
    P = Pair(cfg)
    for s in range(0, N, batch):
        c = min(batch, N - s)
        ip, ix, v = datagen.docs(cfg, s, c)
        P.insert(ip, ix, v, np.arange(s, s + c, dtype=np.uint32))
    return P


@pytest.mark.parametrize("m,h,upper", [(64, 4, False), (64, 6, False), (64, 8, False), (60, 2, False),
                                       (60, 3, True), (512, 3, False), (1024, 2, False), (2048, 5, False)])
def test_map_count_and_sketch_width_paths(m, h, upper):
    """h = 4: pi_2, pi_3 from the directory's high word; h = 6, 8: the generic path reading the pi
    table; m = 60 (fp32, m % 4 != 0): 4-byte column copies; m = 512: a few warps per CTA; m = 1024,
    2048: beyond the tile path's shared memory (dense path).  5,003 documents: 157 tiles, a ragged tail."""
    base = datagen.CONFIGS["tiny"]
    if upper:
        spec = dataclasses.replace(base.doc, val_kind=datagen.VAL_LOGNORMAL, val_a=0.0, val_b=1.0)
        qspec = dataclasses.replace(base.query, val_kind=datagen.VAL_LOGNORMAL, val_a=0.0, val_b=1.0)
        cfg = dataclasses.replace(base, name=f"m{m}h{h}u", m=m, h=h, upper_only=True, doc=spec, query=qspec,
                                  seed=base.seed + 100 + m + h)
    else:
        cfg = dataclasses.replace(base, name=f"m{m}h{h}", m=m, h=h, seed=base.seed + 100 + m + h)
    N = 5003
    P = _pair(cfg, N, 2000)
    check_sketches(P, np.arange(N, dtype=np.uint32)[::3])
    check_postings(P, np.arange(0, cfg.n, 7))
    qp, qi, qv = datagen.queries(cfg, 0, 40)
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


def _empty_queries(nq, n, seed):
    """nq queries: empty rows and rows whose terms occur in no document (every score is exactly 0)."""
    rng = np.random.default_rng(seed)
    ip = [0]
    ix, v = [], []
    for q in range(nq):
        if q % 2:
            cols = np.sort(rng.choice(np.arange(n, n + 1000), 5, replace=False)).astype(np.int32)
            ix.append(cols)
            v.append(rng.normal(size=5).astype(np.float32))
        ip.append(ip[-1] + (5 if q % 2 else 0))
    ix = np.concatenate(ix) if ix else np.zeros(0, np.int32)
    v = np.concatenate(v) if v else np.zeros(0, np.float32)
    return np.array(ip, np.int64), ix, v


@pytest.mark.parametrize("N,kprime,dense", [(5000, 100, False), (40000, 500, False), (20000, 100, True)])
def test_exact_ties_at_kprime_are_taken_by_ascending_id(N, kprime, dense, monkeypatch):
    """Every live document scores exactly 0 (R8): V must be ids 0..k'-1 and the top-k ids 0..k-1 —
    Alg. 3 admits items in order and the build orders ties by ascending id (R10), never by the atomic
    arrival order.  5,000 docs: the register select; 40,000: the three-level histogram select; the
    dense path with 20,000 > 16,384 ties of the threshold key: its tie ranks per slice."""
    if dense:
        monkeypatch.setenv("SINN_FORCE_DENSE", "1")
    base = datagen.CONFIGS["tiny"]
    cfg = dataclasses.replace(base, n=2000, doc=dataclasses.replace(base.doc, n=1000),
                              query=dataclasses.replace(base.query, n=2000), seed=base.seed + 7)
    P = _pair(cfg, N, 10000)
    qp, qi, qv = _empty_queries(6, 1000, 3)
    ci, cs = P.gpu.search_stage1(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), kprime)
    ci, cs = ids_np(ci), cs.cpu().numpy()
    for q in range(qp.size - 1):
        np.testing.assert_array_equal(ci[q], np.arange(kprime, dtype=np.uint32))
        assert np.all(cs[q] == 0.0)
    oi, os_ = P.gpu.search(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 10, kprime, True)
    oi, os_ = ids_np(oi), os_.cpu().numpy()
    for q in range(qp.size - 1):
        np.testing.assert_array_equal(oi[q], np.arange(10, dtype=np.uint32))
        assert np.all(os_[q] == 0.0)


def test_candidate_shortfall_goes_to_the_dense_path(monkeypatch):
    """theta_q raised past the sample's bound (test hook SINN_TEST_THETA_BUMP): the full pass emits
    fewer than k' candidates, and k_cand_select's shortfall guard must finish those queries on the
    dense path — the results still match the oracle (Alg. 7: V = FindLargest(scores, k'))."""
    cfg = datagen.CONFIGS["c2s"]
    P = _pair(cfg, 30000, 15000)
    qp, qi, qv = datagen.queries(cfg, 0, 24)
    monkeypatch.setenv("SINN_TEST_THETA_BUMP", "1")
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


def test_rerank_batch_beyond_65535_queries():
    """70,000 queries with re-rank (grid.y of the re-rank is chunked): the rows past 65,535 equal the
    same queries searched in a small batch, which check_final pins to the oracle."""
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 3000, 3000)
    nq = 70000
    qp, qi, qv = datagen.queries(cfg, 0, nq)
    oi, os_ = P.gpu.search(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.k, cfg.kprime, True)
    oi, os_ = ids_np(oi), os_.cpu().numpy()
    q0 = nq - 40
    sp, si, sv = datagen.queries(cfg, q0, 40)
    wi, ws = check_final(P, sp, si, sv, cfg.k, cfg.kprime, rerank=True)
    np.testing.assert_array_equal(oi[q0:], wi)
    np.testing.assert_allclose(os_[q0:], ws, rtol=0, atol=0)


def test_insert_with_null_arrays_is_einval_not_a_fault():
    """indices/values NULL while rows hold entries: SINN_EINVAL before any entry is read (a fault
    would poison the CUDA context); the index is unchanged and still searchable."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 2000, 2000)
    ip, ix, v = datagen.docs(cfg, 2000, 10)
    d_ip, d_ids = t_i64(ip), t_i32(np.arange(2000, 2010, dtype=np.uint32))
    L = sinn.lib()
    st = L.sinn_insert(P.gpu._h, 10, ctypes.c_void_p(d_ip.data_ptr()), None, None,
                       ctypes.c_void_p(d_ids.data_ptr()), None)
    assert st == sinn.EINVAL
    assert P.gpu.stats()["live"] == 2000
    qp, qi, qv = datagen.queries(cfg, 0, 20)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)


@pytest.mark.parametrize("name", ["c3s", "c5s"])
@pytest.mark.parametrize("mode", ["w16", "w8", "tau"])
def test_head_heavy_scoring_kernels(name, mode, monkeypatch):
    """The Zipf laws of configs 3 and 5 through k_doc_score's per-document dense head product (head
    query rows in TMEM): 16 head terms (default), 8 (SINN_HEAD_W=8), and a low coverage threshold
    (SINN_HEAD_TAU=0.02: every one of the 16 head slots taken, terms of low coverage included)."""
    if mode == "w8":
        monkeypatch.setenv("SINN_HEAD_W", "8")
    if mode == "tau":
        monkeypatch.setenv("SINN_HEAD_TAU", "0.02")
    cfg = datagen.CONFIGS[name]
    P = _pair(cfg, cfg.N, cfg.insert_batch)
    qp, qi, qv = datagen.queries(cfg, 0, cfg.nq)
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


@pytest.mark.parametrize("name", ["tiny", "c2s", "c5s", "c3s"])
def test_per_query_constraint_masks(name):
    """F4 (Eq. 3) with a constraint set PER QUERY: one mixed batch where query q uses
    mask qmask[q] of a table (or none) must return, for every query, what the oracle's filtered search
    returns with that query's mask alone — up to ties at the k-th exact / k'-th approximate score."""
    cfg = datagen.CONFIGS[name]
    N = min(cfg.N, 20000)
    P = _pair(cfg, N, cfg.insert_batch)
    rng = np.random.default_rng(11)
    nmasks, W = 3, (N + 31) // 32 + 1
    allowed = [rng.random(N) < f for f in (0.5, 0.1, 0.003)]  # the last admits fewer than k' documents
    masks = np.zeros((nmasks, W), np.uint32)
    for r, al in enumerate(allowed):
        for i in np.flatnonzero(al):
            masks[r, i >> 5] |= np.uint32(1 << (i & 31))
    nq = 24
    qp, qi, qv = datagen.queries(cfg, 0, nq)
    qmask = np.array([(q % 4) - 1 for q in range(nq)], np.int32)  # -1, 0, 1, 2, -1, ...
    oi, os_ = P.gpu.search_masked(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), cfg.k, cfg.kprime,
                                  torch.from_numpy(masks.view(np.int32)).cuda(), torch.from_numpy(qmask).cuda())
    oi, os_ = ids_np(oi), os_.cpu().numpy()
    for r in range(-1, nmasks):
        qs = [q for q in range(nq) if qmask[q] == r]
        words = masks[r] if r >= 0 else np.full(W, 0xFFFFFFFF, np.uint32)
        sub_p = np.concatenate([[0], np.cumsum([qp[q + 1] - qp[q] for q in qs])]).astype(np.int64)
        sub_i = np.concatenate([qi[qp[q]:qp[q + 1]] for q in qs]).astype(np.int32)
        sub_v = np.concatenate([qv[qp[q]:qp[q + 1]] for q in qs]).astype(np.float32)
        fid, _ = P.orc.search_filtered(sub_p, sub_i, sub_v, cfg.k, cfg.kprime, words)
        al = allowed[r] if r >= 0 else np.ones(N, bool)
        for t, q in enumerate(qs):
            a, b = qp[q], qp[q + 1]
            got = oi[q][oi[q] != oracle.NO_ID]
            assert got.size == min(cfg.k, int(al.sum())) and np.all(al[got]), (q, r)
            ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in got])
            np.testing.assert_array_less(np.abs(os_[q][:got.size] - ex),
                                         1e-5 * P.exact_mass(got, qi[a:b], qv[a:b]) + 1e-30)
            s, smass = P.orc.scores(qi[a:b], qv[a:b])
            s = np.where(np.arange(s.size) < N, s, -np.inf)
            s[:N][~al] = -np.inf
            order = np.lexsort((np.arange(s.size), -s))
            take = min(cfg.kprime, int(np.isfinite(s).sum()))
            kp_th = s[order[take - 1]]
            kex = ex.min() if ex.size else 0.0
            for i in set(fid[t][fid[t] != oracle.NO_ID].tolist()) - set(got.tolist()):
                v = P.orc.exact_dot(int(i), qi[a:b], qv[a:b])
                tie_k = v <= kex + 1e-5 * (abs(kex) + P.exact_mass([i], qi[a:b], qv[a:b])[0])
                tie_kp = abs(s[i] - kp_th) <= 1e-5 * (smass[i] + smass[order[take - 1]]) + 1e-30
                assert tie_k or tie_kp, (q, r, i, v, kex)


def test_per_query_mask_argument_errors():
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 1000, 1000)
    qp, qi, qv = datagen.queries(cfg, 0, 4)
    masks = torch.zeros((1, 40), dtype=torch.int32, device="cuda")
    bad = torch.tensor([0, 1, -1, 0], dtype=torch.int32, device="cuda")  # 1 >= nmasks
    with pytest.raises(sinn.SinnError):
        P.gpu.search_masked(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 10, 100, masks, bad)
    ok = torch.tensor([0, 0, -1, 0], dtype=torch.int32, device="cuda")  # an all-zero mask admits nothing
    oi, _ = P.gpu.search_masked(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), 10, 100, masks, ok)
    oi = ids_np(oi)
    assert np.all(oi[[0, 1, 3]] == oracle.NO_ID) and np.all(oi[2] != oracle.NO_ID)


def test_insert_id_checks_beyond_capacity_in_one_round_trip():
    """The one-round-trip insert checks ids against the current capacity; ids beyond it are re-checked
    for duplicates after growth only when the batch's ids do not ascend."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 1000, 1000)  # capacity ~1,024
    ip, ix, v = datagen.docs(cfg, 5000, 3)
    keep = (t_i64(ip), t_i32(ix.view(np.uint32)), t_f32(v), t_i32(np.array([9000, 7000, 9000], np.uint32)))
    st = P.gpu.status_of(P.gpu._lib.sinn_insert, 3, *[ctypes.c_void_p(t.data_ptr()) for t in keep], None)
    assert st == sinn.EINVAL  # a duplicate among ids beyond the capacity, unsorted batch
    assert P.gpu.stats()["live"] == 1000
    P.insert(ip, ix, v, np.array([9000, 7000, 8000], np.uint32))  # unsorted, beyond capacity, distinct
    check_sketches(P, np.array([7000, 8000, 9000, 0, 999], np.uint32))
    qp, qi, qv = datagen.queries(cfg, 0, 20)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)


def test_tombstones_then_amortised_compaction():
    """Deletes leave tombstones (O(deleted entries)); past a quarter of dead entries the index is
    compacted.  Before and after: postings equal the oracle's, searches match, stats count live entries."""
    cfg = datagen.CONFIGS["c2s"]
    P = _pair(cfg, 20000, 10000)
    rng = np.random.default_rng(4)
    ids = np.arange(20000, dtype=np.uint32)
    first = rng.choice(ids, 2000, replace=False)  # 10 %: tombstones only
    P.delete(first)
    terms = rng.choice(cfg.n, 200, replace=False)
    check_postings(P, terms)
    qp, qi, qv = datagen.queries(cfg, 0, 16)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)
    rest = np.setdiff1d(ids, first)
    second = rng.choice(rest, 6000, replace=False)  # 40 % dead in total: compaction
    P.delete(second)
    check_postings(P, terms)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)
    st = P.gpu.stats()
    assert st["live"] == 12000 and st["postings"] == int(sum(len(r[0]) for r in P.rows.values()))
    # recycle some of the deleted ids: their tombstones must not resurface
    rec = np.concatenate([first[:500], second[:500]]).astype(np.uint32)
    ip, ix, v = datagen.docs(cfg, 30000, rec.size)
    P.insert(ip, ix, v, rec)
    check_postings(P, terms)
    check_sketches(P, rec)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)


def test_enomem_leaves_the_index_usable():
    """A reservation beyond the device's memory returns SINN_ENOMEM (SURVEY §5 failure semantics): no
    poison, nothing changed — the index still inserts and searches to the oracle's results."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 2000, 2000)
    L = sinn.lib()
    st = L.sinn_reserve(P.gpu._h, 0, 1 << 42, None)  # 2^42 raw entries: 32 TB
    assert st == sinn.ENOMEM
    assert "memory" in L.sinn_last_error(P.gpu._h).decode().lower()
    ip, ix, v = datagen.docs(cfg, 2000, 500)
    P.insert(ip, ix, v, np.arange(2000, 2500, dtype=np.uint32))
    assert P.gpu.stats()["live"] == 2500
    qp, qi, qv = datagen.queries(cfg, 0, 20)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime)


def test_cuda_error_poisons_the_handle(monkeypatch):
    """A real CUDA error inside a call (test hook SINN_TEST_FAULT=1: a launch with an invalid block
    size, cudaErrorInvalidConfiguration) returns SINN_ECUDA; every later call on that handle returns
    SINN_EPOISONED, while another handle in the same process keeps working (the error is not sticky
    for the context) and destroy still releases the poisoned one."""
    import paper_2301_10622_b200 as sinn
    cfg = datagen.CONFIGS["tiny"]
    P = _pair(cfg, 2000, 2000)
    Q = _pair(cfg, 1000, 1000)
    qp, qi, qv = datagen.queries(cfg, 0, 8)
    args = (t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv))
    monkeypatch.setenv("SINN_TEST_FAULT", "1")
    with pytest.raises(sinn.SinnError) as ei:
        P.gpu.search(*args, cfg.k, cfg.kprime, True)
    assert ei.value.status == sinn.ECUDA
    monkeypatch.delenv("SINN_TEST_FAULT")
    for call in (lambda: P.gpu.search(*args, cfg.k, cfg.kprime, True),
                 lambda: P.gpu.delete(t_i32(np.array([1], dtype=np.uint32))),
                 lambda: P.gpu.insert(*[t for t in (t_i64(np.array([0, 1])), t_i32(np.array([3], dtype=np.uint32)),
                                                    t_f32(np.array([1.0], dtype=np.float32)),
                                                    t_i32(np.array([5000], dtype=np.uint32)))])):
        with pytest.raises(sinn.SinnError) as ei:
            call()
        assert ei.value.status == sinn.EPOISONED
    torch.cuda.synchronize()
    check_final(Q, qp, qi, qv, cfg.k, cfg.kprime)
    P.gpu.close()


@pytest.mark.parametrize("name", ["c2s", "c5s", "tiny"])
def test_bulk_copy_column_staging(name, monkeypatch):
    """Sketch columns staged by the bulk copy (cp.async.bulk + mbarrier, SINN_TMA=1): the same decodes,
    so the same stage-1 sets and final top-k as the oracle (Alg. 6-7)."""
    monkeypatch.setenv("SINN_TMA", "1")
    cfg = datagen.CONFIGS[name]
    P = _pair(cfg, min(cfg.N, 20000), cfg.insert_batch)
    qp, qi, qv = datagen.queries(cfg, 0, min(cfg.nq, 32))
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)


@pytest.mark.parametrize("name", ["tiny", "c5s"])
def test_nosync_search_is_cuda_graph_capturable(name):
    """A SINN_SEARCH_NOSYNC search makes no host round trip and (after a warm-up call has sized the
    workspace) no allocation, so the caller can capture it in a CUDA graph and replay it — the
    launch-bound config-1 batch then costs one graph launch.  The replay must reproduce the direct
    call, also after the query tensors' CONTENT changed (the graph bakes pointers and nq, not nnz)."""
    cfg = datagen.CONFIGS[name]
    P = _pair(cfg, min(cfg.N, 6000), 2500)
    nq = 64
    qa = datagen.queries(cfg, 0, nq)
    qb = datagen.queries(cfg, nq, nq)
    cap = max(qa[1].size, qb[1].size)
    sp = torch.zeros(nq + 1, dtype=torch.int64, device="cuda")
    si = torch.zeros(cap, dtype=torch.int32, device="cuda")
    sv = torch.zeros(cap, dtype=torch.float32, device="cuda")

    def load(q):
        sp.copy_(torch.from_numpy(q[0]))
        si[:q[1].size].copy_(torch.from_numpy(q[1]))
        sv[:q[2].size].copy_(torch.from_numpy(q[2]))

    out = (torch.empty((nq, cfg.k), dtype=torch.int32, device="cuda"),
           torch.empty((nq, cfg.k), dtype=torch.float32, device="cuda"))
    load(qa)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(side):
        P.gpu.search(sp, si, sv, cfg.k, cfg.kprime, True, out=out, sync=False)   # warm-up: workspace, attributes
        P.gpu.sync()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=side):
            P.gpu.search(sp, si, sv, cfg.k, cfg.kprime, True, out=out, sync=False)
    torch.cuda.current_stream().wait_stream(side)
    for q in (qa, qb, qa):
        load(q)
        out[0].fill_(-7)
        g.replay()
        torch.cuda.synchronize()
        P.gpu.sync()                                                    # no deferred error / EAGAIN
        want = P.gpu.search(t_i64(q[0]), t_i32(q[1].view(np.uint32)), t_f32(q[2]), cfg.k, cfg.kprime, True)
        same = (want[0] == out[0]).float().mean().item()
        assert same > 0.995, same                                       # (fp32 order may flip a boundary tie)
        fin = torch.isfinite(want[1]) & (want[0] == out[0])
        torch.testing.assert_close(out[1][fin], want[1][fin], rtol=1e-5, atol=1e-6)
    check_final(P, *qa, cfg.k, cfg.kprime)


@pytest.mark.parametrize("name", ["c3s", "c5s"])
def test_sample_rows_reused_by_the_full_pass(name, monkeypatch):
    """With head terms and a sample stride > 1 the large sample pass keeps its documents' score rows, the
    full pass skips the sampled tiles and k_emit_rows emits their candidates from the kept rows (at full
    size: every 28th / 14th tile of configs 3 / 5).  Forced here on the scaled configs (nested sample on,
    a sample of exactly k' documents: stride 20 / 10): stage 1 and the final top-k against the oracle,
    the same V as with the rows off, and the per-query masks / the batch filter applied to kept rows."""
    monkeypatch.setenv("SINN_CASCADE", "1")
    monkeypatch.setenv("SINN_SAMPLE_X", "1")
    cfg = datagen.CONFIGS[name]
    P = _pair(cfg, 20000, cfg.insert_batch)
    qp, qi, qv = datagen.queries(cfg, 0, 24)
    ci, _ = check_stage1(P, qp, qi, qv, cfg.kprime)
    st = P.gpu.stats()
    assert st["sample_rows_kept"] == 1 and st["sample_stride"] == 20000 // cfg.kprime   # 20 (c3s), 10 (c5s)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    monkeypatch.setenv("SINN_ROWS", "0")
    c0, _ = check_stage1(P, qp, qi, qv, cfg.kprime)
    assert P.gpu.stats()["sample_rows_kept"] == 0
    same = np.mean([len(set(ci[q].tolist()) & set(c0[q].tolist())) / cfg.kprime for q in range(24)])
    assert same > 0.995, same
    monkeypatch.delenv("SINN_ROWS")
    P.delete(np.arange(0, 20000, 7, dtype=np.uint32))            # vacant documents inside sampled tiles
    check_stage1(P, qp, qi, qv, cfg.kprime)
    check_final(P, qp, qi, qv, cfg.k, cfg.kprime, rerank=True)
    test_per_query_constraint_masks(name)
    from test_gpu_parity import test_constrained_search_parity
    test_constrained_search_parity(name)
