"""Helpers for the GPU-vs-oracle parity tests (tests may import both sides; nothing else does).

Parity protocol:
  sketches / postings / decodes  bit-exact
  approximate scores             |s_gpu - s_orc| <= 1e-5 * M + 1e-30, M = sum_j |q_j e_ij|  (R7)
  stage-1 sets V                 may differ only in ids whose oracle score is within tol of the
                                 oracle's k'-th score
  final top-k                    equals the oracle's exact re-rank of V_gpu, up to ties within tol
"""
import numpy as np
import torch

import datagen
import oracle
import paper_2301_10622_b200 as sinn

REL = 1e-5


def t_i64(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int64)).cuda()


def t_i32(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a).astype(np.uint32).view(np.int32))).cuda()


def t_f32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def ids_np(t):
    return t.cpu().numpy().view(np.uint32)


class Pair:
    """The same index built on both sides from the same seeded rows; keeps the rows for masses."""

    def __init__(self, cfg, table=None, bf16=False, containers=False):
        self.cfg = cfg
        self.table = datagen.hash_table(cfg) if table is None else table
        self.gpu = sinn.Index(cfg.n, cfg.m, cfg.h, self.table, cfg.upper_only, bf16=bf16, containers=containers)
        self.orc = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, self.table, cfg.upper_only, bf16=bf16)
        self.rows = {}  # id -> (idx, val)

    def insert(self, ip, ix, v, ids, host=False):
        ids = np.asarray(ids, np.uint32)
        assert self.orc.insert(ip, ix, v, ids) == oracle.OK
        if host:
            self.gpu.insert_host(ip, ix, v, ids)
        else:
            self.gpu.insert(t_i64(ip), t_i32(ix.view(np.uint32)), t_f32(v), t_i32(ids))
        for r, i in enumerate(ids):
            self.rows[int(i)] = (ix[ip[r]:ip[r + 1]].copy(), v[ip[r]:ip[r + 1]].copy())

    def delete(self, ids):
        ids = np.asarray(ids, np.uint32)
        assert self.orc.delete(ids) == oracle.OK
        self.gpu.delete(t_i32(ids))
        for i in ids:
            del self.rows[int(i)]

    def exact_mass(self, ids, qi, qv):
        qd = {int(j): abs(float(q)) for j, q in zip(qi, qv)}
        out = np.zeros(len(ids))
        for t, i in enumerate(ids):
            if int(i) == oracle.NO_ID or int(i) not in self.rows:
                continue
            cols, vals = self.rows[int(i)]
            out[t] = sum(qd.get(int(j), 0.0) * abs(float(x)) for j, x in zip(cols, vals))
        return out


def check_sketches(P: Pair, ids):
    ids = np.asarray(ids, np.uint32)
    U, L = P.gpu.export_sketch(t_i32(ids))
    oU, oL = P.orc.sketch(ids)
    np.testing.assert_array_equal(U.cpu().numpy(), oU)
    if L is not None:
        np.testing.assert_array_equal(L.cpu().numpy(), oL)


def check_postings(P: Pair, terms):
    for j in terms:
        g = np.sort(ids_np(P.gpu.export_postings(int(j))))
        o = P.orc.postings(int(j))
        np.testing.assert_array_equal(g, o, err_msg=f"term {j}")
        assert np.all(np.diff(ids_np(P.gpu.export_postings(int(j))).astype(np.int64)) > 0)  # sorted, unique


def check_stage1(P: Pair, qp, qi, qv, kprime):
    """Stage-1 candidates and approximate scores vs the oracle's Alg. 6 scores (R7 tolerance)."""
    ci, cs = P.gpu.search_stage1(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), kprime)
    ci, cs = ids_np(ci), cs.cpu().numpy()
    nq = qp.size - 1
    for q in range(nq):
        a, b = qp[q], qp[q + 1]
        s, mass = P.orc.scores(qi[a:b], qv[a:b])
        live = np.isfinite(s)
        nlive = int(live.sum())
        take = min(kprime, nlive)
        gids = ci[q][:take]
        assert np.all(ci[q][take:] == oracle.NO_ID) and np.all(np.isneginf(cs[q][take:]))
        assert np.unique(gids).size == take and np.all(live[gids])
        tol = REL * mass + 1e-30
        np.testing.assert_array_less(np.abs(cs[q][:take] - s[gids]), tol[gids] + 1e-30)
        assert np.all(np.diff(cs[q][:take]) <= 0)  # best first
        if take == 0:
            continue
        order = np.lexsort((np.arange(s.size), -s))
        kth = s[order[take - 1]]
        oset = set(order[:take].tolist())
        for i in set(gids.tolist()) ^ oset:
            assert abs(s[i] - kth) <= tol[i] + REL * abs(mass[order[take - 1]]), (q, i, s[i], kth)
    return ci, cs


def check_final(P: Pair, qp, qi, qv, k, kprime, rerank=True, host=False):
    """Final top-k vs the oracle's re-rank of V_gpu (or the top-k of V_gpu by approximate score).
    V_gpu comes from a separate stage-1 call; fp32 atomics may flip k'-boundary ties between calls,
    so a returned id outside V_gpu is accepted only if its oracle score ties the k'-th (R7)."""
    nq = qp.size - 1
    if host:
        oi, os_ = P.gpu.search_host(qp, qi, qv, k, kprime, rerank)
    else:
        oi, os_ = P.gpu.search(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), k, kprime, rerank)
        oi, os_ = ids_np(oi), os_.cpu().numpy()
    ci, _ = P.gpu.search_stage1(t_i64(qp), t_i32(qi.view(np.uint32)), t_f32(qv), kprime)
    ci = ids_np(ci)
    for q in range(nq):
        a, b = qp[q], qp[q + 1]
        s, smass = P.orc.scores(qi[a:b], qv[a:b])
        V = ci[q][ci[q] != oracle.NO_ID]
        take = min(k, V.size)
        got = oi[q][:take]
        assert np.all(oi[q][take:] == oracle.NO_ID) and np.all(np.isneginf(os_[q][take:]))
        assert np.unique(got).size == take and all(P.orc.is_live(int(i)) for i in got)
        U = np.union1d(V, got).astype(np.uint32)
        if rerank:
            ex = np.array([P.orc.exact_dot(int(i), qi[a:b], qv[a:b]) for i in U])
            mass = P.exact_mass(U, qi[a:b], qv[a:b])
        else:
            ex, mass = s[U], smass[U]
        pos = {int(i): t for t, i in enumerate(U)}
        gi = np.array([pos[int(i)] for i in got], np.int64)
        np.testing.assert_array_less(np.abs(os_[q][:take] - ex[gi]), REL * mass[gi] + 1e-30)
        vi = np.array([pos[int(i)] for i in V], np.int64)
        order = vi[np.lexsort((V, -ex[vi]))][:take]
        want = U[order]
        if take == 0:
            continue
        kth = ex[order[-1]]
        kp_order = np.lexsort((np.arange(s.size), -s))
        kp_th = s[kp_order[min(kprime, int(np.isfinite(s).sum())) - 1]]
        for i in set(got.tolist()) ^ set(want.tolist()):
            t = pos[int(i)]
            in_tie = abs(ex[t] - kth) <= REL * (mass[t] + mass[order[-1]]) + 1e-30
            at_kp_boundary = abs(s[int(i)] - kp_th) <= REL * 2 * smass[int(i)] + 1e-30
            assert in_tie or at_kp_boundary, (q, int(i), ex[t], kth)
    return oi, os_
