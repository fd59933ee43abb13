"""bench.py's roofline accounting against brute-force counts on a
small seeded batch: algorithmic id bytes, sketch bytes and Alg. 6's (document, query) updates."""
import numpy as np

import bench
import datagen


def _brute(cfg, N, nq):
    ip, ix, _ = datagen.docs(cfg, 0, N)
    term_len = np.bincount(ix, minlength=cfg.n)
    docs_of = [set(ix[ip[r]:ip[r + 1]].tolist()) for r in range(N)]
    qp, qi, qv = datagen.queries(cfg, 0, nq)
    return term_len, docs_of, qp, qi, qv


def test_updates_ids_and_sketch_bytes_match_brute_force():
    import dataclasses
    cfg = dataclasses.replace(datagen.CONFIGS["tiny"], N=2000)
    term_len, docs_of, qp, qi, qv = _brute(cfg, 2000, 40)
    alg = bench.algorithmic_bytes(cfg, term_len, qp, qi, qv, mean_doc_nnz=40.0)
    # Alg. 6 updates: for every query term with q_j != 0, one update per document holding j
    upd = 0
    for q in range(40):
        for e in range(qp[q], qp[q + 1]):
            if qv[e] != 0:
                upd += sum(1 for d in docs_of if int(qi[e]) in d)
    assert alg["updates"] == upd
    terms = {int(j) for j, v in zip(qi, qv) if v != 0}
    assert alg["ids"] == 4.0 * sum(int(term_len[j]) for j in terms)
    pos = {int(j) for j, v in zip(qi, qv) if v > 0}
    neg = {int(j) for j, v in zip(qi, qv) if v < 0}
    gather = 4.0 * cfg.h * (sum(int(term_len[j]) for j in pos) + sum(int(term_len[j]) for j in neg))
    stream = 4.0 * cfg.m * cfg.N * (int(bool(pos)) + int(bool(neg)))
    assert alg["sketch"] == min(gather, stream)
    assert alg["rerank"] == 40 * cfg.kprime * (8.0 * 40.0 + 8.0)


def test_upper_only_counts_positive_query_values_only():
    import dataclasses
    cfg = dataclasses.replace(datagen.CONFIGS["tiny"], N=1000, upper_only=True)
    term_len, docs_of, qp, qi, qv = _brute(cfg, 1000, 20)
    alg = bench.algorithmic_bytes(cfg, term_len, qp, qi, qv, mean_doc_nnz=40.0)
    upd = sum(int(term_len[int(qi[e])]) for q in range(20) for e in range(qp[q], qp[q + 1]) if qv[e] > 0)
    assert alg["updates"] == upd
    alg_bf = bench.algorithmic_bytes(cfg, term_len, qp, qi, qv, mean_doc_nnz=40.0, cell_bytes=2)
    assert alg_bf["sketch"] == alg["sketch"] / 2


def test_insert_algorithmic_bytes():
    """SURVEY §8(d) "Insert": 20 B per entry (8 in, 4 postings, 8 raw) + 4 m sides + 4 B per document."""
    c5 = datagen.CONFIGS["c5"]
    assert bench.insert_alg_bytes(c5, 250 * 10, 10) == 250 * 10 * 20 + 10 * (4 * 256 * 2 + 4)
    c3 = datagen.CONFIGS["c3"]  # Sinnamon+: one sketch side
    assert bench.insert_alg_bytes(c3, 120, 1) == 120 * 20 + 4 * 64 + 4
