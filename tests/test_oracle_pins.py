"""Pins of the CPU oracle against what the paper and the mathematics fix (no GPU).

Each test names the pin and the passage it follows.
The oracle is never compared with itself: expected values come from the paper's printed
tables (tests/golden/), closed forms, invariants, textbook special cases, or brute force
written independently in numpy on tiny inputs.
"""
import math

import numpy as np
import pytest

import datagen
import oracle
from oracle import analysis
from testutil import read_golden

TINY = datagen.CONFIGS["tiny"]


def build_oracle(cfg, N=None, ids=None, table=None):
    N = cfg.N if N is None else N
    ip, ix, v = datagen.docs(cfg, 0, N)
    table = datagen.hash_table(cfg) if table is None else table
    X = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, cfg.upper_only)
    ids = np.arange(N, dtype=np.uint32) if ids is None else ids
    assert X.insert(ip, ix, v, ids) == oracle.OK
    return X, (ip, ix, v), table


def decode_all(X, rows, ids):
    """(x, U-decode, L-decode) for every active coordinate of every row."""
    ip, ix, v = rows
    xs, us, ls, js = [], [], [], []
    for r in range(ids.size):
        for e in range(ip[r], ip[r + 1]):
            js.append(ix[e]); xs.append(v[e])
            us.append(X.decode(int(ids[r]), int(ix[e]), True))
            ls.append(X.decode(int(ids[r]), int(ix[e]), False))
    return np.array(xs, np.float32), np.array(us, np.float32), np.array(ls, np.float32)


# ---------------------------------------------------------------- SPEC / paper worked examples
def test_collision_example_max_min():
    """Two coordinates colliding in one bucket with 0.5 and 2.0 -> u = 2.0, l = 0.5 (Alg. 5 l.5-6)."""
    table = np.array([3, 3, 1], np.int32)  # n=3, h=1: coords 0 and 1 share bucket 3
    u, l = oracle.sketch_row(4, 1, table, [0, 1], [0.5, 2.0])
    assert u[3] == 2.0 and l[3] == 0.5
    assert u[0] == -np.inf and l[0] == np.inf and u[1] == -np.inf  # identity elements in untouched cells (R1)


def test_decode_least_upper_bound_example():
    """h=2, the two mapped upper cells hold 2.0 and 1.5 for a true 1.5 -> decode 1.5."""
    table = np.array([0, 1, 0, 2, 1, 3], np.int32)  # n=3,h=2: coord0->{0,1}, coord1->{0,2}, coord2->{1,3}
    X = oracle.OracleIndex(3, 4, 2, table)
    # coord0=1.5 (cells 0,1), coord1=2.0 (cells 0,2), coord2=1.0 (cells 1,3): U[0]=2.0, U[1]=1.5
    assert X.insert([0, 3], [0, 1, 2], [1.5, 2.0, 1.0], [0]) == oracle.OK
    assert X.decode(0, 0, True) == 1.5
    assert X.decode(0, 0, False) == 1.5    # greatest lower bound: max(L[0]=1.5, L[1]=1.0)


def test_decode_least_upper_bound_exact_cells():
    table = np.array([0, 1, 0, 2, 1, 3], np.int32)
    X = oracle.OracleIndex(3, 4, 2, table)
    assert X.insert([0, 3], [0, 1, 2], [1.5, 2.0, 1.0], [0]) == oracle.OK
    U, L = X.sketch([0])
    np.testing.assert_array_equal(U[0], [2.0, 1.5, 2.0, 1.0])
    np.testing.assert_array_equal(L[0], [1.5, 1.0, 2.0, 1.0])
    assert X.decode(0, 2, True) == 1.0 and X.decode(0, 1, True) == 2.0


def test_find_largest_examples():
    """Alg. 3: strict '> theta' admission; boundary ties keep the earlier-scanned id (R10)."""
    ids, sc = oracle.find_largest([0.5, 2.0, 1.0], np.arange(3), 2)
    assert list(ids) == [1, 2] and list(sc) == [2.0, 1.0]
    ids, _ = oracle.find_largest(np.zeros(5), np.arange(5), 2)
    assert list(ids) == [0, 1]
    ids, _ = oracle.find_largest([1.0], [0], 3)
    assert list(ids) == [0]


def test_find_largest_vs_full_sort():
    """FindLargest == full sort by (score desc, id asc), including heavy ties (numpy lexsort)."""
    rng = np.random.default_rng(7)
    for trial in range(20):
        n = int(rng.integers(1, 3000))
        k = int(rng.integers(1, 200))
        s = rng.integers(-5, 6, n).astype(np.float64) if trial % 2 else rng.normal(size=n)
        ids = rng.permutation(n).astype(np.uint32)
        got_i, got_s = oracle.find_largest(s, ids, k)
        order = np.lexsort((ids, -s))[:k]
        np.testing.assert_array_equal(got_i, ids[order])
        np.testing.assert_array_equal(got_s, s[order])


def test_exact_dot_example():
    """<a, b> over the intersection of supports: a={1:2,5:-1}, b={1:0.5,5:4} -> -3 (Eq. 2)."""
    X = oracle.OracleIndex(8, 4, 1, np.zeros(8, np.int32))
    assert X.insert([0, 2, 3], [1, 5, 2], [0.5, 4.0, 3.0], [0, 1]) == oracle.OK
    assert X.exact_dot(0, [1, 5], [2.0, -1.0]) == -3.0
    assert X.exact_dot(1, [1], [2.0]) == 0.0  # disjoint supports


# ---------------------------------------------------------------- sketch pins O1-O4
def test_O1_sandwich_and_O2_extremes():
    """O1: L-decode <= x <= U-decode for every active coordinate (P:486 'Clearly ... always holds').
    O2: the largest value of a vector decodes exactly from U, the smallest from L."""
    N = 2000
    X, rows, _ = build_oracle(TINY, N)
    ids = np.arange(N, dtype=np.uint32)
    x, u, l = decode_all(X, rows, ids)
    assert np.all(l <= x) and np.all(x <= u)
    assert np.mean(u > x) > 0.05  # the sketch is lossy at this (m, h): the pin is not vacuous
    ip, ix, v = rows
    for r in range(N):
        a, b = ip[r], ip[r + 1]
        jmax, jmin = ix[a + np.argmax(v[a:b])], ix[a + np.argmin(v[a:b])]
        assert X.decode(r, int(jmax), True) == v[a:b].max()
        assert X.decode(r, int(jmin), False) == v[a:b].min()


def test_O3_bruteforce_collision_characterisation():
    """O3 (proof of the Theorem at): U-decode(i,j) == x_ij iff some bucket pi_o(j) receives no
    larger active value; L symmetric.  Checked by enumerating all colliding pairs in numpy."""
    rng = np.random.default_rng(3)
    n, m, h = 40, 8, 2
    table = rng.integers(0, m, n * h).astype(np.int32)
    X = oracle.OracleIndex(n, m, h, table)
    for i in range(200):
        nnz = int(rng.integers(1, 20))
        idx = np.sort(rng.choice(n, nnz, replace=False)).astype(np.int32)
        val = rng.normal(size=nnz).astype(np.float32)
        assert X.insert([0, nnz], idx, val, [i]) == oracle.OK
        buckets = [set(table[j * h:(j + 1) * h]) for j in idx]
        for a in range(nnz):
            free_up = free_lo = False
            for k in buckets[a]:
                others = [val[b] for b in range(nnz) if b != a and k in buckets[b]]
                free_up |= all(o <= val[a] for o in others)
                free_lo |= all(o >= val[a] for o in others)
            assert (X.decode(i, int(idx[a]), True) == val[a]) == free_up
            assert (X.decode(i, int(idx[a]), False) == val[a]) == free_lo


def test_O4_injective_table_decodes_exactly_and_scores_are_exact():
    """O4: with all n*h bucket ids distinct (m >= n h) nothing collides, so every decode equals x and
    Sinnamon's score equals the exact inner product (reduces to LinScan, Alg. 2)."""
    rng = np.random.default_rng(11)
    n, h = 300, 2
    m = n * h
    table = rng.permutation(m).astype(np.int32)
    X = oracle.OracleIndex(n, m, h, table)
    N = 500
    ip = np.zeros(N + 1, np.int64)
    ix, v = [], []
    for r in range(N):
        nnz = int(rng.integers(0, 30))
        ix.append(np.sort(rng.choice(n, nnz, replace=False)))
        v.append(rng.normal(size=nnz))
        ip[r + 1] = ip[r] + nnz
    ix = np.concatenate(ix).astype(np.int32)
    v = np.concatenate(v).astype(np.float32)
    assert X.insert(ip, ix, v, np.arange(N)) == oracle.OK
    for r in range(0, N, 7):
        for e in range(ip[r], ip[r + 1]):
            assert X.decode(r, int(ix[e]), True) == v[e] == X.decode(r, int(ix[e]), False)
    dense = np.zeros((N, n))
    for r in range(N):
        dense[r, ix[ip[r]:ip[r + 1]]] = v[ip[r]:ip[r + 1]]
    for t in range(20):
        qi = np.sort(rng.choice(n, 25, replace=False)).astype(np.int32)
        qv = rng.normal(size=25).astype(np.float32)
        s, _ = X.scores(qi, qv)
        assert np.all(np.isneginf(s[N:]))  # columns never inserted are vacant
        np.testing.assert_allclose(s[:N], dense[:, qi] @ qv.astype(np.float64), rtol=0, atol=1e-12)


# ---------------------------------------------------------------- scoring pins O5, O6, O9, O11
def test_O5_theorem1_and_O6_gap_identity():
    """O5 Theorem 1: score >= exact inner product for every (query, document).
    O6: score - exact == sum_j q_j (e_ij - x_ij) (sum over the same terms in the same order)."""
    N = 3000
    X, rows, _ = build_oracle(TINY, N)
    ip, ix, v = rows
    qp, qi, qv = datagen.queries(TINY, 0, 40)
    dense = np.zeros((N, TINY.n))
    for r in range(N):
        dense[r, ix[ip[r]:ip[r + 1]]] = v[ip[r]:ip[r + 1]]
    for q in range(40):
        a, b = qp[q], qp[q + 1]
        s, mass = X.scores(qi[a:b], qv[a:b])
        s, mass = s[:N], mass[:N]
        ex = dense[:, qi[a:b]] @ qv[a:b].astype(np.float64)
        assert np.all(s >= ex - 1e-12 * np.maximum(1.0, mass))
        assert np.mean(s > ex + 1e-9) > 0.01  # non-vacuous
        for r in range(0, N, 97):
            gap = 0.0
            for e in range(a, b):
                j = qi[e]
                if dense[r, j] == 0 and j not in ix[ip[r]:ip[r + 1]]:
                    continue
                d = X.decode(r, int(j), qv[e] > 0)
                gap += float(qv[e]) * (d - dense[r, j])
            assert abs((s[r] - ex[r]) - gap) <= 1e-9 * max(1.0, mass[r])


def _bruteforce_scores(n, m, h, table, ip, ix, v, qi, qv, upper_only=False, with_mass=False):
    """O9: dense numpy brute force of Alg. 5 + Alg. 6 on tiny inputs; with_mass also returns the
    R7 tolerance scale M_i = sum_j |q_j * e_ij| over the query's non-zero terms j in nz(x_i)."""
    N = ip.size - 1
    U = np.full((N, m), -np.inf)
    L = np.full((N, m), np.inf)
    active = np.zeros((N, n), bool)
    for r in range(N):
        cols = ix[ip[r]:ip[r + 1]]
        active[r, cols] = True
        for o in range(h):
            np.maximum.at(U[r], table[cols * h + o], v[ip[r]:ip[r + 1]].astype(np.float64))
            np.minimum.at(L[r], table[cols * h + o], v[ip[r]:ip[r + 1]].astype(np.float64))
    S = np.zeros(N)
    M = np.zeros(N)
    for j, q in zip(qi, qv):
        if q == 0:
            continue
        cells = table[j * h:(j + 1) * h]
        if q > 0:
            e = U[:, cells].min(axis=1)
        else:
            e = np.zeros(N) if upper_only else L[:, cells].max(axis=1)
        S += np.where(active[:, j], float(q) * e, 0.0)
        M += np.where(active[:, j], np.abs(float(q) * e), 0.0)
    return (S, M) if with_mass else S


@pytest.mark.parametrize("upper_only", [False, True])
def test_O9_tiny_bruteforce(upper_only):
    rng = np.random.default_rng(5)
    n, m, h, N = 60, 16, 3, 300
    table = rng.integers(0, m, n * h).astype(np.int32)
    ip = np.zeros(N + 1, np.int64)
    ixs, vs = [], []
    for r in range(N):
        nnz = int(rng.integers(0, 25))
        ixs.append(np.sort(rng.choice(n, nnz, replace=False)))
        val = rng.normal(size=nnz)
        vs.append(np.abs(val) if upper_only else val)
        ip[r + 1] = ip[r] + nnz
    ix = np.concatenate(ixs).astype(np.int32)
    v = np.concatenate(vs).astype(np.float32)
    X = oracle.OracleIndex(n, m, h, table, upper_only)
    assert X.insert(ip, ix, v, np.arange(N)) == oracle.OK
    for t in range(30):
        nq = int(rng.integers(1, 30))
        qi = np.sort(rng.choice(n, nq, replace=False)).astype(np.int32)
        qv = rng.normal(size=nq).astype(np.float32)
        qv[rng.random(nq) < 0.1] = 0.0
        s, mass = X.scores(qi, qv)
        s, mass = s[:N], mass[:N]
        ref, ref_mass = _bruteforce_scores(n, m, h, table, ip, ix, v, qi, qv, upper_only, with_mass=True)
        np.testing.assert_allclose(s, ref, rtol=1e-12, atol=1e-12)
        # R7's tolerance scale is pinned too: an inflated mass would make every GPU score check vacuous
        np.testing.assert_allclose(mass, ref_mass, rtol=1e-12, atol=1e-12)
        assert np.all(mass >= np.abs(s) - 1e-12)


def test_O11_upper_only_equals_full_on_nonnegative():
    """O11: on non-negative documents and queries Sinnamon+ and Sinnamon score identically."""
    cfg = datagen.CONFIGS["c3s"]
    N = 4000
    ip, ix, v = datagen.docs(cfg, 0, N)
    table = datagen.hash_table(cfg)
    A = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, True)
    B = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table, False)
    assert A.insert(ip, ix, v, np.arange(N)) == oracle.OK
    assert B.insert(ip, ix, v, np.arange(N)) == oracle.OK
    qp, qi, qv = datagen.queries(cfg, 0, 10)
    for q in range(10):
        sa, _ = A.scores(qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]])
        sb, _ = B.scores(qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]])
        np.testing.assert_array_equal(sa, sb)
    assert A.insert([0, 1], [0], [-1.0], [N]) == oracle.EINVAL  # negative value rejected under Sinnamon+


# ---------------------------------------------------------------- ranking pin O10, search semantics
def test_O10_kprime_all_gives_exact_topk():
    """O10 (Alg. 7): re-ranking every live document returns the exact top-k, i.e. the
    brute-force dense MIPS answer (ties by ascending id)."""
    N = 1500
    X, rows, _ = build_oracle(TINY, N)
    ip, ix, v = rows
    dense = np.zeros((N, TINY.n))
    for r in range(N):
        dense[r, ix[ip[r]:ip[r + 1]]] = v[ip[r]:ip[r + 1]]
    qp, qi, qv = datagen.queries(TINY, 0, 30)
    ids, sc = X.search(qp, qi, qv, k=10, kprime=N, rerank=True)
    eids, esc = X.exact(qp, qi, qv, k=10)
    for q in range(30):
        ex = dense[:, qi[qp[q]:qp[q + 1]]] @ qv[qp[q]:qp[q + 1]].astype(np.float64)
        order = np.lexsort((np.arange(N), -ex))[:10]
        np.testing.assert_array_equal(ids[q], order)
        np.testing.assert_array_equal(eids[q], order)
        np.testing.assert_allclose(sc[q], ex[order], rtol=0, atol=1e-12)


def test_search_stage1_is_topkprime_of_scores_and_rerank_off():
    N = 2000
    X, rows, _ = build_oracle(TINY, N)
    qp, qi, qv = datagen.queries(TINY, 0, 8)
    ids, sc, cid, csc, cms = X.search(qp, qi, qv, k=10, kprime=100, rerank=False, with_candidates=True)
    for q in range(8):
        s, ms = X.scores(qi[qp[q]:qp[q + 1]], qv[qp[q]:qp[q + 1]])
        s, ms = s[:N], ms[:N]
        order = np.lexsort((np.arange(N), -s))[:100]
        np.testing.assert_array_equal(cid[q], order)
        np.testing.assert_array_equal(csc[q], s[order])
        np.testing.assert_array_equal(cms[q], ms[order])
        np.testing.assert_array_equal(ids[q], order[:10])


def test_search_padding_and_argument_checks():
    X = oracle.OracleIndex(10, 4, 1, np.zeros(10, np.int32))
    assert X.insert([0, 1, 2], [1, 2], [1.0, 2.0], [0, 5]) == oracle.OK
    ids, sc = X.search([0, 1], [1], [1.0], k=4, kprime=4)
    assert list(ids[0][:2]) == [0, 5] and list(ids[0][2:]) == [oracle.NO_ID] * 2
    assert np.all(np.isneginf(sc[0][2:]))
    with pytest.raises(ValueError):
        X.search([0, 1], [1], [1.0], k=5, kprime=4)       # k' < k
    with pytest.raises(ValueError):
        X.search([0, 2], [3, 3], [1.0, 1.0], k=1, kprime=1)  # indices not strictly increasing
    with pytest.raises(ValueError):
        X.search([0, 1], [10], [1.0], k=1, kprime=1)       # index out of range


# ---------------------------------------------------------------- insert/delete semantics, O12
def test_insert_validation_is_all_or_nothing():
    X = oracle.OracleIndex(10, 4, 1, np.arange(10, dtype=np.int32) % 4)
    assert X.insert([0, 1], [3], [1.0], [7]) == oracle.OK
    before = X.postings(3).copy()
    assert X.insert([0, 1, 2], [3, 4], [1.0, 2.0], [1, 7]) == oracle.EEXIST   # live id
    assert X.insert([0, 1, 2], [3, 4], [1.0, 2.0], [1, 1]) == oracle.EINVAL   # duplicate in batch
    assert X.insert([0, 2], [4, 4], [1.0, 2.0], [2]) == oracle.EINVAL         # not strictly increasing
    assert X.insert([0, 1], [10], [1.0], [2]) == oracle.EINVAL                # out of range
    assert X.insert([0, 1], [1], [np.nan], [2]) == oracle.EINVAL              # non-finite
    assert X.insert([0, 1], [1], [1.0], [oracle.NO_ID]) == oracle.EINVAL      # reserved padding id
    np.testing.assert_array_equal(X.postings(3), before)
    assert X.live_count == 1 and not X.is_live(1)
    assert X.delete([3]) == oracle.ENOTFOUND and X.delete([7, 7]) == oracle.EINVAL
    assert X.live_count == 1


def test_O12_postings_equal_recomputation_under_streaming_with_recycling():
    """O12: after any insert/delete sequence, I[j] == {live i : j in nz(x_i)},
    recomputed from the inserted rows kept by the test; recycled ids overwrite their columns."""
    cfg = datagen.CONFIGS["c4s"]
    table = datagen.hash_table(cfg)
    X = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, table)
    rows_of = {}
    free, next_id, gen = [], 0, 0
    rng = np.random.default_rng(0)
    for rnd in range(6):
        B = 700
        ip, ix, v = datagen.docs(cfg, gen, B)
        gen += B
        ids = []
        for _ in range(B):
            if free:
                ids.append(free.pop())
            else:
                ids.append(next_id); next_id += 1
        ids = np.array(ids, np.uint32)
        assert X.insert(ip, ix, v, ids) == oracle.OK
        for r, i in enumerate(ids):
            rows_of[int(i)] = (ix[ip[r]:ip[r + 1]].copy(), v[ip[r]:ip[r + 1]].copy())
        live = np.array(sorted(rows_of), np.uint32)
        dele = rng.choice(live, live.size // 10, replace=False)
        assert X.delete(dele) == oracle.OK
        for i in dele:
            del rows_of[int(i)]
        free.extend(int(i) for i in dele)
    assert next_id == max(rows_of) + 1 or next_id > max(rows_of)
    expect = {}
    for i, (cols, _) in rows_of.items():
        for j in cols:
            expect.setdefault(int(j), []).append(i)
    for j in range(cfg.n):
        np.testing.assert_array_equal(X.postings(j), np.array(sorted(expect.get(j, [])), np.uint32))
    # recycled columns hold the new vector's sketch: O1 sandwich on every live vector
    for i, (cols, vals) in list(rows_of.items())[:300]:
        for j, x in zip(cols, vals):
            assert X.decode(i, int(j), False) <= x <= X.decode(i, int(j), True)
    assert X.live_count == len(rows_of)


def test_deleted_ids_never_returned():
    N = 1000
    X, rows, _ = build_oracle(TINY, N)
    dele = np.arange(0, N, 3, dtype=np.uint32)
    assert X.delete(dele) == oracle.OK
    qp, qi, qv = datagen.queries(TINY, 0, 20)
    ids, _ = X.search(qp, qi, qv, k=10, kprime=N, rerank=True)
    assert not np.isin(ids, dele).any()
    eids, _ = X.exact(qp, qi, qv, k=10)
    assert not np.isin(eids, dele).any()


# ---------------------------------------------------------------- analysis pins O7, O8
def test_O8_closed_form_matches_table1_and_quadrature():
    """O8: Eq. reproduces Table 1 (golden file) within its 2-digit rounding, and equals
    the general Eq. integrated numerically with a Gaussian and a uniform density."""
    rows = read_golden("table1_prob_error.txt")
    cells = [(m, h) for m in (60, 120, 240) for h in (1, 2, 3)]
    for name, printed in rows.items():
        for (m, h), p in zip(cells, printed):
            assert abs(analysis.p_error_gaussian(m, h, 119) - p) <= 0.0051, (name, m, h)
    for (m, h) in cells:
        cf = analysis.p_error_gaussian(m, h, 119)
        assert abs(analysis.p_error_general(m, h, 119, *analysis.gaussian(1.0)) - cf) < 1e-6
        assert abs(analysis.p_error_general(m, h, 119, *analysis.uniform_pm1()) - cf) < 1e-6
    # h = 1 special case, Lemma in Appendix A: 1 - m/((n-1)p) (1 - e^{-(n-1)p/m})
    for m in (60, 120, 240):
        assert abs(analysis.p_error_gaussian(m, 1, 119) - (1 - m / 119 * (1 - math.exp(-119 / m)))) < 1e-15


def test_table2_expected_error_rows():
    """Lemma reproduces Table 2's Uniform and Gaussian(sigma=0.1) rows."""
    rows = read_golden("table2_expected_error.txt")
    dens = {"uniform_pm1": analysis.uniform_pm1(), "gaussian_sigma0.1": analysis.gaussian(0.1)}
    cells = [(m, h) for m in (60, 120, 240) for h in (1, 2, 3)]
    for name, printed in rows.items():
        for (m, h), p in zip(cells, printed):
            # 2-digit rounding (0.005) + 0.002 slack for the paper's own numerical integration
            assert abs(analysis.expected_error_general(m, h, 119, *dens[name]) - p) <= 0.007, (name, m, h)


@pytest.mark.parametrize("m,h", [(60, 1), (60, 3), (120, 2), (240, 1), (240, 3)])
def test_O7_monte_carlo_sketch_vs_table1(m, h):
    """O7: the oracle's sketch over-estimates an active N(0,1) coordinate with the probability of
    Table 1 (psi_d = 120) — Monte Carlo over 1500 vectors with exactly 120 active coordinates."""
    n = 200_000
    spec = datagen.VecSpec(n, datagen.NNZ_FIXED, 120, 0, 120, 120)
    ip, ix, v = datagen.rows(spec, 99 + m * 10 + h, 1, 0, 1500)
    table = datagen.table(n, h, m, 1234 + h)
    over, total = 0, 0
    for r in range(1500):
        idx, val = ix[ip[r]:ip[r + 1]], v[ip[r]:ip[r + 1]]
        u, _ = oracle.sketch_row(m, h, table, idx, val, lower=False)
        dec = u[table.reshape(n, h)[idx]].min(axis=1)
        over += int((dec > val).sum()); total += idx.size
    rate = over / total
    assert abs(rate - analysis.p_error_gaussian(m, h, 119)) < 0.012


def test_O7_config_rate_matches_nnz_weighted_closed_form():
    """O7 at config-1 parameters (m=64, h=2, psi_d ~ U{20..60}): measured rate vs the nnz-weighted
    closed form, within 0.01 (0.2455 simulated vs 0.2403)."""
    N = 4000
    X, rows, _ = build_oracle(TINY, N)
    x, u, _ = decode_all(X, rows, np.arange(N, dtype=np.uint32))
    ip = rows[0]
    rate = float(np.mean(u > x))
    assert abs(rate - analysis.p_error_mixture(TINY.m, TINY.h, np.diff(ip))) < 0.01


def test_anytime_budget_pins():
    """Anytime budget (Alg. 6 with T; R20: T counts query terms in the |q_j|-descending
    order).  Pins: a budget >= nnz(q) reproduces the unbudgeted scores exactly; a budget of 1 gives exactly
    q_j * decode for the single largest-|q_j| term (every other document 0); each budget's scores are the
    prefix sums of per-term contributions (budget b+1 - budget b = one term)."""
    N = 1500
    X, rows, _ = build_oracle(TINY, N)
    qp, qi, qv = datagen.queries(TINY, 0, 6)
    for q in range(6):
        a, b = qp[q], qp[q + 1]
        idx, val = qi[a:b], qv[a:b]
        full, _ = X.scores(idx, val)
        s_all, _ = X.scores(idx, val, max_terms=idx.size + 3)
        np.testing.assert_array_equal(s_all, full)
        order = sorted(range(idx.size), key=lambda e: (-abs(float(val[e])), int(idx[e])))
        j0, v0 = int(idx[order[0]]), float(val[order[0]])
        s1, _ = X.scores(idx, val, max_terms=1)
        want = np.where(np.arange(s1.size) < N, 0.0, -np.inf)  # capacity beyond N: vacant columns
        for i in X.postings(j0):
            want[i] = v0 * X.decode(int(i), j0, v0 > 0)
        np.testing.assert_array_equal(s1, want)
        prev = s1
        for bud in range(2, idx.size + 1):
            cur, _ = X.scores(idx, val, max_terms=bud)
            jb, vb = int(idx[order[bud - 1]]), float(val[order[bud - 1]])
            delta = np.zeros(N)
            for i in X.postings(jb):
                delta[i] = vb * X.decode(int(i), jb, vb > 0)
            np.testing.assert_allclose(cur[:N] - prev[:N], delta, rtol=0, atol=1e-12)
            prev = cur


def test_constrained_search_equals_deleting_masked_documents():
    """Constrained search (Eq. 3: masked-out columns leave the solution set): the filtered result
    over the full index equals the unfiltered result over an index from which the masked-out documents were
    deleted (the deletion protocol, is pinned by O12); an all-ones mask changes nothing; an
    all-zeros mask returns nothing."""
    N = 2000
    X, rows, table = build_oracle(TINY, N)
    rng = np.random.default_rng(5)
    allowed = rng.random(N) < 0.4
    words = np.zeros((N + 31) // 32, np.uint32)
    for i in np.flatnonzero(allowed):
        words[i >> 5] |= np.uint32(1 << (i & 31))
    qp, qi, qv = datagen.queries(TINY, 0, 20)
    fid, fsc = X.search_filtered(qp, qi, qv, 10, 100, words)
    Y, _, _ = build_oracle(TINY, N, table=table)
    assert Y.delete(np.flatnonzero(~allowed).astype(np.uint32)) == oracle.OK
    did, dsc = Y.search(qp, qi, qv, 10, 100)
    np.testing.assert_array_equal(fid, did)
    np.testing.assert_array_equal(fsc, dsc)
    aid, asc = X.search_filtered(qp, qi, qv, 10, 100, np.full_like(words, 0xFFFFFFFF))
    uid, usc = X.search(qp, qi, qv, 10, 100)
    np.testing.assert_array_equal(aid, uid)
    zid, _ = X.search_filtered(qp, qi, qv, 10, 100, np.zeros_like(words))
    assert np.all(zid == oracle.NO_ID)


# ---------------------------------------------------------------- F3: bfloat16 sketch cells (R21)
def _bf16_neighbours(x: np.ndarray):
    """torch's round-to-nearest-even bfloat16 of x and the next bfloat16 values above and below it
    (an independent library routine: the directed roundings are whichever of these brackets x)."""
    import torch
    t = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16)
    up = torch.nextafter(t, torch.full_like(t, float("inf")))
    dn = torch.nextafter(t, torch.full_like(t, float("-inf")))
    return t.float().numpy(), up.float().numpy(), dn.float().numpy()


def test_F3_directed_rounding_matches_library_bracketing():
    """bf16_up(x) is the smallest bfloat16 >= x and bf16_down(x) the largest <= x (R21): checked
    against torch's round-to-nearest bfloat16 and its neighbours, over normal, subnormal, signed,
    huge and already-representable values."""
    rng = np.random.default_rng(21)
    x = np.concatenate([
        rng.standard_normal(4000).astype(np.float32),
        (rng.standard_normal(1000) * 1e-39).astype(np.float32),        # subnormals
        (rng.standard_normal(1000) * 1e37).astype(np.float32),
        np.array([0.0, 1.0, -1.0, 3.0e38, -3.0e38, 1.0078125, -1.0078125,
                  np.finfo(np.float32).max, -np.finfo(np.float32).max], np.float32)])
    rne, nxt, prv = _bf16_neighbours(x)
    up = np.array([oracle.bf16_up(float(v)) for v in x], np.float32)
    dn = np.array([oracle.bf16_down(float(v)) for v in x], np.float32)
    exp_up = np.where(rne >= x, rne, nxt)
    exp_dn = np.where(rne <= x, rne, prv)
    np.testing.assert_array_equal(up, exp_up)
    np.testing.assert_array_equal(dn, exp_dn)
    assert np.all(up >= x) and np.all(dn <= x)
    assert np.all((up.view(np.uint32) & 0xFFFF) == 0) and np.all((dn.view(np.uint32) & 0xFFFF) == 0)
    assert np.isposinf(oracle.bf16_up(float(np.finfo(np.float32).max)))   # no bfloat16 >= it but +inf
    assert oracle.bf16_up(float("-inf")) == float("-inf") and oracle.bf16_down(float("inf")) == float("inf")


def _bf16_index(cfg, N, bf16, upper_only=None):
    ip, ix, v = datagen.docs(cfg, 0, N)
    X = oracle.OracleIndex(cfg.n, cfg.m, cfg.h, datagen.hash_table(cfg),
                           cfg.upper_only if upper_only is None else upper_only, bf16=bf16)
    assert X.insert(ip, ix, v, np.arange(N, dtype=np.uint32)) == oracle.OK
    return X, (ip, ix, v)


def test_F3_bf16_sketch_sandwich_and_theorem1():
    """With bfloat16 cells the decodes still bound x from the correct side (O1) and every score is
    >= the exact inner product (Theorem 1); the bfloat16 index is never tighter than
    the fp32 one."""
    N = 2000
    Xb, rows = _bf16_index(TINY, N, True)
    Xf, _ = _bf16_index(TINY, N, False)
    ids = np.arange(N, dtype=np.uint32)
    x, u, l = decode_all(Xb, rows, ids)
    _, uf, lf = decode_all(Xf, rows, ids)
    assert np.all(l <= x) and np.all(x <= u)
    assert np.all(u >= uf) and np.all(l <= lf)
    assert np.any(u > uf)  # non-vacuous: rounding happened
    ip, ix, v = rows
    dense = np.zeros((N, TINY.n))
    for r in range(N):
        dense[r, ix[ip[r]:ip[r + 1]]] = v[ip[r]:ip[r + 1]]
    qp, qi, qv = datagen.queries(TINY, 0, 20)
    for q in range(20):
        a, b = qp[q], qp[q + 1]
        s, mass = Xb.scores(qi[a:b], qv[a:b])
        ex = dense[:, qi[a:b]] @ qv[a:b].astype(np.float64)
        assert np.all(s[:N] >= ex - 1e-12 * np.maximum(1.0, mass[:N]))


def test_F3_bf16_cells_are_directed_roundings_of_the_exact_extremes():
    """Cell by cell: the bfloat16 U (L) cell is the fp32 max (min) rounded up (down); sentinels
    (untouched cells, -inf / +inf) are unchanged."""
    N = 500
    Xb, _ = _bf16_index(TINY, N, True)
    Xf, _ = _bf16_index(TINY, N, False)
    ids = np.arange(N, dtype=np.uint32)
    Ub, Lb = Xb.sketch(ids)
    Uf, Lf = Xf.sketch(ids)
    rne, nxt, prv = _bf16_neighbours(Uf.ravel())
    np.testing.assert_array_equal(Ub.ravel(), np.where(rne >= Uf.ravel(), rne, nxt))
    rne, nxt, prv = _bf16_neighbours(Lf.ravel())
    np.testing.assert_array_equal(Lb.ravel(), np.where(rne <= Lf.ravel(), rne, prv))


def test_F3_bf16_equals_fp32_on_representable_values():
    """When every inserted value is a bfloat16 already, rounding is the identity: the bfloat16 index
    scores exactly like the fp32 one (special case reducing to the paper's fp32 Sinnamon)."""
    import torch
    N = 1500
    ip, ix, v = datagen.docs(TINY, 0, N)
    v = torch.from_numpy(v).to(torch.bfloat16).float().numpy()
    table = datagen.hash_table(TINY)
    ids = np.arange(N, dtype=np.uint32)
    Xb = oracle.OracleIndex(TINY.n, TINY.m, TINY.h, table, False, bf16=True)
    Xf = oracle.OracleIndex(TINY.n, TINY.m, TINY.h, table, False, bf16=False)
    assert Xb.insert(ip, ix, v, ids) == oracle.OK and Xf.insert(ip, ix, v, ids) == oracle.OK
    qp, qi, qv = datagen.queries(TINY, 0, 10)
    for q in range(10):
        a, b = qp[q], qp[q + 1]
        sb, _ = Xb.scores(qi[a:b], qv[a:b])
        sf, _ = Xf.scores(qi[a:b], qv[a:b])
        np.testing.assert_array_equal(sb, sf)
