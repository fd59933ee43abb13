"""Seeded input generators (host logic, no GPU): determinism, row independence, recipe sanity."""
import numpy as np

import datagen


def test_rows_are_pure_functions_of_seed_stream_row():
    cfg = datagen.CONFIGS["c3s"]
    ip, ix, v = datagen.docs(cfg, 0, 3000, nthreads=4)
    ip2, ix2, v2 = datagen.docs(cfg, 1000, 500, nthreads=1)
    a, b = ip[1000], ip[1500]
    np.testing.assert_array_equal(ix2, ix[a:b])
    np.testing.assert_array_equal(v2, v[a:b])
    ip3, ix3, v3 = datagen.docs(cfg, 0, 3000, nthreads=8)
    np.testing.assert_array_equal(ix3, ix)
    qp, qi, qv = datagen.queries(cfg, 0, 100)
    assert not np.array_equal(qi[:50], ix[:50])  # distinct streams


def test_rows_are_valid_csr():
    for name in ("tiny", "c2s", "c3s", "c5s"):
        cfg = datagen.CONFIGS[name]
        for ip, ix, v in (datagen.docs(cfg, 0, 2000), datagen.queries(cfg, 0, 200)):
            assert ip[0] == 0 and np.all(np.diff(ip) >= 0)
            assert ix.min() >= 0 and ix.max() < cfg.n
            for r in range(0, ip.size - 1, 7):
                assert np.all(np.diff(ix[ip[r]:ip[r + 1]]) > 0)
            assert np.all(np.isfinite(v))
            if cfg.upper_only:
                assert v.min() >= 0


def test_recipe_moments():
    c2 = datagen.CONFIGS["c2"]
    ip, ix, v = datagen.docs(c2, 0, 20000)
    nnz = np.diff(ip)
    assert abs(nnz.mean() - 120) < 0.5 and abs(nnz.var() - 120) < 8        # Poisson(120)
    assert abs(v.mean()) < 0.01 and abs(v.std() - 1) < 0.01                 # N(0,1)
    cnt = np.bincount(ix, minlength=c2.n)
    assert cnt.max() < 3 * cnt.mean()                                       # uniform coordinates
    tiny = datagen.CONFIGS["tiny"]
    nnz = np.diff(datagen.docs(tiny, 0, 5000)[0])
    assert nnz.min() == 20 and nnz.max() == 60
    assert np.all(np.diff(datagen.queries(tiny, 0, 100)[0]) == 10)
    c3 = datagen.CONFIGS["c3"]
    ip, ix, v = datagen.docs(c3, 0, 20000)
    nnz = np.diff(ip)
    assert nnz.min() >= 5 and nnz.max() <= 600 and abs(nnz.mean() - 120) < 2  # log-normal, mean ~120
    assert abs(np.median(v) - 1.0) < 0.03                                     # LogNormal(0,1) median e^0
    cnt = np.bincount(ix, minlength=c3.n)
    assert cnt[0] > 0.99 * 20000 and cnt[:26].min() > 0.5 * 20000          # Zipf(1.1) head
    c5 = datagen.CONFIGS["c5"]
    ip, ix, v = datagen.docs(c5, 0, 5000)
    assert abs(np.mean(np.abs(v)) - 1.0) < 0.02 and abs(np.mean(v)) < 0.02     # Laplace(0,1)


def test_table_and_choose():
    t = datagen.table(1000, 3, 64, 5)
    assert t.min() >= 0 and t.max() < 64 and t.size == 3000
    np.testing.assert_array_equal(t, datagen.table(1000, 3, 64, 5))
    pool = np.arange(1000, dtype=np.uint32)
    c = datagen.choose(pool, 100, seed=1, row=0)
    assert np.unique(c).size == 100 and np.isin(c, pool).all()
    np.testing.assert_array_equal(c, datagen.choose(pool, 100, seed=1, row=0))
