"""Probe cache (gace_cache_*; §V item 3, line 314), CPU only
(host-only C-ABI).  SPEC's examples as written, then random operation streams through the
C-ABI against the plain model (oracle/reference.py CacheModel)."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def G():
    from paper_2512_19750_b200 import build, gace
    build.build()
    return gace


def _p(oracle, *rows):
    return np.array(list(rows), dtype=oracle.PRED_DTYPE)


def test_spec_examples(G, oracle):
    A = (0, oracle.EQ, 0, 3, 0)
    B = (1, oracle.BETWEEN, 0, 10, 20)
    c = G.ProbeCache(capacity=3, range_buckets=64)
    dom = [(0, 639), (0, 639)]
    c.put(7, _p(oracle, A, B), 0.25, 25, 100, domains=dom)
    assert c.lookup(7, _p(oracle, A, B), domains=dom)[:3] == (0.25, 25, 100)          # identical key
    assert c.lookup(7, _p(oracle, B, A), domains=dom[::-1]) is not None                # B and A
    assert c.lookup(7, _p(oracle, (0, oracle.EQ, 0, 5, 0), B), domains=dom) is not None   # same bucket [0,10)
    assert c.lookup(7, _p(oracle, (0, oracle.EQ, 0, 30, 0), B), domains=dom) is None    # other bucket
    assert c.lookup(8, _p(oracle, A, B), domains=dom) is None                          # other table
    for v in range(3):                                                                 # capacity + 1
        c.put(7, _p(oracle, (2, oracle.EQ, 0, 100 * v, 0)), 0.5)
    assert c.lookup(7, _p(oracle, A, B), domains=dom) is None and c.stats()["evictions"] == 1
    c.invalidate(7)
    assert c.stats()["size"] == 0
    c.close()


def test_repeat_stream_hits(G, oracle):
    c = G.ProbeCache()
    q = _p(oracle, (0, oracle.EQ, 0, 1, 0), (1, oracle.LT, 0, 9, 0))
    hits = 0
    for i in range(100):
        if c.lookup(1, q) is None:
            c.put(1, q, 0.1, 1, 10)
        else:
            hits += 1
    assert hits == 99 and c.lookup(1, q)[3] == 100
    c.close()


@pytest.mark.parametrize("buckets", [0, 4, 64])
def test_random_streams_match_model(G, oracle, buckets):
    rng = np.random.default_rng(buckets + 1)
    c = G.ProbeCache(capacity=16, range_buckets=buckets)
    m = oracle.CacheModel(capacity=16, buckets=buckets)
    for step in range(3000):
        k = int(rng.integers(1, 4))
        conj = _p(oracle, *[(int(rng.integers(0, 3)), int(rng.integers(0, 6)), int(rng.integers(0, 2)),
                             int(rng.integers(-5, 60)), int(rng.integers(-5, 60))) for _ in range(k)])
        dom = [(0, 49)] * k if buckets else None
        table = int(rng.integers(0, 3))
        r = rng.random()
        if r < 0.45:
            s = float(rng.random())
            c.put(table, conj, s, step, 1000, domains=dom)
            m.put(table, conj, s, step, 1000, domains=dom)
        elif r < 0.98:
            assert c.lookup(table, conj, domains=dom) == m.lookup(table, conj, domains=dom)
        else:
            c.invalidate(table)
            m.invalidate(table)
    st = c.stats()
    assert (st["hits"], st["misses"], st["evictions"], st["size"]) == (m.hits, m.misses, m.evictions, len(m.entries))
    c.close()


def test_errors(G, oracle):
    c = G.ProbeCache()
    with pytest.raises(G.GaceError):
        c.put(1, _p(oracle, (0, oracle.EQ, 0, 1, 0)), 1.5)
    c.close()
    assert G.lib().gace_cache_stats(None, None, None, None, None) == G.GACE_EHANDLE
