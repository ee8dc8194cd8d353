"""GPU: the set-associative row cache replay (csrc/cache.cu) reproduces the
reference's AccessResult stream and TraceStats bit-exactly: against the
reference's own outputs (tests/golden/cache.npz) and against the C oracle on
large seeded traces; error contract as cache.py (InvalidValue on a negative
row, EmptyTrace on an empty trace)."""
import numpy as np
import pytest
import torch

from oracle import tbe_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cache():
    import paper_2104_05158_b200 as p
    from paper_2104_05158_b200 import cache as c

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    p.load()
    return c


@pytest.fixture(scope="module")
def golden():
    from conftest import GOLDEN

    return dict(np.load(GOLDEN / "cache.npz"))


def _cfg(cache, ns, w, lfu):
    return cache.CacheConfig(num_sets=ns, ways=w, policy=cache.ReplacementPolicy.LFU if lfu else
                             cache.ReplacementPolicy.LRU)


def test_reference_golden_streams(cache, golden):
    for i in range(int(golden["ncases"])):
        ns, w, lfu = (int(x) for x in golden[f"c{i}_cfg"])
        hit, ev, st = cache.access_trace(_cfg(cache, ns, w, lfu), golden[f"c{i}_trace"])
        assert np.array_equal(hit.cpu().numpy(), golden[f"c{i}_hit"]), i
        assert np.array_equal(ev.cpu().numpy(), golden[f"c{i}_evicted"]), i
        assert (st.hits, st.misses, st.evictions) == tuple(int(x) for x in golden[f"c{i}_stats"]), i


@pytest.mark.parametrize("ns,w,lfu,dist", [(4096, 32, 0, "uniform"), (4096, 32, 1, "zipf"), (977, 8, 1, "uniform"),
                                           (50000, 4, 0, "zipf"), (1, 32, 0, "zipf"), (300, 1, 1, "uniform"),
                                           # more than one way per lane (the reference accepts any ways)
                                           (1024, 48, 0, "uniform"), (512, 64, 1, "zipf"), (3, 100, 0, "zipf"),
                                           (64, 128, 1, "uniform")])
def test_large_traces_match_oracle(cache, ns, w, lfu, dist):
    rng = np.random.default_rng(ns + w)
    n = 400_000 if ns > 1 else 50_000
    if dist == "zipf":
        tr = np.minimum(rng.zipf(1.05, n) - 1, 10**8)
    else:
        tr = rng.integers(0, ns * w * 3, n)
    hit, ev, st = cache.access_trace(_cfg(cache, ns, w, lfu), tr)
    oh, oe, ost = O.cache_simulate_c(ns, w, "lfu" if lfu else "lru", tr)
    assert (st.hits, st.misses, st.evictions) == ost
    assert np.array_equal(hit.cpu().numpy(), oh)
    assert np.array_equal(ev.cpu().numpy(), oe)
    assert cache.simulate_trace(_cfg(cache, ns, w, lfu), tr) == st


def test_error_contract(cache):
    with pytest.raises(cache.InvalidValue):
        cache.simulate_trace(cache.CacheConfig(num_sets=4, ways=2), [1, 2, -1, 3])
    with pytest.raises(cache.EmptyTrace):
        cache.simulate_trace(cache.CacheConfig(num_sets=4, ways=2), [])
    with pytest.raises(cache.InvalidValue):
        cache.simulate_trace(cache.CacheConfig(num_sets=4, ways=129), [1])
    assert cache.simulate_trace(cache.CacheConfig(num_sets=2, ways=32), list(range(64)) * 2).hit_rate == 0.5
