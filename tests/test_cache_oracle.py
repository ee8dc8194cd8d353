"""CPU: the cache oracle (oracle.c or_cache_simulate) pinned against the
reference's own access()/simulate_trace outputs (tests/golden/cache.npz,
made by tests/golden/make_cache_golden.py), plus the host-side API of
paper_2104_05158_b200.cache (no GPU calls)."""
import numpy as np
import pytest

from oracle import tbe_oracle as O


@pytest.fixture(scope="module")
def golden():
    from conftest import GOLDEN

    return dict(np.load(GOLDEN / "cache.npz"))


def test_oracle_matches_reference_access_stream(golden):
    for i in range(int(golden["ncases"])):
        ns, w, lfu = (int(x) for x in golden[f"c{i}_cfg"])
        hit, ev, st = O.cache_simulate_c(ns, w, "lfu" if lfu else "lru", golden[f"c{i}_trace"])
        assert np.array_equal(hit, golden[f"c{i}_hit"]), i
        assert np.array_equal(ev, golden[f"c{i}_evicted"]), i
        assert st == tuple(int(x) for x in golden[f"c{i}_stats"]), i


def test_oracle_hand_vectors():
    # cache.py tests: cold miss then hit; LRU evicts the oldest; a hit refreshes recency
    assert O.cache_simulate_c(1, 2, "lru", [5, 5])[2] == (1, 1, 0)
    hit, ev, st = O.cache_simulate_c(1, 2, "lru", [1, 2, 3])
    assert ev.tolist() == [-1, -1, 1] and st == (0, 3, 1)
    hit, ev, st = O.cache_simulate_c(1, 2, "lru", [1, 2, 1, 3])
    assert ev.tolist() == [-1, -1, -1, 2]
    # LFU keeps the frequently used row
    hit, ev, st = O.cache_simulate_c(1, 2, "lfu", [1, 1, 2, 3])
    assert ev.tolist() == [-1, -1, -1, 2]
    with pytest.raises(O.OracleIndexError):
        O.cache_simulate_c(4, 2, "lru", [1, -3])


def test_scan_hot_trace_and_bandwidth_blend(golden):
    from paper_2104_05158_b200 import cache

    assert cache.make_scan_hot_trace() == golden["c0_trace"].tolist()
    assert cache.effective_row_bandwidth(1.0, 8000.0, 50.0) == pytest.approx(8000.0)
    assert cache.effective_row_bandwidth(0.0, 8000.0, 50.0) == pytest.approx(50.0)
    assert cache.effective_row_bandwidth(0.5, 100.0, 50.0) == pytest.approx(1.0 / (0.5 / 100 + 0.5 / 50))
    with pytest.raises(cache.InvalidValue):
        cache.effective_row_bandwidth(1.5, 1.0, 1.0)
    with pytest.raises(cache.InvalidValue):
        cache.CacheConfig(num_sets=0)
    with pytest.raises(cache.InvalidValue):
        cache.CacheConfig(num_sets=4, ways=0)
    assert cache.CacheConfig(num_sets=4, ways=8).capacity_rows == 32
