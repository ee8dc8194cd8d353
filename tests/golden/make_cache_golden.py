"""Golden fixtures for the software row cache (cache.py:68-133), produced by
running the REFERENCE's own `access` / `simulate_trace`.

Run in the build container (where /root/reference exists):
    python tests/golden/make_cache_golden.py
Writes tests/golden/cache.npz: per case the trace, (num_sets, ways, policy),
the per-access AccessResult (hit, evicted or -1) and the TraceStats.
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.dont_write_bytecode = True

from neosim import cache  # noqa: E402

OUT = Path(__file__).resolve().parent


def run(num_sets, ways, policy, trace):
    cfg = cache.CacheConfig(num_sets=num_sets, ways=ways, policy=cache.ReplacementPolicy(policy))
    st = cache.CacheState(cfg)
    hit, ev = [], []
    for r in trace:
        res = cache.access(st, int(r))
        hit.append(1 if res.hit else 0)
        ev.append(-1 if res.evicted is None else res.evicted)
    ts = cache.simulate_trace(cfg, trace)
    assert (ts.hits, ts.misses, ts.evictions) == (st.hits, st.misses, st.evictions)
    return np.array(hit, np.uint8), np.array(ev, np.int64), np.array([ts.hits, ts.misses, ts.evictions], np.int64)


def main():
    rng = np.random.default_rng(2104)
    scan = cache.make_scan_hot_trace()
    cases = [
        (4, 8, "lru", scan), (4, 8, "lfu", scan),
        (1, 2, "lru", [1, 2, 3, 1, 4, 2, 1]), (1, 2, "lfu", [1, 1, 2, 3, 1, 4, 2]),
        (2, 32, "lru", list(range(64)) * 2 + [64, 0, 65, 1]),
        (7, 3, "lru", rng.integers(0, 60, 3000).tolist()),
        (7, 3, "lfu", rng.integers(0, 60, 3000).tolist()),
        (64, 32, "lru", (np.minimum(rng.zipf(1.1, 20000), 10**6) - 1).tolist()),
        (64, 32, "lfu", (np.minimum(rng.zipf(1.1, 20000), 10**6) - 1).tolist()),
        (16, 5, "lfu", rng.integers(0, 2000, 8000).tolist()),
        (3, 1, "lru", rng.integers(0, 12, 500).tolist()),
        (1000, 32, "lru", rng.integers(0, 10**7, 20000).tolist()),
    ]
    out = {"ncases": np.array(len(cases))}
    for i, (ns, w, pol, tr) in enumerate(cases):
        h, e, s = run(ns, w, pol, tr)
        out[f"c{i}_cfg"] = np.array([ns, w, 1 if pol == "lfu" else 0], np.int64)
        out[f"c{i}_trace"] = np.array(tr, np.int64)
        out[f"c{i}_hit"] = h
        out[f"c{i}_evicted"] = e
        out[f"c{i}_stats"] = s
    np.savez_compressed(OUT / "cache.npz", **out)
    print("wrote", OUT / "cache.npz", len(cases), "cases")


if __name__ == "__main__":
    main()
