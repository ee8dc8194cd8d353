"""Set-associative software row cache on the GPU (drop-in for
neosim/cache.py:17-133).

Same names, argument meaning and errors as the reference: ``CacheConfig``
(num_sets >= 1, ways >= 1, LRU/LFU; cache.py:22-37), ``simulate_trace``
returning ``TraceStats`` (cache.py:101-126; EmptyTrace on an empty trace,
InvalidValue("row_id") on a negative row), ``effective_row_bandwidth``
(cache.py:129-136) and ``make_scan_hot_trace`` (cache.py:139-157).  The
replay runs in libneob200 (csrc/cache.cu: stable radix sort of (set,
position) pairs, then one warp per set with one way per lane), producing
the reference's AccessResult stream position for position; ``access_trace``
exposes it.  ways <= 32 (one way per lane); larger associativities raise
InvalidValue.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Iterable, Optional

import numpy as np
import torch

from . import _capi as capi
from .errors import EmptyTrace, InvalidValue  # noqa: F401 (re-exported like cache.py's)


class ReplacementPolicy(str, Enum):
    LRU = "lru"
    LFU = "lfu"


@dataclass(frozen=True)
class CacheConfig:
    num_sets: int
    ways: int = 32
    policy: ReplacementPolicy = ReplacementPolicy.LRU

    def __post_init__(self):  # cache.py:28-32
        if self.num_sets < 1:
            raise InvalidValue("num_sets", "must be >= 1")
        if self.ways < 1:
            raise InvalidValue("ways", "must be >= 1")

    @property
    def capacity_rows(self) -> int:
        return self.num_sets * self.ways


@dataclass(frozen=True)
class AccessResult:
    hit: bool
    evicted: Optional[int] = None


@dataclass(frozen=True)
class TraceStats:
    hits: int
    misses: int
    evictions: int

    @property
    def accesses(self) -> int:
        return self.hits + self.misses

    @property
    def hit_rate(self) -> float:
        return self.hits / self.accesses


def _policy_code(policy) -> int:
    return capi.NEO_CACHE_LFU if ReplacementPolicy(getattr(policy, "value", policy)) is ReplacementPolicy.LFU \
        else capi.NEO_CACHE_LRU


def access_trace(config, trace, with_results: bool = True, device=None):
    """Replay `trace` (row ids, in order) through a fresh cache of `config`
    on the GPU.  Returns (hit uint8[n], evicted int64[n] with -1 = none,
    TraceStats); the arrays are torch tensors on the device (None when
    with_results is False).  Equivalent to calling the reference's access()
    once per element on a new CacheState (cache.py:68-98)."""
    from .tbe import WORKSPACE, ErrorRecord, _stream

    if config.ways > 128:
        raise InvalidValue("ways", "this implementation holds up to four ways per lane (ways <= 128)")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    tr = trace if isinstance(trace, torch.Tensor) else torch.as_tensor(np.asarray(list(trace) if not isinstance(
        trace, np.ndarray) else trace, dtype=np.int64))
    tr = tr.to(device=dev, dtype=torch.int64).contiguous()
    n = int(tr.numel())
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    hit = torch.empty(max(n, 1), dtype=torch.uint8, device=dev) if with_results else None
    ev = torch.empty(max(n, 1), dtype=torch.int64, device=dev) if with_results else None
    if n == 0:
        return (hit[:0] if hit is not None else None), (ev[:0] if ev is not None else None), TraceStats(0, 0, 0)
    err = ErrorRecord(dev).reset()
    wsb = capi.lib().neo_cache_workspace_bytes(n)
    ws = WORKSPACE.get("cache_sim", wsb, dev)
    rc = capi.lib().neo_cache_simulate(int(config.num_sets), int(config.ways), _policy_code(config.policy),
                                       tr.data_ptr(), n, None if hit is None else hit.data_ptr(),
                                       None if ev is None else ev.data_ptr(), stats.data_ptr(), ws.data_ptr(),
                                       ws.numel(), err.ptr, _stream())
    capi.check(rc, "neo_cache_simulate")
    bad = err.read()
    if bad is not None:
        raise InvalidValue("row_id", "must be >= 0")
    h, m, e = (int(x) for x in stats.cpu().tolist())
    return hit, ev, TraceStats(hits=h, misses=m, evictions=e)


def simulate_trace(config: CacheConfig, trace: Iterable[int]) -> TraceStats:
    """cache.py:117-126: hit/miss/eviction counts of `trace` through a fresh
    cache (EmptyTrace if the trace is empty)."""
    _, _, st = access_trace(config, trace, with_results=False)
    if st.accesses == 0:
        raise EmptyTrace("hit rate is undefined on an empty trace")
    return st


def effective_row_bandwidth(hit_rate: float, hbm_bw: float, backing_bw: float) -> float:
    """cache.py:129-136: 1 / (h / hbm + (1 - h) / backing)."""
    if not 0 <= hit_rate <= 1:
        raise InvalidValue("hit_rate", "must be in [0, 1]")
    if not hbm_bw > 0 or not backing_bw > 0:
        raise InvalidValue("bandwidth", "must be > 0")
    return 1.0 / (hit_rate / hbm_bw + (1.0 - hit_rate) / backing_bw)


def make_scan_hot_trace() -> list:
    """cache.py:139-157: 16 hot rows (4 per set of a 4 x 8 cache) re-touched
    three times between one-shot scans of 96 rows, 40 rounds, then the hot
    set once more (LFU keeps the hot rows, LRU does not)."""
    num_sets, ways = 4, 8
    hot = list(range(num_sets * ways // 2))
    trace: list = []
    next_cold = num_sets * ways
    for _ in range(40):
        for _ in range(3):
            trace.extend(hot)
        scan = list(range(next_cold, next_cold + 3 * num_sets * ways))
        next_cold += len(scan)
        trace.extend(scan)
    trace.extend(hot)
    return trace
