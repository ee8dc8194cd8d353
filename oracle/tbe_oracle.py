"""CPU ORACLE — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restatement of the reference hot path; each function cites the reference
file:line (paths relative to /root/reference/pkg/src/neosim) it follows.
Two implementations of the arithmetic:

* ``*_c`` — ctypes into liboracle.so: sequential C loops in the
  reference's exact order (fast enough for full-size tables);
* ``np_*`` — the reference's numpy primitives (add.at, unique, fancy
  indexing), restated; used to time the CPU baseline with the reference's
  own performance profile and to cross-check the C loops.
"""
from __future__ import annotations

import ctypes as C
import math
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = _HERE / "liboracle.so"
_lib = None

_P = C.c_void_p
_I = C.c_int64


def build() -> Path:
    """Compile liboracle.so with the committed Makefile."""
    src = _HERE / "oracle.c"
    if not _LIB.exists() or _LIB.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        h = C.CDLL(str(_LIB))
        h.or_forward_f64.restype = _I
        h.or_forward_f64.argtypes = [_I, _P, _P, _I, _I, _P, _P]
        h.or_backward_aggregate_f64.restype = _I
        h.or_backward_aggregate_f64.argtypes = [_I, _P, _P, _I, _I, _I, _P, _P, _P]
        h.or_apply_f64.restype = None
        h.or_apply_f64.argtypes = [C.c_int, _I, _P, _P, _I, _P, _P, C.c_double, C.c_double]
        h.or_bucketize.restype = _I
        h.or_bucketize.argtypes = [_I, _P, _P, C.c_int, _P, _P, _P]
        h.or_cache_simulate.restype = _I
        h.or_cache_simulate.argtypes = [_I, _I, C.c_int, _I, _P, _P, _P, _P]
        _lib = h
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_P)


def offsets_of(lengths) -> np.ndarray:
    """model.py:365-370 lengths_to_offsets."""
    lengths = np.asarray(lengths, dtype=np.int64)
    out = np.zeros(len(lengths) + 1, dtype=np.int64)
    out[1:] = np.cumsum(lengths)
    return out


class OracleIndexError(Exception):
    """First out-of-range id in buffer order (errors.py:43 IndexOutOfRange)."""

    def __init__(self, position: int, value: int):
        self.position, self.value = position, value
        super().__init__(f"index {value} at position {position} out of range")


# ---------------------------------------------------------------------------
# C-loop oracle


def forward_pooled_c(values: np.ndarray, lengths, indices) -> np.ndarray:
    """embedding.py:136-151 forward_pooled (sum pooling, empty bag -> 0)."""
    values = np.ascontiguousarray(values, dtype=np.float64)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    off = offsets_of(lengths)
    n, (H, D) = len(off) - 1, values.shape
    out = np.empty((n, D), dtype=np.float64)
    bad = lib().or_forward_f64(n, _p(off), _p(idx), H, D, _p(values), _p(out))
    if bad >= 0:
        raise OracleIndexError(int(bad), int(idx[bad]))
    return out


def backward_aggregate_c(lengths, indices, upstream: np.ndarray):
    """embedding.py:175-192 backward_sort_aggregate -> (ids ascending, grads)."""
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    up = np.ascontiguousarray(upstream, dtype=np.float64)
    off = offsets_of(lengths)
    n, D = len(off) - 1, up.shape[1]
    if len(idx) == 0:
        return np.empty(0, dtype=np.int64), np.zeros((0, D))
    lo, hi = int(idx.min()), int(idx.max())
    ids = np.empty(len(idx), dtype=np.int64)
    grads = np.empty((len(idx), D), dtype=np.float64)
    U = lib().or_backward_aggregate_f64(n, _p(off), _p(idx), lo, hi - lo + 1, D, _p(up), _p(ids), _p(grads))
    return ids[:U].copy(), grads[:U].copy()


_KIND = {"sgd": 0, "rowwise_adagrad": 1, "adagrad": 2}


def apply_c(kind: str, values: np.ndarray, moment, ids, grads, lr: float, eps: float) -> None:
    """embedding.py:212-254 (in place on values / moment)."""
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    g = np.ascontiguousarray(grads, dtype=np.float64)
    assert values.flags.c_contiguous and values.dtype == np.float64
    mp = None
    if moment is not None:
        assert moment.flags.c_contiguous and moment.dtype == np.float64
        mp = _p(moment)
    lib().or_apply_f64(_KIND[kind], len(ids), _p(ids), _p(g), values.shape[1], _p(values), mp, lr, eps)


def bucketize_c(lengths, indices, starts):
    """comms.py:107-141 bucketize_rowwise -> list of (lengths, indices)."""
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    off = offsets_of(lengths)
    st = np.ascontiguousarray(starts, dtype=np.int64)
    n, k = len(off) - 1, len(st) - 1
    out_len = np.empty((k, n), dtype=np.int64)
    out_idx = np.empty(max(len(idx), 1), dtype=np.int64)
    bad = lib().or_bucketize(n, _p(off), _p(idx), k, _p(st), _p(out_len), _p(out_idx))
    if bad >= 0:
        raise OracleIndexError(int(bad), int(idx[bad]))
    parts, pos = [], 0
    for s in range(k):
        c = int(out_len[s].sum())
        parts.append((out_len[s].copy(), out_idx[pos:pos + c].copy()))
        pos += c
    return parts


# ---------------------------------------------------------------------------
# numpy-primitive port (the reference's own performance profile)


def np_forward_pooled(values, lengths, indices) -> np.ndarray:
    """embedding.py:147-150: add.at scatters rows in buffer order."""
    lengths = np.asarray(lengths, dtype=np.int64)
    idx = np.asarray(indices, dtype=np.int64)
    pooled = np.zeros((lengths.shape[0], values.shape[1]))
    owner = np.repeat(np.arange(lengths.shape[0]), lengths)
    np.add.at(pooled, owner, values[idx])
    return pooled


def np_backward_sort_aggregate(lengths, indices, upstream):
    """embedding.py:188-191: unique ids, add.at of the owning samples' rows."""
    lengths = np.asarray(lengths, dtype=np.int64)
    idx = np.asarray(indices, dtype=np.int64)
    owner = np.repeat(np.arange(lengths.shape[0]), lengths)
    uniq, slot = np.unique(idx, return_inverse=True)
    acc = np.zeros((uniq.shape[0], upstream.shape[1]))
    np.add.at(acc, slot, upstream[owner])
    return uniq, acc


def np_apply(kind: str, values, moment, ids, grads, lr: float, eps: float) -> None:
    """embedding.py:212-254 with numpy fancy indexing (in place)."""
    if kind == "sgd":
        values[ids] -= lr * grads
        return
    keep = (grads != 0.0).any(axis=1)
    ids, grads = ids[keep], grads[keep]
    if ids.shape[0] == 0:
        return
    if kind == "rowwise_adagrad":
        moment[ids] += (grads * grads).mean(axis=1)
        values[ids] -= lr * grads / (np.sqrt(moment[ids]) + eps)[:, None]
    else:
        moment[ids] += grads * grads
        values[ids] -= lr * grads / (np.sqrt(moment[ids]) + eps)


def fp16_roundtrip(values):
    """embedding.py:288-299: RNE through binary16; (quantized, overflow)."""
    arr = np.asarray(values, dtype=np.float64)
    with np.errstate(over="ignore"):
        q = arr.astype(np.float16).astype(np.float64)
    return q, np.isinf(q)


def bf16_roundtrip(values):
    """BF16 wire format restated as RNE of the f32 value (no reference: the
    reference only rescales byte counts, comms.py:521-540)."""
    f = np.asarray(values, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32).astype(np.float64)


# ---------------------------------------------------------------------------
# steps


def init_tables(specs, kind: str, seed: int, zero_init: bool = False):
    """embedding.py:110-129 build_tables: (values, moment) per table."""
    out = []
    for t, spec in enumerate(specs):
        H, D = spec.num_rows, spec.dim
        if zero_init:
            v = np.zeros((H, D))
        else:
            v = np.random.default_rng([seed, t]).standard_normal((H, D))
            if getattr(spec.value_precision, "value", spec.value_precision) == "FP16":
                v, _ = fp16_roundtrip(v)
        m = None if kind == "sgd" else (np.zeros(H) if kind == "rowwise_adagrad" else np.zeros((H, D)))
        out.append((v, m))
    return out


def train_step(specs, lengths, indices, kind: str, lr: float, eps: float, seed: int,
               zero_init: bool = False, upstream=None):
    """embedding.py:312-329 train_step_reference on the C loops.

    lengths (T, n), indices (table-major).  upstream: optional (n, sum D)
    gradient (default ones, the reference's sum-of-outputs loss).
    Returns (pooled (n, sum D), [(values, moment)])."""
    lengths = np.asarray(lengths, dtype=np.int64)
    n = lengths.shape[1]
    tables = init_tables(specs, kind, seed, zero_init)
    tab_off = offsets_of(lengths.sum(axis=1))
    outs = []
    for t, (v, _) in enumerate(tables):
        outs.append(forward_pooled_c(v, lengths[t], indices[tab_off[t]:tab_off[t + 1]]))
    pooled = np.concatenate(outs, axis=1) if outs else np.zeros((n, 0))
    col = 0
    for t, (v, m) in enumerate(tables):
        D = v.shape[1]
        up = np.ones((n, D)) if upstream is None else np.ascontiguousarray(upstream[:, col:col + D])
        col += D
        ids, g = backward_aggregate_c(lengths[t], indices[tab_off[t]:tab_off[t + 1]], up)
        apply_c(kind, v, m, ids, g, lr, eps)
        if getattr(specs[t].value_precision, "value", specs[t].value_precision) == "FP16":
            v[...], _ = fp16_roundtrip(v)
    return pooled, tables


def synthetic_batch(specs, num_samples: int, seed: int):
    """model.py:384-421 gen_synthetic_batch (same RNG stream):
    returns (lengths (T, n), indices)."""
    rng = np.random.default_rng(seed)
    lengths = np.empty((len(specs), num_samples), dtype=np.int64)
    parts = []
    for t, spec in enumerate(specs):
        base = math.floor(spec.avg_pooling)
        frac = spec.avg_pooling - base
        lens = np.full(num_samples, base, dtype=np.int64)
        if frac > 0:
            lens += rng.random(num_samples) < frac
        lengths[t] = lens
        total = int(lens.sum())
        skew = getattr(spec, "index_skew", None)
        if skew is None or getattr(skew.kind, "value", skew.kind) == "uniform":
            parts.append(rng.integers(0, spec.num_rows, size=total, dtype=np.int64))
        else:
            p = np.arange(1, spec.num_rows + 1, dtype=np.float64) ** (-skew.alpha)
            p /= p.sum()
            parts.append(rng.choice(spec.num_rows, size=total, p=p).astype(np.int64))
    return lengths, (np.concatenate(parts) if parts else np.empty(0, dtype=np.int64))


# ---------------------------------------------------------------------------
# layout (comms.py:197-353)


def permute_blocks(outer: int, inner: int, B: int, lengths, indices):
    """comms.py:222-245 _permute_blocks: (o, i) blocks -> (i, o) order."""
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices)
    mat = lengths.reshape(outer, inner, B)
    starts = offsets_of(mat.sum(axis=2).reshape(-1))
    ol, oi = [], []
    for i in range(inner):
        for o in range(outer):
            blk = o * inner + i
            ol.append(mat[o, i])
            oi.append(indices[starts[blk]:starts[blk + 1]])
    return (np.concatenate(ol) if ol else np.empty(0, np.int64),
            np.concatenate(oi) if oi else np.empty(0, indices.dtype))


def to_wtb(lengths, indices, workers: int):
    """comms.py:197-219: canonical (T, n) batch -> (W, T, B) wire order.
    The canonical batch is the (T, W, B) block order, so this is the inverse
    block permute."""
    lengths = np.asarray(lengths, dtype=np.int64)
    T, n = lengths.shape
    return permute_blocks(T, workers, n // workers, lengths.reshape(-1), indices)


# ---------------------------------------------------------------------------
# table checkpoint format (embedding.py:334-377): b"NEOT", "<QQBB" header
# (rows, dim, precision code FP32=0/FP16=1, moment code none=0/rowwise=1/
# elementwise=2), then the f64 values (row-major) and the f64 moment.

NEOT_MAGIC = b"NEOT"


def neot_write(fh, values, moment=None, precision: int = 0) -> None:
    """dump_table (embedding.py:341-360)."""
    import struct

    values = np.ascontiguousarray(values, dtype=np.float64)
    mcode = 0 if moment is None else (1 if np.ndim(moment) == 1 else 2)
    fh.write(NEOT_MAGIC)
    fh.write(struct.pack("<QQBB", values.shape[0], values.shape[1], precision, mcode))
    fh.write(values.tobytes())
    if moment is not None:
        fh.write(np.ascontiguousarray(moment, dtype=np.float64).tobytes())


def neot_read(fh):
    """load_table (embedding.py:363-377) -> (values, moment | None, precision)."""
    import struct

    if fh.read(4) != NEOT_MAGIC:
        raise ValueError("bad table checkpoint magic")
    rows, dim, prec, mcode = struct.unpack("<QQBB", fh.read(18))
    values = np.frombuffer(fh.read(rows * dim * 8), dtype=np.float64).reshape(rows, dim).copy()
    moment = None
    if mcode == 1:
        moment = np.frombuffer(fh.read(rows * 8), dtype=np.float64).copy()
    elif mcode == 2:
        moment = np.frombuffer(fh.read(rows * dim * 8), dtype=np.float64).reshape(rows, dim).copy()
    return values, moment, prec


def cache_simulate_c(num_sets: int, ways: int, policy: str, trace):
    """cache.py:68-126 (access over a trace): (hit uint8[n], evicted int64[n],
    (hits, misses, evictions)); raises OracleIndexError at a negative row."""
    tr = np.ascontiguousarray(trace, dtype=np.int64)
    n = len(tr)
    hit = np.zeros(max(n, 1), dtype=np.uint8)
    ev = np.zeros(max(n, 1), dtype=np.int64)
    st = np.zeros(3, dtype=np.int64)
    bad = lib().or_cache_simulate(num_sets, ways, 1 if policy == "lfu" else 0, n, _p(tr), _p(hit), _p(ev), _p(st))
    if bad >= 0:
        raise OracleIndexError(int(bad), int(tr[bad]))
    return hit[:n], ev[:n], tuple(int(x) for x in st)
