"""Reference-facing input redistribution and sharded step, on the B200.

Mirrors neosim/comms.py: same names, signatures and error behaviour.  The
integer layout work (bucketize, block permute, replication, send packing)
runs in libneob200's bit-exact kernels; the sharded step runs the same
per-rank pipeline as the NCCL path (``dist.py``) with W logical ranks on
one GPU (``dist.LocalComm``), so the reference's W-worker equivalence tests
exercise the production exchange logic.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np
import torch

from . import tbe
from .errors import IndexOutOfRange, InvalidValue, LayoutMismatch
from .spec import CombinedBatch, GlobalBatchLayout, LayoutTag

LENGTH_BYTES = 8  # comms.py:47 lengths travel as int64 in the metadata phase


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_05158_b200 operators require a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a)).to(_device())


# ---------------------------------------------------------------------------
# bucketize / replicate (comms.py:107-172)


def bucketize_rowwise(lengths, indices, boundaries: Sequence, table_id: str = ""):
    """Route each id to the row shard containing it, rebased; per-shard
    lengths recomputed; order kept inside each shard (comms.py:107-141)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    if int(lengths.sum()) != len(indices):
        raise LayoutMismatch("lengths do not cover the index buffer")
    pos = 0
    for a, b in boundaries:
        if a != pos or b <= a:
            raise InvalidValue("boundaries", "must tile [0, H) in order")
        pos = b
    starts = [int(a) for a, _ in boundaries] + [pos]
    k, n = len(boundaries), len(lengths)
    if n == 0:
        return [(np.zeros(0, np.int64), np.zeros(0, np.int64)) for _ in range(k)]
    err = tbe.ErrorRecord(_device()).reset()
    off = tbe.lengths_to_offsets(_dev(lengths))
    out_len, out_off, out_idx = tbe.bucketize_rowwise(off, _dev(indices), starts, err=err)
    r = err.read()
    if r is not None:
        raise IndexOutOfRange(table_id, r[1])
    L = out_len.cpu().numpy()
    O = out_off.cpu().numpy()
    I = out_idx.cpu().numpy()
    return [(L[s].copy(), I[O[s * n]:O[(s + 1) * n]].copy()) for s in range(k)]


def replicate_columnwise(lengths, indices, num_col_shards: int):
    """k byte-identical input copies (comms.py:164-172).  The NCCL path
    never materialises them: one send buffer feeds every column shard."""
    if num_col_shards < 1:
        raise InvalidValue("num_col_shards", "must be >= 1")
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    out = []
    for src in (lengths, indices):
        if src.size == 0:
            out.append([src.copy() for _ in range(num_col_shards)])
            continue
        d = _dev(src)
        rep = torch.empty(num_col_shards * src.size, dtype=d.dtype, device=d.device)
        tbe.gather_blocks([d] * num_col_shards, [src.size] * num_col_shards, rep)
        h = rep.cpu().numpy().reshape(num_col_shards, src.size)
        out.append([h[i].copy() for i in range(num_col_shards)])
    return list(zip(out[0], out[1]))


# ---------------------------------------------------------------------------
# laid-out batches and the block permute (comms.py:175-264)


@dataclass(frozen=True)
class LaidOutBatch:
    layout: GlobalBatchLayout
    lengths: np.ndarray
    indices: np.ndarray

    def __post_init__(self):
        lay = self.layout
        expected = lay.workers * lay.tables * lay.local_batch
        if len(self.lengths) != expected:
            raise LayoutMismatch(f"expected {expected} length entries, got {len(self.lengths)}")
        if int(np.sum(self.lengths)) != len(self.indices):
            raise LayoutMismatch("lengths do not cover the index buffer")


def _permute(lengths, indices, outer: int, inner: int, B: int):
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    if lengths.size == 0 or B == 0:
        return lengths.copy(), indices.copy()
    if indices.size == 0:
        L, _ = tbe.permute_blocks(outer, inner, B, _dev(lengths), torch.zeros(1, dtype=torch.int64, device=_device()))
        return L.cpu().numpy(), indices.copy()
    L, I = tbe.permute_blocks(outer, inner, B, _dev(lengths), _dev(indices))
    return L.cpu().numpy(), I.cpu().numpy()


def _tag(t):
    return getattr(t, "value", t)


def _permute_laid(laid, new_tag: LayoutTag):
    lay = laid.layout
    W, T, B = lay.workers, lay.tables, lay.local_batch
    outer, inner = (W, T) if _tag(lay.tag) == "WTB" else (T, W)
    L, I = _permute(laid.lengths, laid.indices, outer, inner, B)
    return LaidOutBatch(GlobalBatchLayout(W, T, B, new_tag), L, I)


def permute_WTB_to_TWB(laid) -> LaidOutBatch:
    """comms.py:248-252"""
    if _tag(laid.layout.tag) != "WTB":
        raise LayoutMismatch("expected WTB layout")
    return _permute_laid(laid, LayoutTag.TWB)


def permute_TWB_to_WTB(laid) -> LaidOutBatch:
    """comms.py:255-258"""
    if _tag(laid.layout.tag) != "TWB":
        raise LayoutMismatch("expected TWB layout")
    return _permute_laid(laid, LayoutTag.WTB)


def to_wtb(batch, workers: int) -> LaidOutBatch:
    """Canonical batch -> (W, T, B) wire order (comms.py:197-219).  The
    canonical buffer is already the (T, W, B) block order, so this is one
    device block permute."""
    if workers < 1 or batch.num_samples % workers:
        raise LayoutMismatch("workers must divide the global sample count")
    T, B = batch.num_tables, batch.num_samples // workers
    L, I = _permute(np.asarray(batch.lengths).reshape(-1), batch.indices, T, workers, B)
    return LaidOutBatch(GlobalBatchLayout(workers, T, B, LayoutTag.WTB), L, I)


def from_twb(laid) -> CombinedBatch:
    """comms.py:261-264"""
    if _tag(laid.layout.tag) != "TWB":
        raise LayoutMismatch("expected TWB layout")
    lay = laid.layout
    return CombinedBatch(np.asarray(laid.lengths).reshape(lay.tables, lay.workers * lay.local_batch),
                         laid.indices)


# ---------------------------------------------------------------------------
# redistribution results (comms.py:271-285)


@dataclass
class ShardInput:
    table_id: str
    shard: object
    lengths: np.ndarray
    indices: np.ndarray
    sample_base: int = 0


@dataclass
class WorkerSlice:
    worker: int
    inputs: list = field(default_factory=list)


@dataclass
class ShardedState:
    """comms.py:605-610"""

    shards: dict
    dp_replicas: dict


# ---------------------------------------------------------------------------
# redistribution and the sharded step on W logical ranks (comms.py:292-353,
# comms.py:629-758), through the same engine the NCCL path runs


def _local_batches(batch, W: int, index_dtype=torch.int64):
    """Split a canonical global batch into the W workers' local batches
    ((T, B) lengths, table-major ids on the device): the worker-major wire
    order is one device block permute of the canonical (T, W, B) buffer."""
    T, n = batch.num_tables, batch.num_samples
    B = n // W
    lengths = np.asarray(batch.lengths, dtype=np.int64)
    ids = np.asarray(batch.indices, dtype=np.int64)
    if ids.size:
        L, I = tbe.permute_blocks(T, W, B, _dev(lengths.reshape(-1)), _dev(ids).to(index_dtype))
    else:
        L, I = _dev(lengths.reshape(-1)), torch.zeros(0, dtype=index_dtype, device=_device())
    Lh = L.cpu().numpy().reshape(W, T, B)
    per = Lh.reshape(W, -1).sum(axis=1)
    starts = np.concatenate(([0], np.cumsum(per)))
    return [(Lh[w], I[int(starts[w]):int(starts[w + 1])]) for w in range(W)]


def _engine(model, plan, W, B, kind, init=None, dtype=torch.float64):
    from .dist import LocalComm, ShardedEmbedding

    return ShardedEmbedding(model, plan, LocalComm(W), B, dtype=dtype, optim=kind, init=init)


def alltoall_redistribute(laidout, plan, model) -> list:
    """Two-phase exchange (lengths, then ids) on W logical ranks; each worker
    ends with its shards' global-batch inputs (comms.py:292-353)."""
    from .plan import validate_plan

    lay = laidout.layout
    if _tag(lay.tag) != "WTB":
        raise LayoutMismatch("redistribution consumes the WTB wire order")
    if lay.workers != plan.num_workers or lay.tables != model.num_tables:
        raise LayoutMismatch("batch layout does not match plan/model")
    validate_plan(plan, model)
    W, T, B = lay.workers, lay.tables, lay.local_batch
    Lh = np.asarray(laidout.lengths, dtype=np.int64).reshape(W, T, B)
    ids = _dev(np.asarray(laidout.indices, dtype=np.int64)) if len(laidout.indices) else \
        torch.zeros(0, dtype=torch.int64, device=_device())
    per = Lh.reshape(W, -1).sum(axis=1)
    starts = np.concatenate(([0], np.cumsum(per)))
    batches = [(Lh[w], ids[int(starts[w]):int(starts[w + 1])]) for w in range(W)]
    eng = _engine(model, plan, W, B, "sgd")
    per_rank = eng.redistribute(batches)
    by_id = {a.table_id: a for a in plan.assignments}
    slices = [WorkerSlice(worker=v) for v in range(W)]
    for t, table in enumerate(model.tables):
        a = by_id[table.id]
        kind = getattr(a.scheme.kind, "value", a.scheme.kind)
        if kind == "data_parallel":
            for v in range(W):
                L, I = per_rank[v]["dp"][t]
                slices[v].inputs.append(ShardInput(table.id, a.shards[0], L, I, sample_base=v * B))
            continue
        shards = list(a.shards)
        if kind == "row_wise":
            shards = sorted(shards, key=lambda s: tuple(s.rows))
        for s in shards:
            L, I = per_rank[s.worker]["shards"][(t, list(a.shards).index(s))]
            slices[s.worker].inputs.append(ShardInput(table.id, s, L, I))
    return slices


def _spec_prec(spec) -> str:
    return getattr(spec.value_precision, "value", spec.value_precision)


def train_step_sharded(model, plan, batch, cfg, seed: int = 0, zero_init: bool = False):
    """One iteration across W logical workers through the sharded engine
    (comms.py:629-737): input exchange, fused forward per worker, pooled
    exchange + assembly, backward exchange, fused update per shard, DP
    gradient all-reduce + identical update.  Returns (outputs, ShardedState)."""
    from .embedding import build_tables
    from .plan import validate_plan
    from .spec import EmbeddingTable, kind_value

    validate_plan(plan, model)
    batch.validate_against(model)
    W = plan.num_workers
    if batch.num_samples % W:
        raise LayoutMismatch("global batch must split evenly across workers")
    n = batch.num_samples
    B = n // W
    kind = kind_value(cfg.kind)
    full = build_tables(model, cfg, seed, zero_init=zero_init)

    def init(t, rows, cols):
        return torch.from_numpy(np.ascontiguousarray(full[t].values[rows[0]:rows[1], cols[0]:cols[1]]))

    eng = _engine(model, plan, W, B, kind, init=init)
    pooled = eng.step(_local_batches(batch, W), lr=cfg.lr, eps=cfg.eps)
    out = torch.cat(pooled, dim=0).cpu().numpy() if model.num_tables else np.zeros((n, 0))
    state = ShardedState(shards={}, dp_replicas={})
    lay = eng.lay
    for slot, st in enumerate(eng.states):
        for s, w, m in eng.shard_tensors(slot):
            spec = model.tables[s.table]
            if _spec_prec(spec) == "FP16":
                tbe.fp16_roundtrip_(w)
            state.shards[(s.table_id, s.index)] = EmbeddingTable(
                spec, w.cpu().numpy(), None if m is None else m.cpu().numpy(), row_base=s.rows[0],
                col_base=s.cols[0])
        if st.dp_group is not None:
            for t, w, m in zip(lay.dp_tables, st.dp_group.weights, st.dp_group.moments):
                spec = model.tables[t]
                if _spec_prec(spec) == "FP16":
                    tbe.fp16_roundtrip_(w)
                state.dp_replicas.setdefault(spec.id, []).append(
                    EmbeddingTable(spec, w.cpu().numpy(), None if m is None else m.cpu().numpy()))
    return out, state


def reassemble_values(model, plan, state) -> list:
    """Stitch shard values into full (H, D) matrices; DP from replica 0
    (comms.py:740-758)."""
    out = []
    for table in model.tables:
        a = plan.assignment_for(table.id)
        if getattr(a.scheme.kind, "value", a.scheme.kind) == "data_parallel":
            out.append(state.dp_replicas[table.id][0].values.copy())
            continue
        full = np.zeros((table.num_rows, table.dim), dtype=np.float64)
        for i, s in enumerate(a.shards):
            r0, r1 = s.rows if s.rows else (0, table.num_rows)
            c0, c1 = s.cols if s.cols else (0, table.dim)
            full[r0:r1, c0:c1] = state.shards[(table.id, i)].values
        out.append(full)
    return out
