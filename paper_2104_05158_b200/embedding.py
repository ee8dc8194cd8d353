"""Reference-facing embedding operators, executed on the B200.

Same names, signatures, argument meaning, mutation and error behaviour as
neosim/embedding.py (file:line on each function).  Inputs are the
reference's host arrays / ``EmbeddingTable`` objects; every function moves
its operands to HBM, runs the libneob200 kernels and writes results back
(mutating tables in place exactly where the reference does).  Tables hold
float64 master values, so these calls run the f64 kernel instantiations,
whose accumulation orders reproduce the reference bit for bit.

The production (HBM-resident, f32/f16) path is ``tbe.TableGroup``; this
module is the drop-in boundary that the reference's own tests and callers
exercise.
"""
from __future__ import annotations

from typing import Sequence

import numpy as np
import torch

from . import tbe
from .errors import IndexOutOfRange, InvalidValue, LayoutMismatch
from .spec import (EmbeddingTable, OptimizerConfig, OptimizerKind, RowGradients,  # noqa: F401
                   build_tables, kind_value)

_F64 = torch.float64


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_05158_b200 operators require a CUDA device (no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _dev(a: np.ndarray, dtype=None) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.to(dtype)
    return t.to(_device(), non_blocking=False)


def _offsets_dev(lengths: np.ndarray) -> torch.Tensor:
    return tbe.lengths_to_offsets(_dev(lengths.astype(np.int64)))


def _table_dev(table):
    w = _dev(np.asarray(table.values, dtype=np.float64))
    m = None if table.moment is None else _dev(np.asarray(table.moment, dtype=np.float64))
    return w, m


def _writeback(table, w: torch.Tensor, m) -> None:
    table.values[...] = w.cpu().numpy()
    if m is not None:
        table.moment[...] = m.cpu().numpy()


# ---------------------------------------------------------------------------
# forward


def forward_pooled(table, lengths, indices) -> np.ndarray:
    """Sum-pool rows per sample (embedding.py:136-151)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    if int(lengths.sum()) != len(indices):
        raise LayoutMismatch("lengths do not cover the index buffer")
    n, D = len(lengths), table.dim
    if n == 0:
        return np.zeros((0, D), dtype=np.float64)
    w, _ = _table_dev(table)
    grp = tbe.TableGroup([table.num_rows], [D], dtype=_F64, optim=None, device=w.device,
                         weights=[w], table_ids=[table.spec.id])
    err = tbe.ErrorRecord(w.device).reset()
    out = grp.forward(_dev(indices), _offsets_dev(lengths), n, err=err)
    tbe.raise_if_bad(err, [table.spec.id])
    return out.cpu().numpy()


def fused_forward(tables: Sequence, batch) -> np.ndarray:
    """All tables in ONE TBE launch; equals per-table pooling concatenated
    along columns (embedding.py:154-168)."""
    if batch.num_tables != len(tables):
        raise LayoutMismatch(f"batch has {batch.num_tables} tables, worker has {len(tables)}")
    n = batch.num_samples
    if not tables:
        return np.zeros((n, 0), dtype=np.float64)
    lengths = np.asarray(batch.lengths, dtype=np.int64)
    for t, table in enumerate(tables):  # per-table layout check, as forward_pooled
        lens, idx = batch.table_slice(t)
        if int(np.sum(lens)) != len(idx):
            raise LayoutMismatch("lengths do not cover the index buffer")
    ws = [_table_dev(t)[0] for t in tables]
    ids = [t.spec.id for t in tables]
    grp = tbe.TableGroup([t.num_rows for t in tables], [t.dim for t in tables], dtype=_F64, optim=None,
                         device=ws[0].device, weights=ws, table_ids=ids)
    if n == 0:
        return np.zeros((0, grp.total_dim), dtype=np.float64)
    err = tbe.ErrorRecord(ws[0].device).reset()
    out = grp.forward(_dev(np.asarray(batch.indices, dtype=np.int64)), _offsets_dev(lengths.reshape(-1)),
                      n, err=err)
    tbe.raise_if_bad(err, ids)
    return out.cpu().numpy()


# ---------------------------------------------------------------------------
# backward


def _aggregate_dev(lengths: np.ndarray, indices: np.ndarray, upstream: np.ndarray):
    """Device (ids, grads) of the sort/segment-reduce; ids shifted back by
    the minimum id so negative ids behave as in np.unique."""
    n, D = upstream.shape[0], upstream.shape[1]
    lo = int(indices.min()) if len(indices) else 0
    hi = int(indices.max()) if len(indices) else 0
    shift = min(lo, 0)
    rows = hi - shift + 1
    grp = tbe.TableGroup([rows], [D], dtype=_F64, optim=None, device=_device(), weights=[None])
    idx_dev = _dev(indices - shift if shift else indices)
    ids, grads, count = grp.backward(idx_dev, _offsets_dev(lengths), n, _dev(upstream, _F64),
                                     mode="aggregate")
    return ids, grads, count, shift


def backward_sort_aggregate(lengths, indices, upstream) -> RowGradients:
    """Adjoint of sum pooling (embedding.py:175-192)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    upstream = np.asarray(upstream, dtype=np.float64)
    if int(lengths.sum()) != len(indices):
        raise LayoutMismatch("lengths do not cover the index buffer")
    if upstream.shape[0] != len(lengths):
        raise LayoutMismatch("one upstream gradient row per sample required")
    D = upstream.shape[1] if upstream.ndim == 2 else 0
    if len(indices) == 0 or D == 0 or len(lengths) == 0:
        ids = np.unique(indices)
        return RowGradients(ids, np.zeros((len(ids), D), dtype=np.float64))
    ids, grads, count, shift = _aggregate_dev(lengths, indices, upstream.reshape(len(lengths), D))
    U = int(count.item())
    ids_h = ids[:U].cpu().numpy() + shift
    return RowGradients(ids_h, grads[:U, :D].cpu().numpy().copy())


def merge_row_gradients(parts: Sequence, dim: int) -> RowGradients:
    """Sum per-row gradients across partial results, in part order
    (embedding.py:195-205).  Each part row is treated as a one-id bag whose
    upstream row is its gradient, so the device sort/segment-reduce sums the
    parts in list order — the reference's add.at order."""
    parts = [p for p in parts if len(p.ids)]
    if not parts:
        return RowGradients(np.empty(0, dtype=np.int64), np.zeros((0, dim)))
    ids = np.concatenate([np.asarray(p.ids, dtype=np.int64) for p in parts])
    grads = np.concatenate([np.asarray(p.grads, dtype=np.float64).reshape(-1, dim) for p in parts])
    return backward_sort_aggregate(np.ones(len(ids), dtype=np.int64), ids, grads)


# ---------------------------------------------------------------------------
# sparse optimizers


def _apply(table, grads, cfg, optim: str) -> None:
    ids = np.asarray(grads.ids, dtype=np.int64)
    g = np.asarray(grads.grads, dtype=np.float64)
    if len(ids) == 0:
        return
    w, m = _table_dev(table)
    g_dev = _dev(g.reshape(len(ids), table.dim))
    tbe.apply_row_updates(w, m, _dev(ids), g_dev, optim, cfg.lr, cfg.eps)
    _writeback(table, w, m)


def apply_rowwise_adagrad(table, grads, cfg):
    """embedding.py:212-232"""
    if kind_value(cfg.kind) != "rowwise_adagrad":
        raise InvalidValue("cfg.kind", "expected rowwise_adagrad")
    if table.moment is None or table.moment.ndim != 1:
        raise InvalidValue("moment", "row-wise state must be a length-H vector")
    _apply(table, grads, cfg, "rowwise_adagrad")
    return table


def apply_adagrad(table, grads, cfg):
    """embedding.py:235-247"""
    if table.moment is None or table.moment.ndim != 2:
        raise InvalidValue("moment", "elementwise state must be an (H, D) matrix")
    _apply(table, grads, cfg, "adagrad")
    return table


def apply_sgd(table, grads, cfg):
    """embedding.py:250-254"""
    _apply(table, grads, cfg, "sgd")
    return table


_OPTIMIZERS = {
    OptimizerKind.SGD: apply_sgd,
    OptimizerKind.ROWWISE_ADAGRAD: apply_rowwise_adagrad,
    OptimizerKind.ADAGRAD: apply_adagrad,
}


def apply_optimizer(table, grads, cfg):
    """embedding.py:264-267"""
    return _OPTIMIZERS[OptimizerKind(kind_value(cfg.kind))](table, grads, cfg)


def _check_state(table, kind: str) -> None:
    if kind == "rowwise_adagrad":
        if table.moment is None or table.moment.ndim != 1:
            raise InvalidValue("moment", "row-wise state must be a length-H vector")
    elif kind == "adagrad":
        if table.moment is None or table.moment.ndim != 2:
            raise InvalidValue("moment", "elementwise state must be an (H, D) matrix")


def fused_backward_update(table, lengths, indices, upstream, cfg) -> RowGradients:
    """Sort-aggregate, then exactly one optimizer application per touched
    row, in one fused kernel sequence (embedding.py:270-281)."""
    lengths = np.asarray(lengths, dtype=np.int64)
    indices = np.asarray(indices, dtype=np.int64)
    upstream = np.asarray(upstream, dtype=np.float64)
    if int(lengths.sum()) != len(indices):
        raise LayoutMismatch("lengths do not cover the index buffer")
    if upstream.shape[0] != len(lengths):
        raise LayoutMismatch("one upstream gradient row per sample required")
    kind = kind_value(cfg.kind)
    _check_state(table, kind)
    grads = backward_sort_aggregate(lengths, indices, upstream)
    if len(indices) == 0:
        return grads
    w, m = _table_dev(table)
    grp = tbe.TableGroup([table.num_rows], [table.dim], dtype=_F64, optim=kind, device=w.device,
                         weights=[w], moments=[m], table_ids=[table.spec.id])
    grp.backward(_dev(indices), _offsets_dev(lengths), len(lengths),
                 _dev(upstream.reshape(len(lengths), table.dim)), mode="update", optim=kind,
                 lr=cfg.lr, eps=cfg.eps)
    _writeback(table, w, m)
    return grads


# ---------------------------------------------------------------------------
# precision emulation


def quantize_fp16_roundtrip(values):
    """RNE through binary16 and back; overflow flagged (embedding.py:288-299)."""
    arr = np.asarray(values, dtype=np.float64)
    if not np.isfinite(arr).all():
        raise InvalidValue("values", "inputs must be finite")
    if arr.size == 0:
        return arr.copy(), np.zeros(arr.shape, dtype=bool)
    x = _dev(arr)
    ovf, _ = tbe.fp16_roundtrip_(x)
    return x.cpu().numpy(), ovf.cpu().numpy().astype(bool)


def storage_roundtrip(table) -> None:
    """embedding.py:302-305"""
    if getattr(table.spec.value_precision, "value", table.spec.value_precision) == "FP16":
        table.values[:], _ = quantize_fp16_roundtrip(table.values)


# ---------------------------------------------------------------------------
# single-worker step


def train_step_reference(model, batch, cfg, seed: int = 0, zero_init: bool = False):
    """One fused forward over all tables, upstream of ones (sum-of-outputs
    loss), one fused backward+update over all tables, FP16 storage round
    trip — everything resident on the GPU between the steps
    (embedding.py:312-329)."""
    batch.validate_against(model)
    tables = build_tables(model, cfg, seed, zero_init=zero_init)
    n = batch.num_samples
    kind = kind_value(cfg.kind)
    if not tables:
        return np.zeros((n, 0), dtype=np.float64), tables
    dev = _device()
    ws, ms = zip(*[_table_dev(t) for t in tables])
    ids = [t.spec.id for t in tables]
    grp = tbe.TableGroup([t.num_rows for t in tables], [t.dim for t in tables], dtype=_F64,
                         optim=kind, device=dev, weights=list(ws), moments=list(ms), table_ids=ids)
    idx = _dev(np.asarray(batch.indices, dtype=np.int64))
    off = _offsets_dev(np.asarray(batch.lengths, dtype=np.int64).reshape(-1))
    out = grp.forward(idx, off, n)
    upstream = torch.ones((n, grp.total_dim), dtype=_F64, device=dev)
    grp.backward(idx, off, n, upstream, mode="update", optim=kind, lr=cfg.lr, eps=cfg.eps)
    for t, table in enumerate(tables):
        if getattr(table.spec.value_precision, "value", None) == "FP16":
            tbe.fp16_roundtrip_(ws[t])
        _writeback(table, ws[t], ms[t])
    return out.cpu().numpy(), tables
