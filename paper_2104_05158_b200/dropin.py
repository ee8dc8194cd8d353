"""Drop-in: route a loaded ``neosim`` (the reference package) through the
B200 operators.

``install(neosim_module)`` rebinds, in place, every name on the hot path
wherever the reference binds it:

* ``neosim.embedding``: forward_pooled, fused_forward, backward_sort_aggregate,
  merge_row_gradients, apply_rowwise_adagrad / apply_adagrad / apply_sgd /
  apply_optimizer and the ``_OPTIMIZERS`` dispatch table (embedding.py:257),
  fused_backward_update, quantize_fp16_roundtrip, storage_roundtrip,
  train_step_reference;
* ``neosim.comms``: bucketize_rowwise, replicate_columnwise, to_wtb,
  permute_WTB_to_TWB / permute_TWB_to_WTB, alltoall_redistribute,
  train_step_sharded, reassemble_values, plus the names comms.py binds from
  embedding at import (comms.py:18-28);
* ``neosim.cli``: train_step_reference / train_step_sharded (cli.py:25-26);
* ``neosim.cache.simulate_trace`` (cache.py:117-126; bound by name in
  cli.py:24 and re-exported by neosim/__init__.py:87);
* the ``neosim`` package re-exports (neosim/__init__.py:60-86).

Errors raised by this package are aliased to the reference's exception
classes, so ``except neosim.IndexOutOfRange`` keeps working.  ``uninstall``
restores the originals.
"""
from __future__ import annotations

import importlib

from . import cache as _cache
from . import comms as _comms
from . import embedding as _emb
from . import errors as _errors

_EMBEDDING = ["forward_pooled", "fused_forward", "backward_sort_aggregate", "merge_row_gradients",
              "apply_rowwise_adagrad", "apply_adagrad", "apply_sgd", "apply_optimizer", "fused_backward_update",
              "quantize_fp16_roundtrip", "storage_roundtrip", "train_step_reference"]
_COMMS = ["bucketize_rowwise", "replicate_columnwise", "to_wtb", "permute_WTB_to_TWB", "permute_TWB_to_WTB",
          "alltoall_redistribute", "train_step_sharded", "reassemble_values"]
_COMMS_FROM_EMB = ["apply_optimizer", "backward_sort_aggregate", "forward_pooled", "merge_row_gradients",
                   "storage_roundtrip"]
_ERRORS = ["NeosimError", "MalformedDocument", "MissingKey", "InvalidValue", "NonMonotonicOffsets",
           "InvalidScheme", "IndexOutOfRange", "LayoutMismatch", "EmptyTrace"]

_saved: list = []


def _set(obj, name, value):
    _saved.append((obj, name, getattr(obj, name, None)))
    setattr(obj, name, value)


def install(neosim=None):
    """Patch the reference package in place; returns it."""
    if neosim is None:
        neosim = importlib.import_module("neosim")
    emb = importlib.import_module(neosim.__name__ + ".embedding")
    com = importlib.import_module(neosim.__name__ + ".comms")
    cli = importlib.import_module(neosim.__name__ + ".cli")
    ref_err = importlib.import_module(neosim.__name__ + ".errors")
    ref_cache = importlib.import_module(neosim.__name__ + ".cache")
    # our errors become the reference's classes (raised and caught as such)
    from . import _capi, dist, plan, spec, tbe

    for mod in (_errors, _emb, _comms, _cache, tbe, spec, plan, dist):
        for name in _ERRORS:
            if hasattr(mod, name):
                _set(mod, name, getattr(ref_err, name))
    # the optimizer dispatch table is keyed by the reference's enum
    table = {k: getattr(_emb, {"sgd": "apply_sgd", "rowwise_adagrad": "apply_rowwise_adagrad",
                               "adagrad": "apply_adagrad"}[k.value]) for k in emb.OptimizerKind}
    _set(emb, "_OPTIMIZERS", table)
    # results are built with the reference's own types (identity checks such
    # as `layout.tag is LayoutTag.TWB` in the unpatched from_twb must hold)
    _set(_emb, "RowGradients", emb.RowGradients)
    _set(_emb, "EmbeddingTable", emb.EmbeddingTable)
    for name in ("CombinedBatch", "GlobalBatchLayout", "LayoutTag", "LaidOutBatch", "ShardInput", "WorkerSlice",
                 "ShardedState"):
        if hasattr(com, name):
            _set(_comms, name, getattr(com, name))
    for name in _EMBEDDING:
        _set(emb, name, getattr(_emb, name))
        if hasattr(neosim, name):
            _set(neosim, name, getattr(_emb, name))
    for name in _COMMS:
        _set(com, name, getattr(_comms, name))
        if hasattr(neosim, name):
            _set(neosim, name, getattr(_comms, name))
    for name in _COMMS_FROM_EMB:
        _set(com, name, getattr(_emb, name))
    _set(_cache, "TraceStats", ref_cache.TraceStats)
    _set(ref_cache, "simulate_trace", _cache.simulate_trace)
    if hasattr(neosim, "simulate_trace"):
        _set(neosim, "simulate_trace", _cache.simulate_trace)
    _set(cli, "simulate_trace", _cache.simulate_trace)
    _set(cli, "train_step_reference", _emb.train_step_reference)
    _set(cli, "train_step_sharded", _comms.train_step_sharded)
    _capi.lib()  # fail loudly now if the native library is missing
    return neosim


def uninstall() -> None:
    while _saved:
        obj, name, old = _saved.pop()
        setattr(obj, name, old)
