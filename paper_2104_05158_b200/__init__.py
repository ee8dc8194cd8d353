"""paper_2104_05158_b200 — B200-native hot path of Neo (arXiv 2104.05158).

Table-batched embedding bags (TBE) with a fused sort/segment-reduce backward
and exact sparse optimizers, row-wise bucketisation, the (W,T,B)<->(T,W,B)
permute and the sharded-embedding all-to-all, as hand-written sm_100a
kernels behind a C ABI (include/neo_tbe.h, libneob200.so), driven from
PyTorch with NCCL for the collectives.

The public names mirror the reference package ``neosim`` for this path
(neosim/__init__.py:60-86), so code written against the reference's
operator API runs here unchanged; ``dropin.install()`` patches a loaded
``neosim`` in place.
"""
from __future__ import annotations

__version__ = "0.1.0"

from . import _capi
from . import cache, checkpoint  # noqa: F401
from .errors import (IndexOutOfRange, InvalidScheme, InvalidValue, LayoutMismatch,  # noqa: F401
                     MalformedDocument, MissingKey, NeosimError, NonMonotonicOffsets)
from .spec import (CombinedBatch, EmbeddingTable, GlobalBatchLayout, IndexSkew, LayoutTag,  # noqa: F401
                   ModelSpec, OptimizerConfig, OptimizerKind, Precision, RowGradients, SkewKind,
                   TableSpec, build_tables, gen_synthetic_batch, lengths_to_offsets, offsets_to_lengths)
from .embedding import (apply_adagrad, apply_optimizer, apply_rowwise_adagrad, apply_sgd,  # noqa: F401
                        backward_sort_aggregate, forward_pooled, fused_backward_update, fused_forward,
                        merge_row_gradients, quantize_fp16_roundtrip, storage_roundtrip,
                        train_step_reference)
from .comms import (LaidOutBatch, ShardedState, ShardInput, WorkerSlice, alltoall_redistribute,  # noqa: F401
                    bucketize_rowwise, from_twb, permute_TWB_to_WTB, permute_WTB_to_TWB, reassemble_values,
                    replicate_columnwise, to_wtb, train_step_sharded)
from .plan import (Scheme, SchemeKind, Shard, ShardingPlan, TableAssignment, even_bounds,  # noqa: F401
                   plan_from_json, plan_to_json, validate_plan)


def load():
    """Load libneob200.so (raises if it was not built; there is no fallback)."""
    return _capi.lib()
