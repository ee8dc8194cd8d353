"""Host-side mirror of the reference's input contract for the hot path.

Restates, with the same names and field meanings, the types the TBE and the
sharded all-to-all consume:

* tables / model (neosim/model.py:28-168): ``Precision``, ``IndexSkew``,
  ``TableSpec``, ``ModelSpec``;
* the jagged batch (model.py:283-377): ``CombinedBatch`` (per-table lengths
  plus one table-major, sample-major index buffer), ``lengths_to_offsets``,
  ``offsets_to_lengths``, ``LayoutTag``, ``GlobalBatchLayout``;
* the synthetic generator (model.py:384-421) — same RNG stream, so batches
  are identical to the reference's for a given seed;
* optimizer state (embedding.py:24-129): ``OptimizerKind``,
  ``OptimizerConfig``, ``EmbeddingTable``, ``RowGradients``,
  ``build_tables``.

Objects from the reference package are accepted wherever these are (duck
typing on the same attribute names).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import Optional

import numpy as np

from .errors import IndexOutOfRange, InvalidValue, NonMonotonicOffsets


class Precision(str, Enum):
    FP32 = "FP32"
    TF32 = "TF32"
    FP16 = "FP16"
    BF16 = "BF16"


PRECISION_BYTES = {Precision.FP32: 4, Precision.TF32: 4, Precision.FP16: 2, Precision.BF16: 2}


class SkewKind(str, Enum):
    UNIFORM = "uniform"
    ZIPF = "zipf"


@dataclass(frozen=True)
class IndexSkew:
    kind: SkewKind = SkewKind.UNIFORM
    alpha: float = 0.0

    def __post_init__(self):
        if self.kind is SkewKind.ZIPF and not self.alpha > 0:
            raise InvalidValue("index_skew.alpha", "Zipf alpha must be > 0")


@dataclass(frozen=True)
class TableSpec:
    """H rows of dimension D, average pooling L (model.py:63-97)."""

    id: str
    num_rows: int
    dim: int
    avg_pooling: float
    value_precision: Precision = Precision.FP32
    index_skew: IndexSkew = field(default_factory=IndexSkew)

    def __post_init__(self):
        for name, ok in (("num_rows", self.num_rows >= 1), ("dim", self.dim >= 1),
                         ("avg_pooling", self.avg_pooling > 0)):
            if not ok:
                raise InvalidValue(f"tables[{self.id}].{name}", "out of range")
        if self.value_precision not in (Precision.FP32, Precision.FP16):
            raise InvalidValue(f"tables[{self.id}].value_precision", "must be FP32 or FP16")

    @property
    def elem_bytes(self) -> int:
        return PRECISION_BYTES[self.value_precision]

    @property
    def num_params(self) -> int:
        return self.num_rows * self.dim

    @property
    def index_bytes(self) -> int:
        return 4 if self.num_rows <= 2**31 else 8


def model_from_json(text: str) -> "ModelSpec":
    """ModelSpec from the reference's model document (serialize_model_spec /
    parse_model_spec, model.py:611-683): the table list (id, num_rows, dim,
    avg_pooling, value_precision, index_skew) and the batch/dense fields.
    Generator-expanded table lists (model.py:544-578) are not accepted here."""
    import json

    doc = json.loads(text)
    tabs = []
    for i, t in enumerate(doc.get("tables", [])):
        sk = t.get("index_skew", {"kind": "uniform"})
        skew = IndexSkew(SkewKind(sk["kind"]), float(sk.get("alpha", 0.0)))
        tabs.append(TableSpec(id=str(t["id"]), num_rows=int(t["num_rows"]), dim=int(t["dim"]),
                              avg_pooling=float(t["avg_pooling"]),
                              value_precision=Precision(t.get("value_precision", "FP32")), index_skew=skew))
    return ModelSpec(tables=tuple(tabs), bottom_mlp_layers=tuple(tuple(x) for x in doc.get("bottom_mlp_layers", [])),
                     top_mlp_layers=tuple(tuple(x) for x in doc.get("top_mlp_layers", [])),
                     local_batch=int(doc.get("local_batch", 1)),
                     mflops_per_sample=float(doc.get("mflops_per_sample", 0.0)),
                     interaction_flops_per_sample=float(doc.get("interaction_flops_per_sample", 0.0)),
                     dense_param_bytes=int(doc.get("dense_param_bytes", 0)))


@dataclass(frozen=True)
class ModelSpec:
    """Embedding tables plus the per-worker batch (model.py:100-168); the
    dense-MLP fields are carried for interface parity only."""

    tables: tuple
    bottom_mlp_layers: tuple = ()
    top_mlp_layers: tuple = ()
    local_batch: int = 1
    mflops_per_sample: float = 0.0
    interaction_flops_per_sample: float = 0.0
    dense_param_bytes: int = 0

    @property
    def num_tables(self) -> int:
        return len(self.tables)

    @property
    def total_dim(self) -> int:
        return sum(t.dim for t in self.tables)

    def table_index(self, table_id: str) -> int:
        for i, t in enumerate(self.tables):
            if t.id == table_id:
                return i
        raise KeyError(table_id)


class LayoutTag(str, Enum):
    WTB = "WTB"
    TWB = "TWB"


@dataclass(frozen=True)
class GlobalBatchLayout:
    workers: int
    tables: int
    local_batch: int
    tag: LayoutTag


class CombinedBatch:
    """lengths[t, s] plus the concatenated table-major index buffer
    (model.py:301-358)."""

    def __init__(self, lengths, indices):
        lengths = np.asarray(lengths, dtype=np.int64)
        indices = np.asarray(indices, dtype=np.int64)
        if lengths.ndim != 2:
            raise InvalidValue("lengths", "must be a (tables, samples) matrix")
        if (lengths < 0).any():
            raise InvalidValue("lengths", "must be >= 0")
        if int(lengths.sum()) != indices.shape[0]:
            raise InvalidValue("indices", "total index count must equal the sum of lengths")
        self.lengths = lengths
        self.indices = indices
        self._table_offsets = np.zeros(lengths.shape[0] + 1, dtype=np.int64)
        np.cumsum(lengths.sum(axis=1), out=self._table_offsets[1:])

    @property
    def num_tables(self) -> int:
        return self.lengths.shape[0]

    @property
    def num_samples(self) -> int:
        return self.lengths.shape[1]

    def table_slice(self, t: int):
        lo, hi = self._table_offsets[t], self._table_offsets[t + 1]
        return self.lengths[t], self.indices[lo:hi]

    def validate_against(self, model) -> None:
        if self.num_tables != model.num_tables:
            raise InvalidValue("lengths", "table count does not match model")
        for t, table in enumerate(model.tables):
            _, idx = self.table_slice(t)
            bad = (idx < 0) | (idx >= table.num_rows)
            if bad.any():
                raise IndexOutOfRange(table.id, int(idx[np.argmax(bad)]))

    def __eq__(self, other) -> bool:
        return (hasattr(other, "lengths") and hasattr(other, "indices")
                and np.array_equal(self.lengths, other.lengths)
                and np.array_equal(self.indices, other.indices))


def lengths_to_offsets(lengths) -> np.ndarray:
    lengths = np.asarray(lengths, dtype=np.int64)
    out = np.zeros(lengths.shape[0] + 1, dtype=np.int64)
    np.cumsum(lengths, out=out[1:])
    return out


def offsets_to_lengths(offsets) -> np.ndarray:
    offsets = np.asarray(offsets, dtype=np.int64)
    if offsets.shape[0] == 0 or offsets[0] != 0 or (np.diff(offsets) < 0).any():
        raise NonMonotonicOffsets("offsets must start at 0 and be nondecreasing")
    return np.diff(offsets)


def gen_synthetic_batch(model, num_samples: int, seed: int) -> CombinedBatch:
    """Same RNG stream as model.py:384-421: per table, floor(L) plus a
    Bernoulli(frac L) extra id per sample, then uniform or Zipf ids."""
    if num_samples < 1:
        raise InvalidValue("num_samples", "must be >= 1")
    rng = np.random.default_rng(seed)
    T = len(model.tables)
    lengths = np.empty((T, num_samples), dtype=np.int64)
    parts = []
    for t, spec in enumerate(model.tables):
        whole = math.floor(spec.avg_pooling)
        extra = spec.avg_pooling - whole
        lens = np.full(num_samples, whole, dtype=np.int64)
        if extra > 0:
            lens += rng.random(num_samples) < extra
        lengths[t] = lens
        n = int(lens.sum())
        skew = getattr(spec, "index_skew", None)
        if skew is None or skew.kind.value == "uniform":
            parts.append(rng.integers(0, spec.num_rows, size=n, dtype=np.int64))
        else:
            if spec.num_rows > 10**7:
                raise InvalidValue(f"tables[{spec.id}].index_skew",
                                   "zipf trace generation supports at most 1e7 rows")
            w = np.arange(1, spec.num_rows + 1, dtype=np.float64) ** (-skew.alpha)
            w /= w.sum()
            parts.append(rng.choice(spec.num_rows, size=n, p=w).astype(np.int64))
    idx = np.concatenate(parts) if parts else np.empty(0, dtype=np.int64)
    return CombinedBatch(lengths, idx)


# ---------------------------------------------------------------------------
# optimizer state (embedding.py:24-129)


class OptimizerKind(str, Enum):
    SGD = "sgd"
    ROWWISE_ADAGRAD = "rowwise_adagrad"
    ADAGRAD = "adagrad"


@dataclass(frozen=True)
class OptimizerConfig:
    kind: OptimizerKind
    lr: float
    eps: float = 0.0

    def __post_init__(self):
        if not self.lr > 0:
            raise InvalidValue("lr", "must be > 0")
        if self.eps < 0:
            raise InvalidValue("eps", "must be >= 0")


class EmbeddingTable:
    """Values (H, D) float64 plus optional moment ((H,) or (H, D))."""

    def __init__(self, spec, values, moment=None, row_base: int = 0, col_base: int = 0):
        values = np.asarray(values, dtype=np.float64)
        if values.ndim != 2:
            raise InvalidValue("values", "must be a 2-D matrix")
        if moment is not None:
            moment = np.asarray(moment, dtype=np.float64)
            if moment.shape not in ((values.shape[0],), values.shape):
                raise InvalidValue("moment", "must be (H,) or (H, D)")
            if (moment < 0).any():
                raise InvalidValue("moment", "must be >= 0")
        self.spec = spec
        self.values = values
        self.moment = moment
        self.row_base = row_base
        self.col_base = col_base

    @property
    def num_rows(self) -> int:
        return self.values.shape[0]

    @property
    def dim(self) -> int:
        return self.values.shape[1]

    def copy(self) -> "EmbeddingTable":
        return EmbeddingTable(self.spec, self.values.copy(),
                              None if self.moment is None else self.moment.copy(),
                              self.row_base, self.col_base)


@dataclass(frozen=True)
class RowGradients:
    ids: np.ndarray
    grads: np.ndarray

    def __post_init__(self):
        if len(self.ids) != len(self.grads):
            raise InvalidValue("grads", "one gradient per row id required")
        if len(self.ids) > 1 and not (np.diff(self.ids) > 0).all():
            raise InvalidValue("ids", "must be strictly increasing")


def kind_value(kind) -> str:
    """Optimizer kind as its string value (accepts either package's enum)."""
    return kind.value if hasattr(kind, "value") else str(kind)


def moment_for(rows: int, dim: int, cfg) -> Optional[np.ndarray]:
    k = kind_value(cfg.kind)
    if k == "sgd":
        return None
    if k == "rowwise_adagrad":
        return np.zeros(rows, dtype=np.float64)
    return np.zeros((rows, dim), dtype=np.float64)


def build_tables(model, cfg, seed: int = 0, zero_init: bool = False) -> list:
    """Per-(seed, table) initialisation, same stream as embedding.py:110-129."""
    from .embedding import quantize_fp16_roundtrip

    out = []
    for t, spec in enumerate(model.tables):
        if zero_init:
            values = np.zeros((spec.num_rows, spec.dim), dtype=np.float64)
        else:
            values = np.random.default_rng([seed, t]).standard_normal((spec.num_rows, spec.dim))
            if spec.value_precision.value == "FP16":
                values, _ = quantize_fp16_roundtrip(values)
        out.append(EmbeddingTable(spec, values, moment_for(spec.num_rows, spec.dim, cfg)))
    return out
