"""Table checkpoints in the reference's NEOT format, dumped from and loaded
into HBM-resident tables (the reference's dump_table / load_table,
embedding.py:334-377; its CLI writes one ``tables/<id>.bin`` per table,
cli.py:350-357).

File layout (little endian): b"NEOT", then struct "<QQBB" = rows, dim,
precision code (FP32 = 0, FP16 = 1), moment code (none = 0, row-wise = 1,
element-wise = 2); then rows*dim f64 values (row-major) and the f64 moment
(rows or rows*dim).  The payload is always f64, so:

* f64 tables round-trip bit-exactly;
* f32 / f16 tables widen exactly on dump (every f32/f16 value is an f64)
  and narrow with round-to-nearest-even on load (``neo_cast``), i.e. a
  dump -> load cycle of an f32/f16 table is the identity.

Conversion runs on the device; host traffic goes through two pinned
staging buffers so the file I/O of one chunk overlaps the copy of the next.
"""
from __future__ import annotations

import struct
from pathlib import Path
from typing import BinaryIO, Optional

import torch

from . import tbe
from .errors import InvalidValue, MalformedDocument

MAGIC = b"NEOT"
_HDR = struct.Struct("<QQBB")
PRECISION_FP32, PRECISION_FP16 = 0, 1
MOMENT_NONE, MOMENT_ROWWISE, MOMENT_ELEMENTWISE = 0, 1, 2
CHUNK_BYTES = 64 << 20


def _moment_code(moment: Optional[torch.Tensor]) -> int:
    if moment is None:
        return MOMENT_NONE
    return MOMENT_ROWWISE if moment.dim() == 1 else MOMENT_ELEMENTWISE


class _Stager:
    """Two pinned f64 host buffers + one device f64 buffer per chunk size."""

    def __init__(self, device, chunk_bytes: int):
        self.n = max(chunk_bytes // 8, 1)
        self.host = [torch.empty(self.n, dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.dev = [torch.empty(self.n, dtype=torch.float64, device=device) for _ in range(2)]
        self.ev = [torch.cuda.Event() for _ in range(2)]

    def write(self, x: torch.Tensor, fh: BinaryIO) -> None:
        """Write device tensor x (any table dtype) as f64 bytes."""
        flat = x.reshape(-1)
        total = flat.numel()
        chunks = [(s, min(self.n, total - s)) for s in range(0, total, self.n)]
        pending = None  # (slot, m) whose D2H is in flight
        for i, (s, m) in enumerate(chunks):
            k = i % 2
            src = flat[s:s + m]
            d = self.dev[k][:m]
            if src.dtype == torch.float64:
                d.copy_(src)
            else:
                tbe.cast(src, torch.float64, out=d)
            self.host[k][:m].copy_(d, non_blocking=True)
            self.ev[k].record()
            if pending is not None:
                self._flush(*pending, fh)
            pending = (k, m)
        if pending is not None:
            self._flush(*pending, fh)

    def _flush(self, k: int, m: int, fh: BinaryIO) -> None:
        self.ev[k].synchronize()
        fh.write(memoryview(self.host[k].numpy()[:m]).cast("B"))

    def read(self, fh: BinaryIO, out: torch.Tensor) -> None:
        """Fill device tensor out (any table dtype) from f64 bytes."""
        flat = out.reshape(-1)
        total = flat.numel()
        for i, s in enumerate(range(0, total, self.n)):
            k = i % 2
            m = min(self.n, total - s)
            self.ev[k].synchronize()  # the H2D that last used this slot has finished
            buf = memoryview(self.host[k].numpy()[:m]).cast("B")
            got = fh.readinto(buf)
            if got != m * 8:
                raise MalformedDocument("truncated table checkpoint")
            d = self.dev[k][:m]
            d.copy_(self.host[k][:m], non_blocking=True)
            self.ev[k].record()
            if flat.dtype == torch.float64:
                flat[s:s + m].copy_(d)
            else:
                tbe.cast(d, flat.dtype, out=flat[s:s + m])
        torch.cuda.current_stream(out.device).synchronize()


def dump_tensor(fh: BinaryIO, values: torch.Tensor, moment: Optional[torch.Tensor] = None,
                precision: Optional[int] = None, chunk_bytes: int = CHUNK_BYTES) -> None:
    """Write one (H, D) device table (+ moment) as a NEOT record."""
    if values.dim() != 2:
        raise InvalidValue("values", "must be a 2-D matrix")
    if precision is None:
        precision = PRECISION_FP16 if values.dtype == torch.float16 else PRECISION_FP32
    fh.write(MAGIC)
    fh.write(_HDR.pack(values.shape[0], values.shape[1], precision, _moment_code(moment)))
    st = _Stager(values.device, chunk_bytes)
    st.write(values.contiguous(), fh)
    if moment is not None:
        st.write(moment.contiguous(), fh)


def read_header(fh: BinaryIO) -> tuple:
    """(rows, dim, precision code, moment code); raises MalformedDocument."""
    if fh.read(4) != MAGIC:
        raise MalformedDocument("bad table checkpoint magic")
    raw = fh.read(_HDR.size)
    if len(raw) != _HDR.size:
        raise MalformedDocument("truncated table checkpoint")
    return _HDR.unpack(raw)


def load_tensor(fh: BinaryIO, values: torch.Tensor, moment: Optional[torch.Tensor] = None,
                chunk_bytes: int = CHUNK_BYTES) -> int:
    """Read a NEOT record into existing device tensors (shape and moment
    kind must match: a resumed table keeps its optimizer state).  Returns
    the record's precision code."""
    rows, dim, prec, mcode = read_header(fh)
    if (rows, dim) != tuple(values.shape):
        raise InvalidValue("checkpoint", f"table is {tuple(values.shape)}, record is ({rows}, {dim})")
    if mcode != _moment_code(moment):
        raise InvalidValue("checkpoint.moment", f"record moment code {mcode}, table expects "
                           f"{_moment_code(moment)}")
    st = _Stager(values.device, chunk_bytes)
    st.read(fh, values)
    if moment is not None:
        st.read(fh, moment)
    return prec


# ---------------------------------------------------------------------------
# TableGroup / ShardedEmbedding helpers


def dump_group(group: "tbe.TableGroup", directory, precision: Optional[int] = None) -> list:
    """One ``<table id>.bin`` per table of the group (cli.py:350-357 layout)."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    paths = []
    for tid, w, m in zip(group.table_ids, group.weights, group.moments):
        p = d / f"{tid}.bin"
        with open(p, "wb") as fh:
            dump_tensor(fh, w, m, precision)
        paths.append(p)
    return paths


def load_group(group: "tbe.TableGroup", directory) -> None:
    d = Path(directory)
    for tid, w, m in zip(group.table_ids, group.weights, group.moments):
        with open(d / f"{tid}.bin", "rb") as fh:
            load_tensor(fh, w, m)


def _shard_name(table_id: str, index: int) -> str:
    return f"{table_id}.shard{index}.bin"


def dump_sharded(engine, directory) -> list:
    """Each rank of a ShardedEmbedding writes its own shards
    (``<id>.shard<k>.bin``: the shard's values and its moment, comms.py:605-626);
    DP tables are written once, by the rank that holds logical rank 0."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    paths = []
    for slot, st in enumerate(engine.states):
        for s, w, m in engine.shard_tensors(slot):
            p = d / _shard_name(s.table_id, s.index)
            with open(p, "wb") as fh:
                dump_tensor(fh, w, m)
            paths.append(p)
        if st.rank == 0 and st.dp_group is not None:
            paths += dump_group(st.dp_group, d)
    return paths


def load_sharded(engine, directory) -> None:
    d = Path(directory)
    for slot, st in enumerate(engine.states):
        for s, w, m in engine.shard_tensors(slot):
            with open(d / _shard_name(s.table_id, s.index), "rb") as fh:
                load_tensor(fh, w, m)
        if st.dp_group is not None:
            load_group(st.dp_group, d)


__all__ = ["MAGIC", "dump_tensor", "load_tensor", "read_header", "dump_group", "load_group",
           "dump_sharded", "load_sharded", "PRECISION_FP32", "PRECISION_FP16"]
