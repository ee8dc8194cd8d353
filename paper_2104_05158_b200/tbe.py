"""Device-side operator layer: torch tensors in HBM -> libneob200 C ABI.

``TableGroup`` is the production embedding-bag operator: T tables resident
in HBM (one contiguous weight buffer, per-table views), their optimizer
state, and the device metadata one TBE launch needs.  Its forward is one
``neo_tbe_forward`` launch for all tables; its backward is the fused
sort / segment-reduce / optimizer sequence of ``neo_tbe_backward``.

The free functions wrap the layout kernels (bucketize, permute, offsets,
piece copies, block gathers, casts).  All calls are stream-ordered on the
current torch stream and never synchronise, except ``ErrorRecord.read``.
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi as capi
from .errors import IndexOutOfRange, InvalidValue

DTYPE_CODE = {
    torch.float32: capi.NEO_F32,
    torch.float16: capi.NEO_F16,
    torch.float64: capi.NEO_F64,
    torch.bfloat16: capi.NEO_BF16,
}
INDEX_CODE = {torch.int32: capi.NEO_I32, torch.int64: capi.NEO_I64}
OPTIM_CODE = {"sgd": capi.NEO_OPT_SGD, "rowwise_adagrad": capi.NEO_OPT_ROWWISE_ADAGRAD,
              "adagrad": capi.NEO_OPT_ADAGRAD}
POOL_CODE = {"sum": capi.NEO_POOL_SUM, "mean": capi.NEO_POOL_MEAN}
SORT_BITS = 24  # CUB onesweep: 8-bit digits, so <= 24-bit keys sort in 3 passes


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def acc_dtype(weight_dtype: torch.dtype) -> torch.dtype:
    """Accumulator / optimizer-state type: f64 for f64 tables, else f32."""
    return torch.float64 if weight_dtype == torch.float64 else torch.float32


class _Workspace:
    """Grow-only per-device scratch buffers (one per purpose)."""

    def __init__(self):
        self._bufs: dict = {}

    def get(self, key: str, nbytes: int, device) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        k = (key, str(device))
        b = self._bufs.get(k)
        if b is None or b.numel() < nbytes:
            b = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._bufs[k] = b
        return b


WORKSPACE = _Workspace()


class ErrorRecord:
    """Device-side neo_error (first bad index in buffer order)."""

    def __init__(self, device):
        self.buf = torch.empty(3, dtype=torch.int64, device=device)

    def reset(self) -> "ErrorRecord":
        capi.check(capi.lib().neo_error_reset(self.buf.data_ptr(), _stream()), "neo_error_reset")
        return self

    @property
    def ptr(self) -> int:
        return self.buf.data_ptr()

    def read(self):
        """(position, value, table) of the first bad index, or None (syncs)."""
        h = self.buf.cpu().numpy()
        if int(h[0]) == np.iinfo(np.int64).max:
            return None
        table = int(np.int32(h[2] & 0xFFFFFFFF))
        return int(h[0]), int(h[1]), table


def _u64_ptrs(tensors, device) -> torch.Tensor:
    return torch.tensor([0 if t is None else t.data_ptr() for t in tensors], dtype=torch.int64,
                        device=device)


def bucket_rule(h: int, n: int) -> bool:
    """Does a table of h rows with n ids get warp-sorted buckets (<= 2^10
    rows, <= 1280 ids on average)?  Else the bucketed path would fall back to
    its CTA sort, slower than the pipelined walk."""
    if not h or not n:
        return True
    sb = _bucket_bits(h, n)
    return sb <= 10 and n * (1 << sb) <= 1280 * h


def _bucket_bits(h: int, n: int, target: int = 1024) -> int:
    """Row bits per bucket bkt_setup_kernel picks for a table of h rows and n
    ids (tbe_bucket.cu: <= 2048 buckets, about `target` ids per bucket)."""
    s = 4
    while -(-h // (1 << s)) > 2048:
        s += 1
    hb = max(0, (h - 1).bit_length()) if h > 1 else 0
    while s < hb and n * (1 << s) < target * h:
        s += 1
    return s


class TableGroup:
    """T embedding tables sharing one TBE launch.

    rows/dims: per-table H_t, D_t.  weights: optional existing (H_t, D_t)
    tensors (e.g. shards); otherwise one contiguous HBM buffer is allocated
    and each table is a view into it.  optim: "sgd" | "rowwise_adagrad" |
    "adagrad" | None — determines the moment state allocated.
    """

    def __init__(self, rows: Sequence[int], dims: Sequence[int], dtype=torch.float32,
                 optim: Optional[str] = "rowwise_adagrad", device="cuda",
                 weights: Optional[Sequence[torch.Tensor]] = None,
                 moments: Optional[Sequence[Optional[torch.Tensor]]] = None,
                 table_ids: Optional[Sequence[str]] = None):
        if dtype not in (torch.float32, torch.float16, torch.float64):
            raise InvalidValue("dtype", "tables are stored as f32, f16 or f64")
        self.rows = [int(r) for r in rows]
        self.dims = [int(d) for d in dims]
        self.T = len(self.rows)
        self.dtype = dtype
        self.acc = acc_dtype(dtype)
        self.device = torch.device(device)
        self.optim = optim
        self.table_ids = list(table_ids) if table_ids is not None else [str(i) for i in range(self.T)]
        if weights is None:
            total = sum(r * d for r, d in zip(self.rows, self.dims))
            self._storage = torch.empty(total, dtype=dtype, device=self.device)
            self.weights, off = [], 0
            for r, d in zip(self.rows, self.dims):
                self.weights.append(self._storage[off:off + r * d].view(r, d))
                off += r * d
        else:
            self.weights = list(weights)
            for w, r, d in zip(self.weights, self.rows, self.dims):
                if w is None:  # gradient-only group (AGGREGATE / DENSE modes)
                    continue
                if tuple(w.shape) != (r, d) or w.dtype != dtype or not w.is_contiguous():
                    raise InvalidValue("weights", "must be contiguous (H, D) tensors of the group dtype")
        if moments is not None:
            self.moments = list(moments)
        elif optim in ("rowwise_adagrad", "adagrad"):
            self.moments = [
                torch.zeros(r if optim == "rowwise_adagrad" else (r, d), dtype=self.acc, device=self.device)
                for r, d in zip(self.rows, self.dims)
            ]
        else:
            self.moments = [None] * self.T
        self.row_offsets_h = np.concatenate(([0], np.cumsum(self.rows))).astype(np.int64)
        self.dim_offsets_h = np.concatenate(([0], np.cumsum(self.dims))).astype(np.int32)
        self.total_rows = int(self.row_offsets_h[-1])
        self.total_dim = int(self.dim_offsets_h[-1])
        self.max_dim = max(self.dims) if self.dims else 0
        self.row_offsets = torch.from_numpy(self.row_offsets_h).to(self.device)
        self.dim_offsets = torch.from_numpy(self.dim_offsets_h).to(self.device)
        self.weight_ptrs = _u64_ptrs(self.weights, self.device)
        self.moment_ptrs = _u64_ptrs(self.moments, self.device)

    # ------------------------------------------------------------------
    def forward(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, pooling: str = "sum",
                out: Optional[torch.Tensor] = None, out_dtype: Optional[torch.dtype] = None,
                err: Optional[ErrorRecord] = None) -> torch.Tensor:
        """Pooled (batch, sum D) output; offsets has T*batch+1 entries."""
        if out is None:
            od = out_dtype or (torch.float64 if self.dtype == torch.float64 else torch.float32)
            out = torch.empty((batch, self.total_dim), dtype=od, device=self.device)
        stride = out.stride(0) if out.dim() == 2 else self.total_dim
        rc = capi.lib().neo_tbe_forward(
            self.T, batch, self.row_offsets.data_ptr(), self.dim_offsets.data_ptr(), self.max_dim,
            self.weight_ptrs.data_ptr(), DTYPE_CODE[self.dtype], indices.data_ptr(),
            INDEX_CODE[indices.dtype], offsets.data_ptr(), POOL_CODE[pooling], out.data_ptr(),
            DTYPE_CODE[out.dtype], stride, err.ptr if err else None, _stream())
        capi.check(rc, "neo_tbe_forward")
        return out

    def forward_scatter(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, out_ptrs: torch.Tensor,
                        rows_per_dst: int, out_stride: int, out_dtype: torch.dtype, pooling: str = "sum",
                        err: Optional[ErrorRecord] = None) -> None:
        """Forward whose pooled row b is stored at out_ptrs[b // rows_per_dst]
        (row b % rows_per_dst, columns dim_offsets[t]..): with peer pointers
        this performs the pooled all-to-all inside the TBE epilogue."""
        rc = capi.lib().neo_tbe_forward_scatter(
            self.T, batch, self.row_offsets.data_ptr(), self.dim_offsets.data_ptr(), self.max_dim,
            self.weight_ptrs.data_ptr(), DTYPE_CODE[self.dtype], indices.data_ptr(), INDEX_CODE[indices.dtype],
            offsets.data_ptr(), POOL_CODE[pooling], out_ptrs.data_ptr(), rows_per_dst, DTYPE_CODE[out_dtype],
            out_stride, err.ptr if err else None, _stream())
        capi.check(rc, "neo_tbe_forward_scatter")

    def backward(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, grad: torch.Tensor,
                 mode: str = "update", optim: Optional[str] = None, lr: float = 0.0,
                 eps: float = 0.0, pooling: str = "sum", err: Optional[ErrorRecord] = None,
                 dense_grads: Optional[Sequence[torch.Tensor]] = None,
                 table_counts: Optional[Sequence[int]] = None, timers: Optional[dict] = None):
        """mode "update": fused aggregate + one optimizer step per touched row
        (in place); "aggregate": returns (ids, grads, count) with global row
        keys; "dense": accumulates into dense_grads (per table, pre-zeroed).
        table_counts: optional host per-table id counts; lets an UPDATE over
        more than 2^SORT_BITS rows run as sub-groups with shorter sort keys.
        The ids covered are offsets[0] .. offsets[T*batch]; indices may be a
        larger buffer, so its length is only used when table_counts is None."""
        n_idx = int(indices.numel()) if table_counts is None else int(sum(table_counts))
        out_ids = out_grads = out_count = None
        dense_ptrs = None
        mode_code = {"update": capi.NEO_BWD_UPDATE, "aggregate": capi.NEO_BWD_AGGREGATE,
                     "dense": capi.NEO_BWD_DENSE}[mode]
        if mode == "aggregate":
            out_ids = torch.empty(max(n_idx, 1), dtype=torch.int64, device=self.device)
            out_grads = torch.empty((max(n_idx, 1), max(self.max_dim, 1)), dtype=self.acc, device=self.device)
            out_count = torch.zeros(1, dtype=torch.int64, device=self.device)
        if mode == "dense":
            dense_ptrs = _u64_ptrs(dense_grads, self.device)
        optim = optim or self.optim or "sgd"
        stride = grad.stride(0) if grad.dim() == 2 else self.total_dim
        if mode in ("update", "dense"):  # layout promises that select the specialised fast paths
            vec = 16 // torch.empty(0, dtype=self.dtype).element_size()
            aligned = (all(d % vec == 0 for d in self.dims) and stride % vec == 0
                       and grad.data_ptr() % 16 == 0
                       and all(w is None or w.data_ptr() % 16 == 0 for w in self.weights)
                       and (mode != "dense" or all(g.data_ptr() % 16 == 0 for g in dense_grads)))
            if aligned:
                mode_code |= capi.NEO_BWD_FLAG_ALIGNED
                if all(d == 32 * vec for d in self.dims):
                    mode_code |= capi.NEO_BWD_FLAG_FULL_ROWS
        if self._bucketed(mode, batch, grad, stride, pooling, dense_grads, table_counts):
            # hand-written bucketed sort + fused reduce/optimizer over the whole group
            mode_code |= capi.NEO_BWD_FLAG_DIM8
            n_b = n_idx if table_counts is None else int(sum(table_counts))
            prep = getattr(self, "_prepared", None)
            self._prepared = None
            if (prep is not None and prep.get("bucketed") and mode == "update"
                    and prep["key"] == (indices.data_ptr(), offsets.data_ptr(), batch, n_b)):
                # the sort phase was issued by prepare_backward (side stream): APPLY only
                main = torch.cuda.current_stream(self.device)
                main.wait_event(prep["event"])
                if timers is not None:
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_APPLY,
                                    optim, lr, eps, pooling, err, 0, self.T, None, None, None, None, dense_ptrs, n_b,
                                    ws=prep["ws"])
                if timers is not None:
                    e1.record()
                    timers.setdefault("apply", []).append((e0, e1, 0, self.T))
                self._prep_side.wait_stream(main)  # the workspace is free again after APPLY
                return None
            wsb = capi.lib().neo_tbe_bucket_workspace_bytes(self.T, batch, max(n_b, 1), self.total_rows, self.max_dim)
            ws = WORKSPACE.get("tbe_bucket", wsb, self.device)
            if timers is None:
                self._backward_call(indices, offsets, batch, grad, stride, mode_code, optim, lr, eps, pooling, err,
                                    0, self.T, None, None, None, None, dense_ptrs, n_b, ws=ws)
                return None
            # timed: the sort phase and the fused update kernel as two calls
            self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_PREPARE, optim,
                                lr, eps, pooling, err, 0, self.T, None, None, None, None, dense_ptrs, n_b, ws=ws)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_APPLY, optim,
                                lr, eps, pooling, err, 0, self.T, None, None, None, None, dense_ptrs, n_b, ws=ws)
            e1.record()
            timers.setdefault("apply", []).append((e0, e1, 0, self.T))
            return None
        prep = getattr(self, "_prepared", None)
        if (mode == "update" and prep is not None and prep["key"] == (indices.data_ptr(), offsets.data_ptr(), batch)
                and table_counts is not None):
            # keys + sorts were issued by prepare_backward (side stream, e.g. under the forward)
            self._prepared = None
            self._backward_apply_prepared(prep, indices, offsets, batch, grad, stride, mode_code, optim, lr, eps,
                                          pooling, err, table_counts, timers)
            return None
        if mode == "update" and table_counts is not None and self.total_rows >= (1 << SORT_BITS):
            # rows of the whole group need > SORT_BITS key bits: run sub-groups whose
            # rows fit, so each radix sort needs one pass fewer (same results: the
            # groups' row sets are disjoint and each row is still updated once)
            groups = self._sort_groups()
            if self._streamed(batch, stride, pooling) and len(groups) > 1:
                self._backward_pipelined(groups, indices, offsets, batch, grad, stride, mode_code, optim, lr,
                                         eps, pooling, err, table_counts, timers)
                return None
            for (t0, t1) in groups:
                self._backward_call(indices, offsets, batch, grad, stride, mode_code, optim, lr, eps, pooling,
                                    err, t0, t1, table_counts)
            return None
        self._backward_call(indices, offsets, batch, grad, stride, mode_code, optim, lr, eps, pooling, err, 0,
                            self.T, None, out_ids, out_grads, out_count, dense_ptrs, n_idx)
        if mode == "aggregate":
            return out_ids, out_grads, out_count
        return None

    def _bucketed(self, mode: str, batch: int, grad: torch.Tensor, stride: int, pooling: str,
                  dense_grads=None, table_counts=None) -> bool:
        """Mirror of the C side's bucketed-path condition (bkt_eligible):
        f32/f16 tables (f32 for DENSE), SUM, every D a multiple of 8 and
        <= 256, 16-byte aligned rows and gradient.  Also routes to the
        pipelined path groups with a table whose row buckets would span more
        than 2^10 rows or average more than 1280 ids (bkt_setup_kernel's
        rule, at most 2048 buckets per table): those buckets miss the
        warp-per-bucket sorts and take the CTA sort, which is slower than the
        pipelined walk (measured on c3 / c5 at 4 GPUs)."""
        if os.environ.get("NEO_BWD_VARIANT") in ("pipe", "stream"):
            return False
        force = getattr(self, "force_bucketed", None)  # a caller's decision for several groups at once
        if force is False:
            return False
        if table_counts is not None and os.environ.get("NEO_BWD_VARIANT") != "bucket" and force is None:
            if not all(bucket_rule(h, c) for h, c in zip(self.rows, table_counts)):
                return False  # CTA-sorted buckets (see below)
        if pooling != "sum" or mode not in ("update", "dense") or self.max_dim > 256 or self.T == 0:
            return False
        if self.dtype not in (torch.float32, torch.float16) or (mode == "dense" and self.dtype != torch.float32):
            return False
        if grad.dtype not in (torch.float32, torch.bfloat16, torch.float16):
            return False
        if any(d % 8 for d in self.dims) or stride % 8 or grad.data_ptr() % 16:
            return False
        if any(w is not None and w.data_ptr() % 16 for w in self.weights):
            return False
        if mode == "dense" and any(g.data_ptr() % 16 for g in dense_grads):
            return False
        s = 4
        while (self.total_rows + (1 << s) - 1) >> s > 2048:
            s += 1
        return s + max(1, (batch - 1).bit_length()) <= 32

    def prepare_backward(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, grad: torch.Tensor,
                         table_counts: Sequence[int], optim: Optional[str] = None, pooling: str = "sum",
                         err: Optional[ErrorRecord] = None) -> bool:
        """Issue the key build + radix sort of every sort sub-group of the
        next UPDATE backward over (indices, offsets) on a side stream, now.
        They depend on the ids only, so they can run under the forward (cap
        its residency with set_forward_residency so both fit on the SMs).
        `grad` is the upstream buffer the backward will receive (only its
        layout is used here).  The next backward() with the same indices and
        offsets then runs only the segment walks + optimizer.  Returns False
        (nothing issued) when the streamed path does not apply."""
        optim = optim or self.optim or "sgd"
        stride = grad.stride(0) if grad.dim() == 2 else self.total_dim
        if not self._streamed(batch, stride, pooling) or self.total_rows < 1:
            return False
        if self._bucketed("update", batch, grad, stride, pooling, table_counts=table_counts):
            # the bucketed sort phase (count, scan, stable scatter, per-bucket
            # row sort, batch records) reads only the ids and writes only its
            # workspace, so it may run under the forward on a side stream
            n_b = int(sum(table_counts))
            mode_code = capi.NEO_BWD_UPDATE | capi.NEO_BWD_FLAG_DIM8 | capi.NEO_BWD_FLAG_PREPARE
            wsb = capi.lib().neo_tbe_bucket_workspace_bytes(self.T, batch, max(n_b, 1), self.total_rows, self.max_dim)
            ws = WORKSPACE.get("tbe_bucket_prep", wsb, self.device)
            main = torch.cuda.current_stream(self.device)
            if getattr(self, "_prep_side", None) is None:
                self._prep_side = torch.cuda.Stream(device=self.device)
            side = self._prep_side
            side.wait_stream(main)
            with torch.cuda.stream(side):
                if n_b > 0:
                    self._backward_call(indices, offsets, batch, grad, stride, mode_code, optim, 0.05, 0.0, pooling, err,
                                        0, self.T, None, None, None, None, None, n_b, ws=ws)
                ev = torch.cuda.Event()
                ev.record(side)
            self._prepared = {"key": (indices.data_ptr(), offsets.data_ptr(), batch, n_b), "event": ev, "ws": ws,
                              "bucketed": True}
            return True
        groups = self._sort_groups() if self.total_rows >= (1 << SORT_BITS) else [(0, self.T)]
        if len(groups) == 1 and not hasattr(self, "_group_meta"):
            self._group_meta = {}
        if (0, self.T) in groups and (0, self.T) not in self._group_meta:
            self._group_meta[(0, self.T)] = self.row_offsets
        mode_code = capi.NEO_BWD_UPDATE | self._layout_flags(grad, stride)
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "_prep_side", None) is None:
            self._prep_side = torch.cuda.Stream(device=self.device)
        side = self._prep_side
        side.wait_stream(main)
        events, wss = [], []
        with torch.cuda.stream(side):
            for i, (t0, t1) in enumerate(groups):
                n = int(sum(table_counts[t0:t1]))
                rows = int(self.row_offsets_h[t1] - self.row_offsets_h[t0])
                wsb = capi.lib().neo_tbe_backward_workspace_bytes(max(n, 1), rows, self.max_dim)
                ws = WORKSPACE.get(f"tbe_bwd_prep{i}", wsb, self.device)
                if n > 0:
                    self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_PREPARE,
                                        optim, 0.05, 0.0, pooling, err, t0, t1, table_counts, ws=ws)
                ev = torch.cuda.Event()
                ev.record(side)
                events.append(ev)
                wss.append(ws)
        self._prepared = {"key": (indices.data_ptr(), offsets.data_ptr(), batch), "groups": groups,
                          "events": events, "ws": wss}
        return True

    def _layout_flags(self, grad: torch.Tensor, stride: int) -> int:
        vec = 16 // torch.empty(0, dtype=self.dtype).element_size()
        aligned = (all(d % vec == 0 for d in self.dims) and stride % vec == 0 and grad.data_ptr() % 16 == 0
                   and all(w is None or w.data_ptr() % 16 == 0 for w in self.weights))
        flags = 0
        if aligned:
            flags |= capi.NEO_BWD_FLAG_ALIGNED
            if all(d == 32 * vec for d in self.dims):
                flags |= capi.NEO_BWD_FLAG_FULL_ROWS
        return flags

    def _backward_apply_prepared(self, prep, indices, offsets, batch, grad, stride, mode_code, optim, lr, eps,
                                 pooling, err, table_counts, timers):
        main = torch.cuda.current_stream(self.device)
        for (t0, t1), ev, ws in zip(prep["groups"], prep["events"], prep["ws"]):
            main.wait_event(ev)
            if int(sum(table_counts[t0:t1])) == 0:
                continue
            if timers is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(main)
            self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_APPLY, optim,
                                lr, eps, pooling, err, t0, t1, table_counts, ws=ws)
            if timers is not None:
                e1.record(main)
                timers.setdefault("apply", []).append((e0, e1, t0, t1))
        # the side stream must not reuse these workspaces before the applies ran
        self._prep_side.wait_stream(main)

    def _sort_groups(self):
        """Consecutive table ranges whose total rows fit SORT_BITS-bit keys."""
        groups = getattr(self, "_groups", None)
        if groups is None:
            groups, t0, rows = [], 0, 0
            for t, r in enumerate(self.rows):
                if t > t0 and rows + r >= (1 << SORT_BITS):
                    groups.append((t0, t))
                    t0, rows = t, 0
                rows += r
            groups.append((t0, self.T))
            self._groups = groups
            self._group_meta = {}
            for g0, g1 in groups:  # device metadata of each sub-group (row offsets rebased)
                ro = torch.from_numpy(self.row_offsets_h[g0:g1 + 1] - self.row_offsets_h[g0]).to(self.device)
                self._group_meta[(g0, g1)] = ro
        return groups

    def _streamed(self, batch: int, stride: int, pooling: str) -> bool:
        """Mirror of the C side's streamed-path condition (f32/f16 tables,
        rows of <= 32 vectors, SUM, 32-bit upstream offsets)."""
        vec = 16 // torch.empty(0, dtype=self.dtype).element_size()
        return (self.dtype != torch.float64 and pooling == "sum" and self.max_dim <= 32 * vec
                and batch * stride < (1 << 32))

    def _backward_pipelined(self, groups, indices, offsets, batch, grad, stride, mode_code, optim, lr, eps,
                            pooling, err, table_counts, timers):
        """PREPARE (keys + sort) of sub-group g+1 on a side stream overlaps
        APPLY (segment walk + optimizer) of sub-group g on the caller's
        stream; two workspaces alternate."""
        main = torch.cuda.current_stream(self.device)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=self.device)
            self._free = [torch.cuda.Event(), torch.cuda.Event()]
        side = self._side
        nmax = max(int(sum(table_counts[t0:t1])) for t0, t1 in groups)
        rmax = max(int(self.row_offsets_h[t1] - self.row_offsets_h[t0]) for t0, t1 in groups)
        wsb = capi.lib().neo_tbe_backward_workspace_bytes(nmax, rmax, self.max_dim)
        wss = [WORKSPACE.get("tbe_bwd_a", wsb, self.device), WORKSPACE.get("tbe_bwd_b", wsb, self.device)]
        for e in self._free:
            e.record(main)
        side.wait_stream(main)  # ids, offsets and weights are ready
        prepared = []

        def prepare(i):
            t0, t1 = groups[i]
            with torch.cuda.stream(side):
                side.wait_event(self._free[i % 2])
                self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_PREPARE,
                                    optim, lr, eps, pooling, err, t0, t1, table_counts, ws=wss[i % 2])
                ev = torch.cuda.Event()
                ev.record(side)
                prepared.append(ev)

        prepare(0)
        for i, (t0, t1) in enumerate(groups):
            if i + 1 < len(groups):
                prepare(i + 1)
            main.wait_event(prepared[i])
            if timers is not None:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(main)
            self._backward_call(indices, offsets, batch, grad, stride, mode_code | capi.NEO_BWD_FLAG_APPLY, optim,
                                lr, eps, pooling, err, t0, t1, table_counts, ws=wss[i % 2])
            if timers is not None:
                e1.record(main)
                timers.setdefault("apply", []).append((e0, e1, t0, t1))
            self._free[i % 2].record(main)

    def _backward_call(self, indices, offsets, batch, grad, stride, mode_code, optim, lr, eps, pooling, err,
                       t0, t1, table_counts, out_ids=None, out_grads=None, out_count=None, dense_ptrs=None,
                       n_idx=None, ws=None):
        T = t1 - t0
        if table_counts is not None:
            n_idx = int(sum(table_counts[t0:t1]))
            ro = self._group_meta[(t0, t1)]
            total_rows = int(self.row_offsets_h[t1] - self.row_offsets_h[t0])
        else:
            ro, total_rows = self.row_offsets, self.total_rows
        if n_idx == 0:
            return
        if ws is None:
            ws_bytes = capi.lib().neo_tbe_backward_workspace_bytes(n_idx, total_rows, self.max_dim)
            ws = WORKSPACE.get("tbe_bwd", ws_bytes, self.device)
        i8, i4 = 8, 4
        rc = capi.lib().neo_tbe_backward(
            T, batch, ro.data_ptr(), total_rows, self.dim_offsets.data_ptr() + t0 * i4,
            self.max_dim, self.weight_ptrs.data_ptr() + t0 * i8, DTYPE_CODE[self.dtype],
            self.moment_ptrs.data_ptr() + t0 * i8, indices.data_ptr(), INDEX_CODE[indices.dtype],
            offsets.data_ptr() + t0 * batch * i8, n_idx, POOL_CODE[pooling], grad.data_ptr(),
            DTYPE_CODE[grad.dtype], stride, mode_code, OPTIM_CODE[optim], float(lr), float(eps), _ptr(out_ids),
            _ptr(out_grads), _ptr(out_count), _ptr(dense_ptrs), ws.data_ptr(), ws.numel(),
            err.ptr if err else None, _stream())
        capi.check(rc, "neo_tbe_backward")


# ---------------------------------------------------------------------------
# layout kernels


def set_forward_residency(ctas_per_sm: int) -> None:
    """Cap the TBE forward at ctas_per_sm CTAs per SM (0 = uncapped) so a
    side-stream prepare_backward() can co-reside with it."""
    capi.check(capi.lib().neo_set_forward_residency(int(ctas_per_sm)), "neo_set_forward_residency")


def lengths_to_offsets(lengths: torch.Tensor) -> torch.Tensor:
    """int64 offsets (n+1) of int64 lengths (model.py:365-370), on device."""
    n = int(lengths.numel())
    out = torch.empty(n + 1, dtype=torch.int64, device=lengths.device)
    ws_bytes = capi.lib().neo_scan_workspace_bytes(n)
    ws = WORKSPACE.get("scan", ws_bytes, lengths.device)
    capi.check(capi.lib().neo_lengths_to_offsets(n, lengths.data_ptr(), out.data_ptr(), ws.data_ptr(),
                                                 ws.numel(), _stream()), "neo_lengths_to_offsets")
    return out


def bucketize_rowwise(offsets: torch.Tensor, indices: torch.Tensor, starts: Sequence[int],
                      err: Optional[ErrorRecord] = None):
    """Row-wise bucketisation (comms.py:107-141) of n bags.

    starts: k+1 shard boundaries (host ints).  Returns (lengths (k, n),
    offsets (k*n+1), indices) with shard s's ids at
    indices[offsets[s*n]:offsets[(s+1)*n]], rebased to the shard."""
    n = int(offsets.numel()) - 1
    k = len(starts) - 1
    dev = indices.device
    out_len = torch.empty((k, n), dtype=torch.int64, device=dev)
    out_off = torch.empty(k * n + 1, dtype=torch.int64, device=dev)
    out_idx = torch.empty_like(indices)
    ws_bytes = capi.lib().neo_bucketize_workspace_bytes(n, k)
    ws = WORKSPACE.get("bucketize", ws_bytes, dev)
    starts_arr = np.asarray(starts, dtype=np.int64)
    st = starts_arr.ctypes.data_as(capi.C.POINTER(capi.C.c_int64))
    capi.check(capi.lib().neo_bucketize_rowwise(
        n, offsets.data_ptr(), indices.data_ptr(), INDEX_CODE[indices.dtype], k, st,
        out_len.data_ptr(), out_off.data_ptr(), out_idx.data_ptr(), -1,
        err.ptr if err else None, ws.data_ptr(), ws.numel(), _stream()), "neo_bucketize_rowwise")
    return out_len, out_off, out_idx


def permute_blocks(outer: int, inner: int, B: int, lengths: torch.Tensor, indices: torch.Tensor):
    """(outer, inner, B) block order -> (inner, outer, B) (comms.py:222-257)."""
    dev = lengths.device
    out_len = torch.empty_like(lengths)
    out_idx = torch.empty_like(indices)
    ws_bytes = capi.lib().neo_permute_workspace_bytes(outer, inner)
    ws = WORKSPACE.get("permute", ws_bytes, dev)
    capi.check(capi.lib().neo_permute_blocks(
        outer, inner, B, lengths.data_ptr(), indices.data_ptr(), INDEX_CODE[indices.dtype],
        out_len.data_ptr(), out_idx.data_ptr(), ws.data_ptr(), ws.numel(), _stream()),
        "neo_permute_blocks")
    return out_len, out_idx


@dataclass
class Piece:
    """One column block copy src[:, src_col:src_col+width] -> dst[:, dst_col:...]."""

    src: torch.Tensor
    dst: torch.Tensor
    src_col: int
    dst_col: int
    width: int
    accumulate: bool = False


class PackedPieces:
    """Device tables of a piece list: pieces cut into independent 16-byte
    chunks (neo_copy_chunks, lane-parallel) and the pieces that must stay
    ordered (accumulating ones and anything not 16-byte aligned)."""

    def __init__(self, chunks: Optional[torch.Tensor], n_chunks: int, rest: Optional[torch.Tensor], n_rest: int,
                 sd, dd):
        self.chunks, self.n_chunks, self.rest, self.n_rest, self.sd, self.dd = chunks, n_chunks, rest, n_rest, sd, dd


def copy_pieces(rows: int, pieces: Sequence[Piece], pieces_dev=None) -> None:
    """Apply pieces to rows [0, rows) (neo_copy_chunks + neo_copy_pieces):
    the same result as applying them in array order, given that overwriting
    pieces have disjoint destinations."""
    if not pieces:
        return
    if pieces_dev is None:
        pieces_dev = pack_pieces(pieces, pieces[0].src.device)
    pk = pieces_dev
    if pk.n_chunks:
        capi.check(capi.lib().neo_copy_chunks(rows, pk.chunks.data_ptr(), pk.n_chunks, DTYPE_CODE[pk.sd],
                                              DTYPE_CODE[pk.dd], _stream()), "neo_copy_chunks")
    if pk.n_rest:
        capi.check(capi.lib().neo_copy_pieces(rows, pk.rest.data_ptr(), pk.n_rest, DTYPE_CODE[pk.sd],
                                              DTYPE_CODE[pk.dd], _stream()), "neo_copy_pieces")


def _pieces_disjoint(pieces: Sequence[Piece]) -> bool:
    by_dst = {}
    for p in pieces:
        if not p.accumulate:
            by_dst.setdefault((p.dst.data_ptr(), p.dst.stride(0)), []).append((p.dst_col, p.dst_col + p.width))
    for iv in by_dst.values():
        iv.sort()
        if any(b[0] < a[1] for a, b in zip(iv, iv[1:])):
            return False
    return True


def pack_pieces(pieces: Sequence[Piece], device) -> PackedPieces:
    sd, dd = pieces[0].src.dtype, pieces[0].dst.dtype
    es, ed = pieces[0].src.element_size(), pieces[0].dst.element_size()
    V = 16 // min(es, ed)
    flat_ok = es <= 4 and ed <= 4 and _pieces_disjoint(pieces)
    chunks, rest = [], []
    for p in pieces:
        sa, da = p.src.data_ptr() + p.src_col * es, p.dst.data_ptr() + p.dst_col * ed
        ss, ds = p.src.stride(0) * es, p.dst.stride(0) * ed
        if (flat_ok and not p.accumulate and p.width % V == 0 and sa % 16 == 0 and da % 16 == 0
                and ss % 16 == 0 and ds % 16 == 0):
            for j in range(0, p.width, V):
                chunks.append((sa + j * es, da + j * ed, ss, ds))
        else:
            rest.append(p)
    ch = None
    if chunks:
        ch = torch.from_numpy(np.array(chunks, dtype=np.uint64).view(np.int64)).to(device)
    arr = None
    if rest:
        a = (capi.NeoPiece * len(rest))()
        for i, p in enumerate(rest):
            a[i] = capi.NeoPiece(p.src.data_ptr(), p.dst.data_ptr(), p.src.stride(0), p.dst.stride(0),
                                 p.src_col, p.dst_col, p.width, int(p.accumulate))
        arr = torch.from_numpy(np.frombuffer(bytes(a), dtype=np.uint8).copy()).to(device)
    return PackedPieces(ch, len(chunks), arr, len(rest), sd, dd)


def gather_blocks(srcs: Sequence[torch.Tensor], counts: Sequence[int], dst: torch.Tensor) -> torch.Tensor:
    """Concatenate the first counts[i] elements of each srcs[i] into dst
    (one launch; dst element size 4 or 8)."""
    n = len(srcs)
    if n == 0:
        return dst
    offs = np.concatenate(([0], np.cumsum(counts)[:-1])).astype(np.int64)
    meta = torch.tensor(np.stack([np.array([s.data_ptr() for s in srcs], dtype=np.int64),
                                  np.asarray(counts, dtype=np.int64), offs]),
                        dtype=torch.int64).to(dst.device)
    capi.check(capi.lib().neo_gather_blocks(n, meta[0].data_ptr(), meta[1].data_ptr(), meta[2].data_ptr(),
                                            dst.data_ptr(), dst.element_size(), _stream()),
               "neo_gather_blocks")
    return dst


def gather_blocks_dev(ptrs: torch.Tensor, counts: torch.Tensor, dst_offsets: torch.Tensor,
                      dst: torch.Tensor) -> torch.Tensor:
    """As gather_blocks, with the block table already on the device (int64
    source pointers, counts, destination offsets) — no host sync."""
    n = int(ptrs.numel())
    if n:
        capi.check(capi.lib().neo_gather_blocks(n, ptrs.data_ptr(), counts.data_ptr(), dst_offsets.data_ptr(),
                                                dst.data_ptr(), dst.element_size(), _stream()),
                   "neo_gather_blocks")
    return dst


def cast(x: torch.Tensor, dtype: torch.dtype, out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """RNE element-wise conversion on device (neo_cast)."""
    out = torch.empty(x.shape, dtype=dtype, device=x.device) if out is None else out
    capi.check(capi.lib().neo_cast(x.numel(), x.data_ptr(), DTYPE_CODE[x.dtype], out.data_ptr(),
                                   DTYPE_CODE[dtype], _stream()), "neo_cast")
    return out


def fp16_roundtrip_(x: torch.Tensor):
    """In-place f64 -> binary16 (RNE) -> f64; returns (overflow mask, nonfinite flag) device tensors."""
    assert x.dtype == torch.float64 and x.is_contiguous()
    ovf = torch.zeros(x.shape, dtype=torch.uint8, device=x.device)
    nonfinite = torch.zeros(1, dtype=torch.int32, device=x.device)
    capi.check(capi.lib().neo_fp16_roundtrip(x.numel(), x.data_ptr(), ovf.data_ptr(), nonfinite.data_ptr(),
                                             _stream()), "neo_fp16_roundtrip")
    return ovf, nonfinite


def apply_row_updates(weight: torch.Tensor, moment: Optional[torch.Tensor], ids: Optional[torch.Tensor],
                      grads: torch.Tensor, optim: str, lr: float, eps: float) -> None:
    """One optimizer step per listed row (embedding.py:212-267)."""
    n = int(grads.shape[0])
    capi.check(capi.lib().neo_apply_row_updates(
        n, _ptr(ids), grads.data_ptr(), int(weight.shape[1]), weight.data_ptr(),
        DTYPE_CODE[weight.dtype], _ptr(moment), OPTIM_CODE[optim], float(lr), float(eps), _stream()),
        "neo_apply_row_updates")


def check_indices(rows: torch.Tensor, offsets: torch.Tensor, indices: torch.Tensor, batch: int,
                  err: ErrorRecord) -> None:
    """Record the first id outside [0, rows[t]) of every table (device int64
    rows [T], offsets [T*batch+1]) in err (neo_check_indices); no sync."""
    T = int(rows.numel())
    capi.check(capi.lib().neo_check_indices(T, batch, rows.data_ptr(), offsets.data_ptr(), indices.data_ptr(),
                                            INDEX_CODE[indices.dtype], err.ptr, _stream()), "neo_check_indices")


def raise_if_bad(err: ErrorRecord, table_ids: Sequence[str]) -> None:
    """Raise the reference's IndexOutOfRange for the first bad id (syncs)."""
    r = err.read()
    if r is not None:
        _, value, table = r
        tid = table_ids[table] if 0 <= table < len(table_ids) else ""
        raise IndexOutOfRange(tid, value)
