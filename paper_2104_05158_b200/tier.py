"""HBM tier over host-resident embedding tables.

The reference sizes this tier analytically: a plan whose shards exceed HBM is
classified ``hbm+dram`` (planner.py:512-522) and served at the harmonic blend
of the two bandwidths (cache.py:129-136), with a 32-way set-associative row
cache (cache.py:17-98) deciding residency.  Here the tier is real: each
table's rows and optimizer state live in pinned host memory that the GPU
addresses directly (UVA), a ``num_sets x ways`` slot cache per table lives in
HBM as an ordinary ``TableGroup``, and every batch is mapped onto slots by
``neo_tier_prepare`` (csrc/cache.cu) before the unchanged TBE forward and
fused backward run on the slots.  Evicted rows (values + moments) are written
back, missing rows fetched, in the same stream.  Rows a batch uses are never
evicted by it, so the same rows feed the same kernels as with the whole table
in HBM: results are bitwise identical on uniform ids, and within f32
summation order where hot rows are folded through 128-entry chunk partials
(their grouping follows slot order instead of row order;
tests/test_gpu_tier.py).
"""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np
import torch

from . import _capi as capi
from .errors import InvalidValue
from .tbe import INDEX_CODE, WORKSPACE, ErrorRecord, TableGroup, _stream, raise_if_bad


class TieredTableGroup:
    """spill: extra HBM slots per table for rows of sets that overflow their
    ways within one batch (default: ways x 256); they are fetched like misses
    and written back after the backward.  Only a batch that also exhausts
    the spill slots raises InvalidValue."""

    def __init__(self, rows: Sequence[int], dims: Sequence[int], num_sets, ways: int = 32,
                 dtype=torch.float32, optim: str = "rowwise_adagrad", device=None,
                 table_ids: Optional[Sequence[str]] = None, spill: Optional[int] = None):
        if ways < 1 or ways > 32:
            raise InvalidValue("ways", "1..32 (one way per lane)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.rows, self.dims, self.T = [int(r) for r in rows], [int(d) for d in dims], len(rows)
        self.num_sets = [int(num_sets)] * self.T if np.isscalar(num_sets) else [int(s) for s in num_sets]
        self.ways, self.optim, self.dtype = ways, optim, dtype
        self.table_ids = list(table_ids) if table_ids else [f"t{i}" for i in range(self.T)]
        slots = [s * ways for s in self.num_sets]
        self.spill = int(ways * 256 if spill is None else spill)
        if self.spill < 0:
            raise InvalidValue("spill", "must be >= 0")
        self.cache = TableGroup([n + self.spill for n in slots], self.dims, dtype=dtype, optim=optim,
                                device=self.device)
        self.spill_lists = [torch.zeros(2 * max(self.spill, 1), dtype=torch.int64, device=self.device)
                            for _ in range(self.T)]
        esz = torch.empty(0, dtype=dtype).element_size()
        self.row_bytes = [d * esz for d in self.dims]
        acc = self.cache.acc
        if optim == "rowwise_adagrad":
            self.host_m = [torch.zeros(r, dtype=acc, pin_memory=True) for r in self.rows]
            self.mom_bytes = [torch.empty(0, dtype=acc).element_size()] * self.T
        elif optim == "adagrad":
            self.host_m = [torch.zeros((r, d), dtype=acc, pin_memory=True) for r, d in zip(self.rows, self.dims)]
            self.mom_bytes = [d * torch.empty(0, dtype=acc).element_size() for d in self.dims]
        else:
            self.host_m = [None] * self.T
            self.mom_bytes = [0] * self.T
        self.host_w = [torch.zeros((r, d), dtype=dtype, pin_memory=True) for r, d in zip(self.rows, self.dims)]
        self.tags = [torch.full((n,), -1, dtype=torch.int64, device=self.device) for n in slots]
        self.stamps = [torch.zeros(n, dtype=torch.int32, device=self.device) for n in slots]
        self.stamp = 0
        self.counters = torch.zeros((self.T, 5), dtype=torch.int64, device=self.device)
        self.stats = {"misses": 0, "writebacks": 0, "accesses": 0, "spills": 0}
        self._slots = None

    # ------------------------------------------------------------------
    def map_batch(self, indices: torch.Tensor, table_counts: Sequence[int], err: Optional[ErrorRecord] = None):
        """Slot ids (int32, the layout of `indices`) of one batch; fetches and
        writes back rows as needed.  Rows of a set that needs more than `ways`
        rows in this batch take spill slots (up to 32 per set, `spill` per
        table); InvalidValue only when those run out, IndexOutOfRange on a bad
        id."""
        self.stamp += 1
        n = int(indices.numel())
        slots = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        own_err = err is None
        err = err or ErrorRecord(self.device).reset()
        off = np.concatenate(([0], np.cumsum(table_counts))).astype(np.int64)
        isz = indices.element_size()
        for t in range(self.T):
            cnt = int(off[t + 1] - off[t])
            if cnt == 0:
                continue
            ws = WORKSPACE.get("tier", capi.lib().neo_tier_workspace_bytes(cnt), self.device)
            m = self.cache.moments[t]
            rc = capi.lib().neo_tier_prepare_spill(
                self.rows[t], self.num_sets[t], self.ways, indices.data_ptr() + int(off[t]) * isz,
                INDEX_CODE[indices.dtype], cnt, self.tags[t].data_ptr(), self.stamps[t].data_ptr(), self.stamp,
                self.cache.weights[t].data_ptr(), None if m is None else m.data_ptr(), self.host_w[t].data_ptr(),
                None if self.host_m[t] is None else self.host_m[t].data_ptr(), self.row_bytes[t], self.mom_bytes[t],
                slots.data_ptr() + int(off[t]) * 4, self.counters[t].data_ptr(), self.spill,
                self.spill_lists[t].data_ptr(), ws.data_ptr(), ws.numel(), err.ptr, _stream())
            capi.check(rc, "neo_tier_prepare_spill")
        c = self.counters.cpu().numpy()
        if own_err:
            raise_if_bad(err, self.table_ids)
        if c[:, 2].sum() > 0:
            raise InvalidValue("num_sets", f"{int(c[:, 2].sum())} accesses found no free way: a set needs more than "
                                           f"{self.ways} rows in one batch and the {self.spill} spill slots "
                                           "(or 32 per set) are used up")
        self.stats["spills"] += int(c[:, 4].sum())
        self.stats["misses"] += int(c[:, 0].sum())
        self.stats["writebacks"] += int(c[:, 1].sum())
        self.stats["accesses"] += n
        self._slots = slots[:n]
        return self._slots

    def forward(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int, table_counts: Sequence[int],
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        slots = self.map_batch(indices, table_counts)
        return self.cache.forward(slots, offsets, batch, out=out)

    def backward(self, offsets: torch.Tensor, batch: int, grad: torch.Tensor, table_counts: Sequence[int],
                 lr: float, eps: float, optim: Optional[str] = None) -> None:
        """Fused backward + optimizer for the batch of the last forward()."""
        if self._slots is None:
            raise InvalidValue("backward", "no mapped batch: call forward() first")
        self.cache.backward(self._slots, offsets, batch, grad, mode="update", optim=optim or self.optim, lr=lr,
                            eps=eps, table_counts=table_counts)
        for t in range(self.T):  # spilled rows go home (their slots are per-batch)
            m = self.cache.moments[t]
            capi.check(capi.lib().neo_tier_spill_writeback(
                self.spill_lists[t].data_ptr(), self.counters[t].data_ptr(), self.spill,
                self.cache.weights[t].data_ptr(), None if m is None else m.data_ptr(), self.host_w[t].data_ptr(),
                None if self.host_m[t] is None else self.host_m[t].data_ptr(), self.row_bytes[t], self.mom_bytes[t],
                _stream()), "neo_tier_spill_writeback")

    def flush(self) -> None:
        """Write every cached row (and its optimizer state) back to host memory."""
        for t in range(self.T):
            m = self.cache.moments[t]
            rc = capi.lib().neo_tier_flush(self.tags[t].numel(), self.tags[t].data_ptr(),
                                           self.cache.weights[t].data_ptr(), None if m is None else m.data_ptr(),
                                           self.host_w[t].data_ptr(),
                                           None if self.host_m[t] is None else self.host_m[t].data_ptr(),
                                           self.row_bytes[t], self.mom_bytes[t], _stream())
            capi.check(rc, "neo_tier_flush")
        torch.cuda.current_stream(self.device).synchronize()


class HybridTableGroup:
    """Tables larger than HBM, split by rows (the reference's "hbm+dram"
    worker tier, planner.py:512-522): rows [0, hbm_rows[t]) of table t live
    in HBM (a TableGroup), the rest in host memory behind the slot cache
    (TieredTableGroup).  A batch is bucketised into the two row ranges in one
    launch (neo_bucketize_rowwise_multi), (table, part, bag) blocks are
    permuted to (part, table, bag) (neo_permute_blocks), each part runs the
    unchanged TBE kernels, and the pooled rows are the two partial sums added
    in part order, exactly as a row-wise table with two shards
    (comms.py:692-711).  Every row lives in one part and sees its
    occurrences in batch order, so updated weights and optimizer state are
    bitwise those of the whole table in HBM."""

    def __init__(self, rows: Sequence[int], dims: Sequence[int], hbm_rows: Sequence[int], num_sets, ways: int = 32,
                 dtype=torch.float32, optim: str = "rowwise_adagrad", device=None, spill: Optional[int] = None):
        self.rows, self.dims, self.T = [int(r) for r in rows], [int(d) for d in dims], len(rows)
        self.hbm_rows = [int(h) for h in hbm_rows]
        if any(not 0 < h < r for h, r in zip(self.hbm_rows, self.rows)):
            raise InvalidValue("hbm_rows", "each table needs rows in both parts (0 < hbm_rows < rows)")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.optim = optim
        self.hbm = TableGroup(self.hbm_rows, self.dims, dtype=dtype, optim=optim, device=self.device)
        self.host = TieredTableGroup([r - h for r, h in zip(self.rows, self.hbm_rows)], self.dims, num_sets, ways,
                                     dtype=dtype, optim=optim, device=self.device, spill=spill)
        st = np.zeros((self.T, 3), dtype=np.int64)
        st[:, 1] = self.hbm_rows
        st[:, 2] = self.rows
        self._tables = torch.arange(self.T, dtype=torch.int32, device=self.device)
        self._starts = torch.from_numpy(st.reshape(-1)).to(self.device)
        self._k = torch.full((self.T,), 2, dtype=torch.int32, device=self.device)
        self._parts = None

    def _split(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int):
        T, B, dev = self.T, batch, self.device
        lens = torch.empty(T * 2 * B, dtype=torch.int64, device=dev)
        offs = torch.empty(T * 2 * B + 1, dtype=torch.int64, device=dev)
        idx = torch.empty(max(int(indices.numel()), 1), dtype=indices.dtype, device=dev)
        ws = WORKSPACE.get("bucketize", capi.lib().neo_bucketize_workspace_bytes(T * B, 2), dev)
        capi.check(capi.lib().neo_bucketize_rowwise_multi(
            T, B, self._tables.data_ptr(), offsets.data_ptr(), indices.data_ptr(), INDEX_CODE[indices.dtype], 2,
            self._starts.data_ptr(), self._k.data_ptr(), lens.data_ptr(), offs.data_ptr(), idx.data_ptr(),
            ws.data_ptr(), ws.numel(), _stream()), "neo_bucketize_rowwise_multi")
        # (table, part, bag) -> (part, table, bag): each part's ids table-major
        from .tbe import lengths_to_offsets, permute_blocks
        plen, pidx = permute_blocks(T, 2, B, lens, idx)
        plen = plen.view(2, T * B)
        cnt = plen.view(2, T, B).sum(dim=2).cpu().numpy()  # host counts per (part, table)
        n0 = int(cnt[0].sum())
        off0 = lengths_to_offsets(plen[0])
        off1 = lengths_to_offsets(plen[1])
        return (pidx[:max(n0, 1)], off0, cnt[0].tolist()), (pidx[n0:], off1, cnt[1].tolist())

    def forward(self, indices: torch.Tensor, offsets: torch.Tensor, batch: int,
                out: Optional[torch.Tensor] = None) -> torch.Tensor:
        """Pooled (batch, sum D) outputs: HBM part + host part, in that order.
        offsets: int64 over T * batch bags (table-major, the CombinedBatch layout)."""
        p0, p1 = self._split(indices, offsets, batch)
        self._parts = (p0, p1)
        out = self.hbm.forward(p0[0], p0[1], batch, out=out)
        out += self.host.forward(p1[0], p1[1], batch, p1[2])
        return out

    def backward(self, batch: int, grad: torch.Tensor, lr: float, eps: float) -> None:
        """Fused backward + optimizer of both parts for the last forward()."""
        if self._parts is None:
            raise InvalidValue("backward", "no split batch: call forward() first")
        (i0, o0, c0), (_, o1, c1) = self._parts
        self.hbm.backward(i0, o0, batch, grad, mode="update", optim=self.optim, lr=lr, eps=eps, table_counts=c0)
        self.host.backward(o1, batch, grad, c1, lr=lr, eps=eps)

    def flush(self) -> None:
        self.host.flush()

    def row(self, t: int, r: int):
        """(weight row, optimizer state) of table t's row r, wherever it lives
        (call flush() first for host rows)."""
        h = self.hbm_rows[t]
        if r < h:
            m = self.hbm.moments[t]
            return self.hbm.weights[t][r].cpu(), None if m is None else m[r].cpu()
        m = self.host.host_m[t]
        return self.host.host_w[t][r - h], None if m is None else m[r - h]
