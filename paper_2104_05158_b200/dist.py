"""Sharded embedding step across GPUs (one process per GPU, NCCL over NVLink).

The per-rank pipeline of one training step (reference semantics:
neosim/comms.py:292-353 alltoall_redistribute and comms.py:629-737
train_step_sharded):

  1. input exchange, two-phase (comms.py:292-353): every rank bucketises its
     local batch for row-wise shards on the device (neo_bucketize_rowwise),
     packs per-destination length blocks (static sizes) and id blocks (one
     device gather), exchanges lengths with all_to_all, then ids with
     all_to_all using the counts read back once per step;
  2. the received (W, S, B) blocks are permuted to (S, W, B) on the device
     (neo_permute_blocks) — each local shard now sees the global batch in
     sample order — and one fused TBE forward runs over all local shards;
  3. pooled all-to-all: rows [v*B, (v+1)*B) of the local output go to rank v
     (contiguous, zero-copy), optionally as fp16 written directly by the TBE
     epilogue; received column blocks are placed / summed (row-wise partial
     pools, in shard order) into the model-order pooled output by one
     neo_copy_pieces launch;
  4. the upstream gradient's column blocks are packed per destination
     (optionally bf16) and exchanged back; the receive buffer is already the
     (global batch, local columns) upstream of the local TBE backward, which
     runs fused with the optimizer;
  5. data-parallel tables: local forward on the local batch, dense gradient
     from the segment-reduce, NCCL all-reduce, identical update everywhere.

``Comm`` abstracts the collectives: ``NcclComm`` (torch.distributed, one
rank per process) and ``LocalComm`` (W logical ranks inside one process on
one GPU, collectives as device copies) — the latter runs the reference's
W-worker equivalence checks through exactly the same code.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import tbe
from .errors import LayoutMismatch
from .plan import RankLayout, rank_layout


# ---------------------------------------------------------------------------
# collectives


class Comm:
    """Collectives over the ranks this process drives (``ranks``)."""

    world: int
    ranks: list

    def all_to_all(self, outs, ins, out_splits, in_splits) -> None:  # pragma: no cover
        raise NotImplementedError

    def all_reduce_sum(self, tensors) -> None:  # pragma: no cover
        raise NotImplementedError


class NcclComm(Comm):
    """torch.distributed (NCCL on GPUs; gloo works for CPU tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.ranks = [dist.get_rank(group)]
        self.bytes_sent = 0

    def all_to_all(self, outs, ins, out_splits, in_splits) -> None:
        out, inp = outs[0], ins[0]
        self.bytes_sent += (sum(in_splits[0]) - in_splits[0][self.ranks[0]]) * inp.element_size()
        self.dist.all_to_all_single(out, inp, list(map(int, out_splits[0])), list(map(int, in_splits[0])),
                                    group=self.group)

    def all_reduce_sum(self, tensors) -> None:
        self.dist.all_reduce(tensors[0], group=self.group)


class LocalComm(Comm):
    """W logical ranks in one process: the all-to-all is a set of device
    copies, the all-reduce a rank-ordered sum (the reference's merge order,
    embedding.py:195-205)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))
        self.bytes_sent = 0

    def all_to_all(self, outs, ins, out_splits, in_splits) -> None:
        W = self.world
        ioff = [np.concatenate(([0], np.cumsum(s)))[:-1] for s in in_splits]
        ooff = [np.concatenate(([0], np.cumsum(s)))[:-1] for s in out_splits]
        for v in range(W):
            for w in range(W):
                n = int(in_splits[w][v])
                if n != int(out_splits[v][w]):
                    raise LayoutMismatch(f"all_to_all split mismatch {w}->{v}: {n} vs {out_splits[v][w]}")
                if n:
                    outs[v][ooff[v][w]:ooff[v][w] + n].copy_(ins[w][ioff[w][v]:ioff[w][v] + n])
                    if v != w:
                        self.bytes_sent += n * ins[w].element_size()

    def all_reduce_sum(self, tensors) -> None:
        acc = tensors[0].clone()
        for t in tensors[1:]:
            acc += t
        for t in tensors:
            t.copy_(acc)


# ---------------------------------------------------------------------------
# per-rank state


@dataclass
class RankState:
    rank: int
    group: Optional[tbe.TableGroup] = None       # local TW/RW/CW shards
    dp_group: Optional[tbe.TableGroup] = None    # replicated DP tables
    dp_dense: Optional[torch.Tensor] = None      # flat dense DP gradient buffer
    dp_dense_views: list = field(default_factory=list)
    # per-step scratch
    scratch: dict = field(default_factory=dict)


def _dtype_bytes(dt) -> int:
    return torch.empty(0, dtype=dt).element_size()


class ShardedEmbedding:
    """The embedding tables of a model, sharded by a reference plan.

    model: ModelSpec-like (tables with id/num_rows/dim); plan: ShardingPlan
    (reference or ours); comm: NcclComm / LocalComm; local_batch: B per rank.
    dtype: table storage (f32 / f16 production, f64 oracle-order).
    fwd_comm / bwd_comm: wire dtype of the pooled all-to-all (None = the
    compute dtype; torch.float16 / torch.bfloat16 for quantized comm,
    PAPER.md:656).
    """

    def __init__(self, model, plan, comm: Comm, local_batch: int, device=None, dtype=torch.float32,
                 optim: str = "rowwise_adagrad", fwd_comm: Optional[torch.dtype] = None,
                 bwd_comm: Optional[torch.dtype] = None, index_dtype=torch.int64,
                 init: Optional[Callable] = None):
        self.model = model
        self.lay: RankLayout = rank_layout(model, plan)
        if self.lay.world != comm.world:
            raise LayoutMismatch("plan worker count does not match the communicator")
        self.comm = comm
        self.W = comm.world
        self.B = local_batch
        self.n = self.W * local_batch
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.dtype = dtype
        self.acc = tbe.acc_dtype(dtype)
        self.optim = optim
        self.fwd_comm = fwd_comm or self.acc
        self.bwd_comm = bwd_comm or self.acc
        self.index_dtype = index_dtype
        self.T = len(model.tables)
        self.states = [self._make_state(r, init) for r in comm.ranks]

    # -- construction ----------------------------------------------------
    def _make_state(self, r: int, init) -> RankState:
        lay = self.lay
        st = RankState(rank=r)
        shards = lay.owned[r]
        if shards:
            st.group = tbe.TableGroup([s.num_rows for s in shards], [s.dim for s in shards], dtype=self.dtype,
                                      optim=self.optim, device=self.device,
                                      table_ids=[f"{s.table_id}#{s.index}" for s in shards])
            if init is not None:
                for s, w in zip(shards, st.group.weights):
                    w.copy_(init(s.table, s.rows, s.cols).to(w.dtype))
        if lay.dp_tables:
            st.dp_group = tbe.TableGroup([lay.rows[t] for t in lay.dp_tables], [lay.dims[t] for t in lay.dp_tables],
                                         dtype=self.dtype, optim=self.optim, device=self.device,
                                         table_ids=[lay.ids[t] for t in lay.dp_tables])
            if init is not None:
                for t, w in zip(lay.dp_tables, st.dp_group.weights):
                    w.copy_(init(t, (0, lay.rows[t]), (0, lay.dims[t])).to(w.dtype))
            total = sum(lay.rows[t] * lay.dims[t] for t in lay.dp_tables)
            st.dp_dense = torch.zeros(total, dtype=self.acc, device=self.device)
            off = 0
            for t in lay.dp_tables:
                sz = lay.rows[t] * lay.dims[t]
                st.dp_dense_views.append(st.dp_dense[off:off + sz].view(lay.rows[t], lay.dims[t]))
                off += sz
        return st

    # -- byte contract ---------------------------------------------------
    def pooled_send_bytes(self, rank: int, elem_bytes: Optional[int] = None) -> int:
        """Per-rank pooled all-to-all send bytes excluding self: sum over
        local shards of width x (n - B) x elem (comms.py:366-392 for TW/CW;
        row-wise partial pools ride the same exchange, (k-1)/k n D for k=W)."""
        e = elem_bytes or _dtype_bytes(self.fwd_comm)
        return self.lay.width(rank) * (self.n - self.B) * e

    # -- the step --------------------------------------------------------
    def step(self, batches: Sequence, lr: float, eps: float = 0.0,
             upstream_fn: Optional[Callable] = None, timers: Optional[dict] = None):
        """One training step.  batches[i] = (lengths (T, B) int64 numpy,
        ids device tensor, table-major) for local rank slot i.  Returns the
        pooled (B, sum D) outputs per local rank (model table order).
        upstream_fn(pooled) -> gradient (default: ones, the reference's
        sum-of-outputs loss)."""
        lay, W, B = self.lay, self.W, self.B
        S = self.states
        # ---- phase 1: local bucketise + pack lengths
        for st, (lengths, ids) in zip(S, batches):
            self._pack_lengths(st, np.asarray(lengths, dtype=np.int64), ids)
        self.comm.all_to_all([st.scratch["recv_len"] for st in S], [st.scratch["send_len"] for st in S],
                             [st.scratch["len_out_splits"] for st in S], [st.scratch["len_in_splits"] for st in S])
        # ---- phase 2: counts (one host sync for all local ranks)
        cnts = []
        for st in S:
            nS = len(lay.owned[st.rank])
            rl = st.scratch["recv_len"].view(W, nS * B) if nS else None
            recv = rl.sum(dim=1) if nS else torch.zeros(W, dtype=torch.int64, device=self.device)
            cnts.append(torch.cat([st.scratch["send_counts"], recv]))
        host = torch.stack(cnts).cpu().numpy()
        for st, h in zip(S, host):
            st.scratch["idx_in_splits"] = h[:W].tolist()
            st.scratch["idx_out_splits"] = h[W:].tolist()
            self._pack_ids(st)
        self.comm.all_to_all([st.scratch["recv_ids"] for st in S], [st.scratch["send_ids"] for st in S],
                             [st.scratch["idx_out_splits"] for st in S], [st.scratch["idx_in_splits"] for st in S])
        # ---- phase 3: permute + fused forward
        for st in S:
            self._forward_local(st)
        self.comm.all_to_all([st.scratch["recv_pool"] for st in S], [st.scratch["send_pool"] for st in S],
                             [st.scratch["pool_out_splits"] for st in S], [st.scratch["pool_in_splits"] for st in S])
        pooled = []
        for st in S:
            pooled.append(self._assemble(st))
        # ---- phase 4: upstream, backward exchange
        for st, p in zip(S, pooled):
            g = upstream_fn(p) if upstream_fn is not None else torch.ones_like(p)
            self._pack_grad(st, g)
        self.comm.all_to_all([st.scratch["recv_grad"] for st in S], [st.scratch["send_grad"] for st in S],
                             [st.scratch["grad_out_splits"] for st in S], [st.scratch["grad_in_splits"] for st in S])
        for st in S:
            self._backward_local(st, lr, eps)
        if lay.dp_tables:
            self.comm.all_reduce_sum([st.dp_dense for st in S])
            for st in S:
                self._dp_update(st, lr, eps)
        return pooled

    def redistribute(self, batches: Sequence) -> list:
        """Run only the input exchange (phases 1-2 + permute) and return, per
        local rank, {"shards": {(table, shard index): (lengths, ids)},
        "dp": {table: (lengths, ids)}} as host arrays (comms.py:292-353)."""
        lay, W, B = self.lay, self.W, self.B
        S = self.states
        for st, (lengths, ids) in zip(S, batches):
            self._pack_lengths(st, np.asarray(lengths, dtype=np.int64), ids)
        self.comm.all_to_all([st.scratch["recv_len"] for st in S], [st.scratch["send_len"] for st in S],
                             [st.scratch["len_out_splits"] for st in S], [st.scratch["len_in_splits"] for st in S])
        cnts = []
        for st in S:
            nS = len(lay.owned[st.rank])
            recv = st.scratch["recv_len"].view(W, nS * B).sum(dim=1) if nS else \
                torch.zeros(W, dtype=torch.int64, device=self.device)
            cnts.append(torch.cat([st.scratch["send_counts"], recv]))
        host = torch.stack(cnts).cpu().numpy()
        for st, h in zip(S, host):
            st.scratch["idx_in_splits"] = h[:W].tolist()
            st.scratch["idx_out_splits"] = h[W:].tolist()
            self._pack_ids(st)
        self.comm.all_to_all([st.scratch["recv_ids"] for st in S], [st.scratch["send_ids"] for st in S],
                             [st.scratch["idx_out_splits"] for st in S], [st.scratch["idx_in_splits"] for st in S])
        res = []
        for st, (lengths, _) in zip(S, batches):
            sc = st.scratch
            shards = lay.owned[st.rank]
            nS = len(shards)
            out = {"shards": {}, "dp": {}}
            if nS:
                total = int(sum(sc["idx_out_splits"]))
                rl = sc["recv_len"][:W * nS * B]
                if total:
                    pl, pi = tbe.permute_blocks(W, nS, B, rl, sc["recv_ids"][:total])
                    pi = pi.cpu().numpy()
                else:
                    pl, _ = tbe.permute_blocks(W, nS, B, rl, torch.zeros(1, dtype=self.index_dtype, device=self.device))
                    pi = np.zeros(0, dtype=np.int64)
                pl = pl.cpu().numpy().reshape(nS, W * B)
                pos = 0
                for k, s in enumerate(shards):
                    c = int(pl[k].sum())
                    out["shards"][(s.table, s.index)] = (pl[k].copy(), pi[pos:pos + c].astype(np.int64))
                    pos += c
            ids_h = sc["ids"].cpu().numpy()
            tab_off = sc["tab_off"]
            for t in lay.dp_tables:
                out["dp"][t] = (np.asarray(lengths[t], dtype=np.int64).copy(),
                                ids_h[int(tab_off[t]):int(tab_off[t + 1])].astype(np.int64))
            res.append(out)
        return res

    # -- phase helpers ---------------------------------------------------
    def _pack_lengths(self, st: RankState, lengths: np.ndarray, ids: torch.Tensor) -> None:
        lay, W, B, T = self.lay, self.W, self.B, self.T
        dev = self.device
        if lengths.shape != (T, B):
            raise LayoutMismatch(f"rank {st.rank}: lengths must be ({T}, {B})")
        sc = st.scratch
        ids = ids.to(dev)
        if int(ids.numel()) != int(lengths.sum()):
            raise LayoutMismatch("lengths do not cover the index buffer")
        sc["ids"] = ids
        cnt = lengths.sum(axis=1)
        tab_off = np.concatenate(([0], np.cumsum(cnt)))
        sc["tab_off"] = tab_off
        L_dev = torch.from_numpy(lengths.reshape(-1)).to(dev)
        sc["L_dev"] = L_dev
        es = ids.element_size()
        # row-wise tables: bucketise this rank's block once per table
        rw = {}
        for t, bounds in lay.rw_bounds.items():
            starts = [b[0] for b in bounds] + [bounds[-1][1]]
            sub = ids[int(tab_off[t]):int(tab_off[t + 1])]
            off_t = tbe.lengths_to_offsets(L_dev[t * B:(t + 1) * B])
            if sub.numel() == 0:
                sub = torch.zeros(1, dtype=ids.dtype, device=dev)
            rw[t] = tbe.bucketize_rowwise(off_t, sub, starts)
        sc["rw"] = rw
        # blocks in send order: destination-major, then the destination's shards
        len_srcs, blk_ptr, blk_cnt, dest_of_blk = [], [], [], []
        for v in range(W):
            for s in lay.owned[v]:
                if s.kind == "row_wise":
                    j = lay.rw_bounds[s.table].index(s.rows)
                    o_len, o_off, o_idx = rw[s.table]
                    len_srcs.append(o_len[j])
                    lo = o_off[j * B]
                    blk_ptr.append(o_idx.data_ptr() + lo * es)
                    blk_cnt.append(o_off[(j + 1) * B] - lo)
                else:
                    len_srcs.append(L_dev[s.table * B:(s.table + 1) * B])
                    blk_ptr.append(ids.data_ptr() + int(tab_off[s.table]) * es)
                    blk_cnt.append(int(cnt[s.table]))
                dest_of_blk.append(v)
        nsend = len(len_srcs)
        send_len = torch.empty(max(nsend * B, 1), dtype=torch.int64, device=dev)
        if nsend:
            tbe.gather_blocks(len_srcs, [B] * nsend, send_len)
        sc["send_len"] = send_len
        sc["len_in_splits"] = [len(lay.owned[v]) * B for v in range(W)]
        nS = len(lay.owned[st.rank])
        sc["recv_len"] = torch.empty(max(W * nS * B, 1), dtype=torch.int64, device=dev)
        sc["len_out_splits"] = [nS * B] * W
        # device block table for the id gather (counts of row-wise blocks live on the device)
        if nsend:
            cnt_dev = torch.stack([c if torch.is_tensor(c) else torch.tensor(c, device=dev) for c in blk_cnt])
            ptr_dev = torch.stack([p if torch.is_tensor(p) else torch.tensor(p, device=dev) for p in blk_ptr])
            dst_dev = torch.cumsum(cnt_dev, 0) - cnt_dev
            dest = torch.tensor(dest_of_blk, device=dev)
            send_counts = torch.zeros(W, dtype=torch.int64, device=dev).index_add_(0, dest, cnt_dev)
        else:
            cnt_dev = ptr_dev = dst_dev = None
            send_counts = torch.zeros(W, dtype=torch.int64, device=dev)
        sc["blk"] = (ptr_dev, cnt_dev, dst_dev)
        sc["send_counts"] = send_counts

    def _pack_ids(self, st: RankState) -> None:
        sc = st.scratch
        dev = self.device
        total_send = int(sum(sc["idx_in_splits"]))
        total_recv = int(sum(sc["idx_out_splits"]))
        sc["send_ids"] = torch.empty(max(total_send, 1), dtype=self.index_dtype, device=dev)
        sc["recv_ids"] = torch.empty(max(total_recv, 1), dtype=self.index_dtype, device=dev)
        ptr, cnt, dst = sc["blk"]
        if ptr is not None and total_send:
            ids = sc["ids"]
            if ids.dtype != self.index_dtype:
                raise LayoutMismatch("ids dtype must match the engine's index dtype")
            tbe.gather_blocks_dev(ptr, cnt, dst, sc["send_ids"])

    def _forward_local(self, st: RankState) -> None:
        lay, W, B, n = self.lay, self.W, self.B, self.n
        sc = st.scratch
        dev = self.device
        shards = lay.owned[st.rank]
        nS = len(shards)
        width = lay.width(st.rank)
        sc["send_pool"] = torch.empty(max(n * width, 1), dtype=self.fwd_comm, device=dev)
        if nS:
            # (W, S, B) wire blocks -> (S, W, B): each shard sees the global batch in sample order
            total = int(sum(sc["idx_out_splits"]))
            rl = sc["recv_len"][:W * nS * B]
            ri = sc["recv_ids"][:max(total, 1)]
            if total == 0:
                perm_len, _ = tbe.permute_blocks(W, nS, B, rl, torch.zeros(1, dtype=self.index_dtype, device=dev))
                perm_ids = ri
            else:
                perm_len, perm_ids = tbe.permute_blocks(W, nS, B, rl, ri)
            off = tbe.lengths_to_offsets(perm_len)
            sc["perm_ids"], sc["perm_off"] = perm_ids, off
            out = sc["send_pool"][:n * width].view(n, width)
            st.group.forward(perm_ids, off, n, out=out)
        sc["pool_in_splits"] = [B * width] * W
        widths = [lay.width(w) for w in range(W)]
        sc["pool_out_splits"] = [B * wd for wd in widths]
        sc["recv_pool"] = torch.empty(max(B * sum(widths), 1), dtype=self.fwd_comm, device=dev)
        # data-parallel tables: local batch only
        if st.dp_group is not None:
            ids, tab_off, L_dev = sc["ids"], sc["tab_off"], sc["L_dev"]
            dp = lay.dp_tables
            cnts = [int(tab_off[t + 1] - tab_off[t]) for t in dp]
            dp_ids = torch.empty(max(sum(cnts), 1), dtype=ids.dtype, device=dev)
            tbe.gather_blocks([ids[int(tab_off[t]):] if cnts[i] else ids for i, t in enumerate(dp)], cnts, dp_ids)
            dp_len = torch.empty(len(dp) * B, dtype=torch.int64, device=dev)
            tbe.gather_blocks([L_dev[t * B:(t + 1) * B] for t in dp], [B] * len(dp), dp_len)
            dp_off = tbe.lengths_to_offsets(dp_len)
            sc["dp_ids"], sc["dp_off"] = dp_ids, dp_off
            sc["dp_out"] = st.dp_group.forward(dp_ids, dp_off, B, out_dtype=self.acc)

    def _assemble(self, st: RankState) -> torch.Tensor:
        """Place received column blocks (TW copy, CW column placement, RW
        partial sum in shard order: comms.py:692-711) into model order."""
        lay, W, B = self.lay, self.W, self.B
        sc = st.scratch
        dev = self.device
        pooled = torch.empty((B, lay.total_dim), dtype=self.acc, device=dev)
        widths = [lay.width(w) for w in range(W)]
        starts = np.concatenate(([0], np.cumsum([B * wd for wd in widths])))
        views = [sc["recv_pool"][int(starts[w]):int(starts[w + 1])].view(B, widths[w]) if widths[w] else None
                 for w in range(W)]
        where = {}
        for w in range(W):
            for s in lay.owned[w]:
                where[(s.table, s.index)] = (w, s)
        pieces, dp_pieces = [], []
        dp_col = {t: c for t, c in zip(lay.dp_tables, np.concatenate(([0], np.cumsum([lay.dims[t] for t in lay.dp_tables])))[:-1])}
        for t in range(self.T):
            if t in dp_col:
                dp_pieces.append(tbe.Piece(sc["dp_out"], pooled, int(dp_col[t]), lay.model_cols[t], lay.dims[t]))
                continue
            idxs = sorted(i for (tt, i) in where if tt == t)
            for n_i, i in enumerate(idxs):
                w, s = where[(t, i)]
                acc = s.kind == "row_wise" and n_i > 0
                pieces.append(tbe.Piece(views[w], pooled, s.out_col, lay.model_cols[t] + s.cols[0], s.dim, acc))
        tbe.copy_pieces(B, pieces)
        tbe.copy_pieces(B, dp_pieces)
        return pooled

    def _pack_grad(self, st: RankState, grad: torch.Tensor) -> None:
        lay, W, B = self.lay, self.W, self.B
        sc = st.scratch
        dev = self.device
        grad = grad.contiguous()
        widths = [lay.width(v) for v in range(W)]
        send = torch.empty(max(B * sum(widths), 1), dtype=self.bwd_comm, device=dev)
        starts = np.concatenate(([0], np.cumsum([B * wd for wd in widths])))
        pieces = []
        for v in range(W):
            if not widths[v]:
                continue
            chunk = send[int(starts[v]):int(starts[v + 1])].view(B, widths[v])
            for s in lay.owned[v]:
                pieces.append(tbe.Piece(grad, chunk, lay.model_cols[s.table] + s.cols[0], s.out_col, s.dim))
        tbe.copy_pieces(B, pieces)
        sc["send_grad"] = send
        sc["grad_in_splits"] = [B * wd for wd in widths]
        me = lay.width(st.rank)
        sc["grad_out_splits"] = [B * me] * W
        sc["recv_grad"] = torch.empty(max(self.n * me, 1), dtype=self.bwd_comm, device=dev)
        if st.dp_group is not None:
            dpw = sum(lay.dims[t] for t in lay.dp_tables)
            g_dp = torch.empty((B, dpw), dtype=self.acc, device=dev)
            c = 0
            dp_pieces = []
            for t in lay.dp_tables:
                dp_pieces.append(tbe.Piece(grad, g_dp, lay.model_cols[t], c, lay.dims[t]))
                c += lay.dims[t]
            tbe.copy_pieces(B, dp_pieces)
            sc["dp_grad"] = g_dp

    def _backward_local(self, st: RankState, lr: float, eps: float) -> None:
        sc = st.scratch
        if st.group is not None and "perm_ids" in sc:
            me = self.lay.width(st.rank)
            g = sc["recv_grad"][:self.n * me].view(self.n, me)
            st.group.backward(sc["perm_ids"], sc["perm_off"], self.n, g, mode="update", optim=self.optim,
                              lr=lr, eps=eps)
        if st.dp_group is not None:
            st.dp_dense.zero_()
            st.dp_group.backward(sc["dp_ids"], sc["dp_off"], self.B, sc["dp_grad"], mode="dense",
                                 dense_grads=st.dp_dense_views)

    def _dp_update(self, st: RankState, lr: float, eps: float) -> None:
        for w, m, g in zip(st.dp_group.weights, st.dp_group.moments, st.dp_dense_views):
            tbe.apply_row_updates(w, m, None, g, self.optim, lr, eps)

    # -- state access ----------------------------------------------------
    def shard_tensors(self, rank_slot: int = 0):
        """[(LocalShard, weight, moment)] of a local rank."""
        st = self.states[rank_slot]
        shards = self.lay.owned[st.rank]
        if st.group is None:
            return []
        return list(zip(shards, st.group.weights, st.group.moments))
