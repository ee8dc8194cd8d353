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
from .errors import IndexOutOfRange, LayoutMismatch
from .plan import RankLayout, rank_layout


# ---------------------------------------------------------------------------
# collectives


class Comm:
    """Collectives over the ranks this process drives (``ranks``).

    Byte accounting (the reference's byte contract, comms.py:366-540):
    ``sent[label][w]`` is what rank w sent to OTHER ranks through the
    collectives labelled ``label`` ("lengths", "ids", "pooled", "grad"),
    ``recv[label][w]`` what it received from them;
    ``reduced[label][w]`` the payload bytes rank w contributed to an
    all-reduce (ring traffic is 2(W-1)/W of it, comms.py:433-439)."""

    world: int
    ranks: list

    def _count(self, table: str, label: str, rank: int, nbytes: int) -> None:
        d = getattr(self, table, None)
        if d is None:
            d = {}
            setattr(self, table, d)
        d.setdefault(label, [0] * self.world)[rank] += int(nbytes)

    def all_to_all(self, outs, ins, out_splits, in_splits, async_op: bool = False,
                   label: str = "other"):  # pragma: no cover
        """Returns a handle with .wait() when async_op (None otherwise)."""
        raise NotImplementedError

    def all_reduce_sum(self, tensors, label: str = "other", async_op: bool = False):  # pragma: no cover
        """Sum over ranks in place; with async_op a handle with wait() (or None
        when already done)."""
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

    def all_to_all(self, outs, ins, out_splits, in_splits, async_op: bool = False, label: str = "other"):
        osp = [int(x) for x in out_splits[0]]
        isp = [int(x) for x in in_splits[0]]
        # persistent buffers may be larger than this step's payload
        out, inp = outs[0][:sum(osp)], ins[0][:sum(isp)]
        sent = (sum(isp) - isp[self.ranks[0]]) * inp.element_size()
        self.bytes_sent += sent
        self._count("sent", label, self.ranks[0], sent)
        self._count("recv", label, self.ranks[0], (sum(osp) - osp[self.ranks[0]]) * out.element_size())
        return self.dist.all_to_all_single(out, inp, osp, isp, group=self.group, async_op=async_op)

    def all_reduce_sum(self, tensors, label: str = "other", async_op: bool = False):
        self._count("reduced", label, self.ranks[0], tensors[0].numel() * tensors[0].element_size())
        return self.dist.all_reduce(tensors[0], group=self.group, async_op=async_op)


class LocalComm(Comm):
    """W logical ranks in one process: the all-to-all is a set of device
    copies, the all-reduce a rank-ordered sum (the reference's merge order,
    embedding.py:195-205)."""

    def __init__(self, world: int):
        self.world = world
        self.ranks = list(range(world))
        self.bytes_sent = 0

    def all_to_all(self, outs, ins, out_splits, in_splits, async_op: bool = False, label: str = "other"):
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
                        self._count("sent", label, w, n * ins[w].element_size())
                        self._count("recv", label, v, n * ins[w].element_size())

    def all_reduce_sum(self, tensors, label: str = "other", async_op: bool = False):
        for w, t in enumerate(tensors):
            self._count("reduced", label, w, t.numel() * t.element_size())
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
    group: Optional[tbe.TableGroup] = None       # first non-empty local group (None: no shards)
    groups: list = field(default_factory=list)   # local TW/RW/CW shards, one TableGroup per overlap group
    all_group: Optional[tbe.TableGroup] = None   # all local shards as one group (views)
    dp_group: Optional[tbe.TableGroup] = None    # replicated DP tables
    dp_dense: Optional[torch.Tensor] = None      # flat dense DP gradient buffer
    dp_dense_views: list = field(default_factory=list)
    bufs: dict = field(default_factory=dict)     # persistent device buffers (grow-only)
    cache: dict = field(default_factory=dict)    # packed piece tables keyed by buffer pointers
    sc: dict = field(default_factory=dict)       # per-step values


def _dtype_bytes(dt) -> int:
    return torch.empty(0, dtype=dt).element_size()


class ShardedEmbedding:
    """The embedding tables of a model, sharded by a reference plan.

    model: ModelSpec-like (tables with id/num_rows/dim); plan: ShardingPlan
    (reference or ours); comm: NcclComm / LocalComm; local_batch: B per rank.
    dtype: table storage (f32 / f16 production, f64 oracle-order).
    fwd_comm / bwd_comm: wire dtype of the pooled all-to-all (None = the
    accumulator dtype; torch.float16 / torch.bfloat16 for the paper's
    quantized communication).  Pooled outputs returned by
    ``step`` live in persistent buffers valid until the next step.
    """

    def __init__(self, model, plan, comm: Comm, local_batch: int, device=None, dtype=torch.float32,
                 optim: str = "rowwise_adagrad", fwd_comm: Optional[torch.dtype] = None,
                 bwd_comm: Optional[torch.dtype] = None, index_dtype=torch.int64,
                 init: Optional[Callable] = None, overlap_groups: int = 4, transport: str = "nccl"):
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
        lay = self.lay
        self.widths = [lay.width(w) for w in range(self.W)]
        # Local shards are split into G groups (same G on every rank: each group
        # is one all-to-all); group g's pooled rows form their own contiguous
        # block, so its exchange overlaps the TBE of group g+1 (and, backward,
        # the exchange of group g+1 overlaps the fused update of group g).
        from .plan import even_bounds

        self.G = max(1, min(overlap_groups, max(len(lay.owned[v]) for v in range(self.W)) or 1))
        self.gbounds, self.gwidth = [], []
        for v in range(self.W):
            bounds = even_bounds(len(lay.owned[v]), self.G) if lay.owned[v] else [(0, 0)] * self.G
            widths = []
            for g, (k0, k1) in enumerate(bounds):
                c = 0
                for s_ in lay.owned[v][k0:k1]:
                    s_.grp, s_.out_col = g, c
                    c += s_.dim
                widths.append(c)
            self.gbounds.append(bounds)
            self.gwidth.append(widths)
        # send order of input blocks: destination-major, then the destination's shards
        self.send_blocks = [(v, s) for v in range(self.W) for s in lay.owned[v]]
        self.rw_slot = {}
        for t, bounds in lay.rw_bounds.items():
            for s in (s for v in range(self.W) for s in lay.owned[v] if s.table == t):
                self.rw_slot[(t, s.index)] = bounds.index(s.rows)
        # every row-wise table is bucketised in ONE launch per step
        # (neo_bucketize_rowwise_multi): table r's shard boundaries padded to
        # kmax slots; send blocks located by (table, shard slot) -> flat block
        self.rw_tables = sorted(lay.rw_bounds)
        self.rw_kmax = max((len(b) for b in lay.rw_bounds.values()), default=1)
        self.rw_starts = np.zeros((len(self.rw_tables), self.rw_kmax + 1), dtype=np.int64)
        self.rw_k = np.zeros(len(self.rw_tables), dtype=np.int32)
        for r, t in enumerate(self.rw_tables):
            b = lay.rw_bounds[t]
            self.rw_starts[r, :len(b)] = [x[0] for x in b]
            self.rw_starts[r, len(b):] = b[-1][1]
            self.rw_k[r] = len(b)
        rpos = {t: r for r, t in enumerate(self.rw_tables)}
        self.blk_table = np.array([s.table for _, s in self.send_blocks], dtype=np.int64)
        self.blk_rw = np.array([s.kind == "row_wise" for _, s in self.send_blocks], dtype=bool)
        self.blk_flat = np.array([rpos[s.table] * self.rw_kmax + self.rw_slot[(s.table, s.index)]
                                  if s.kind == "row_wise" else 0 for _, s in self.send_blocks], dtype=np.int64)
        self.dp_cols = {}
        c = 0
        for t in lay.dp_tables:
            self.dp_cols[t] = c
            c += lay.dims[t]
        self.dp_width = c
        self.states = [self._make_state(r, init) for r in comm.ranks]
        # column of each shard inside its rank's full pooled row (all groups)
        for v in range(self.W):
            goff = np.concatenate(([0], np.cumsum(self.gwidth[v])))
            for s_ in lay.owned[v]:
                s_.chunk_col = int(goff[s_.grp]) + s_.out_col
        if transport not in ("nccl", "nvlink"):
            raise LayoutMismatch("transport must be 'nccl' or 'nvlink'")
        if transport == "nvlink" and not isinstance(comm, NcclComm):
            raise LayoutMismatch("the nvlink transport needs one process per GPU (NcclComm)")
        self.transport = transport
        if transport == "nvlink":
            self._init_symmetric()

    # -- construction ----------------------------------------------------
    def _make_state(self, r: int, init) -> RankState:
        lay = self.lay
        st = RankState(rank=r)
        for (k0, k1) in self.gbounds[r]:
            shards = lay.owned[r][k0:k1]
            if not shards:
                st.groups.append(None)
                continue
            grp = tbe.TableGroup([s.num_rows for s in shards], [s.dim for s in shards], dtype=self.dtype,
                                 optim=self.optim, device=self.device,
                                 table_ids=[f"{s.table_id}#{s.index}" for s in shards])
            if init is not None:
                for s, w in zip(shards, grp.weights):
                    w.copy_(init(s.table, s.rows, s.cols).to(w.dtype))
            st.groups.append(grp)
        st.group = next((g for g in st.groups if g is not None), None)
        # every local shard as ONE group (views of the overlap groups' tables):
        # the NVLink transport moves the whole exchange at once, so its forward
        # and fused backward run as single launches over all local shards
        live = [g for g in st.groups if g is not None]
        if len(live) > 1:
            shards = lay.owned[r]
            st.all_group = tbe.TableGroup([s.num_rows for s in shards], [s.dim for s in shards], dtype=self.dtype,
                                          optim=self.optim, device=self.device,
                                          weights=[w for g in live for w in g.weights],
                                          moments=[m for g in live for m in g.moments],
                                          table_ids=[f"{s.table_id}#{s.index}" for s in shards])
        else:
            st.all_group = st.group
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

    def _buf(self, st: RankState, name: str, numel: int, dtype) -> torch.Tensor:
        b = st.bufs.get(name)
        if b is None or b.numel() < max(numel, 1) or b.dtype != dtype:
            b = torch.empty(max(int(numel), 1), dtype=dtype, device=self.device)
            st.bufs[name] = b
        return b

    # -- NVLink transport (symmetric memory) ------------------------------
    def _init_symmetric(self) -> None:
        """Receive buffers every rank can store into over NVLink: pooled rows
        (B x sum_w width_w, source-major chunks) and upstream gradients
        (n x max width, source-major row blocks)."""
        import torch.distributed._symmetric_memory as symm

        W, B, n = self.W, self.B, self.n
        me = self.comm.ranks[0]
        group = self.comm.group if self.comm.group is not None else self.comm.dist.group.WORLD
        ef, eb = _dtype_bytes(self.fwd_comm), _dtype_bytes(self.bwd_comm)
        self._pool_elems = B * sum(self.widths)
        self._grad_elems = n * max(self.widths)
        self.sym_pool = symm.empty(max(self._pool_elems, 1), dtype=self.fwd_comm, device=self.device)
        self.sym_grad = symm.empty(max(self._grad_elems, 1), dtype=self.bwd_comm, device=self.device)
        self.hdl_pool = symm.rendezvous(self.sym_pool, group)
        self.hdl_grad = symm.rendezvous(self.sym_grad, group)
        src_off = np.concatenate(([0], np.cumsum([B * wd for wd in self.widths])))
        self.src_off = src_off
        ptrs = self.hdl_pool.buffer_ptrs
        # where my pooled rows land in every destination: my chunk of its receive buffer
        self.pool_dst = torch.tensor([ptrs[v] + int(src_off[me]) * ef for v in range(W)], dtype=torch.int64,
                                     device=self.device)
        self.group_col = np.concatenate(([0], np.cumsum(self.gwidth[me])))
        # remote gradient views: rows [me*B, (me+1)*B) of each owner's receive buffer
        self.grad_peer = [self.hdl_grad.get_buffer(v, (B, max(self.widths[v], 1)), self.bwd_comm,
                                                   me * B * max(self.widths[v], 1)) for v in range(W)]

    def _step_nvlink(self, st: RankState, lr: float, eps: float, upstream_fn, ev) -> torch.Tensor:
        lay, W, B, n = self.lay, self.W, self.B, self.n
        me = st.rank
        sc = st.sc
        ev.start("fwd")
        self._prepare_forward(st)
        if st.all_group is not None:
            st.all_group.forward_scatter(sc["perm_ids"], sc["perm_off"], n, self.pool_dst, B, self.widths[me],
                                         self.fwd_comm)
        self.hdl_pool.barrier(channel=0)  # every rank's rows have landed in every receive buffer
        ev.stop("fwd")
        pooled = self._assemble_sym(st)
        g = upstream_fn(pooled) if upstream_fn is not None else self._ones_like(st, pooled)
        ev.start("bwd")
        self._pack_grad_sym(st, g)
        # data-parallel tables first: their dense gradient's all-reduce then
        # runs (NCCL stream) under the sharded backward
        dp_handle = self._backward_dp_start(st)
        self.hdl_grad.barrier(channel=1)  # all upstream blocks have landed
        wd = self.widths[me]
        recv = self.sym_grad[:n * wd].view(n, wd) if wd else None
        if st.all_group is not None:
            st.all_group.backward(sc["perm_ids"], sc["perm_off"], n, recv, mode="update", optim=self.optim, lr=lr,
                                  eps=eps, table_counts=sc["shard_counts"])
        ev.stop("bwd")
        return pooled, dp_handle

    def _ones_like(self, st: RankState, p: torch.Tensor) -> torch.Tensor:
        g = self._buf(st, "ones", p.numel(), p.dtype)[:p.numel()].view_as(p)
        if st.cache.get("ones_ready") != g.data_ptr():
            g.fill_(1.0)
            st.cache["ones_ready"] = g.data_ptr()
        return g

    def _assemble_sym(self, st: RankState) -> torch.Tensor:
        lay, W, B = self.lay, self.W, self.B
        sc = st.sc
        pooled = self._buf(st, "pooled", B * lay.total_dim, self.acc)[:B * lay.total_dim].view(B, lay.total_dim)
        key = ("asm_sym", pooled.data_ptr(), sc["dp_out"].data_ptr() if "dp_out" in sc else 0)
        packed = st.cache.get(key)
        if packed is None:
            views = {w: self.sym_pool[int(self.src_off[w]):int(self.src_off[w + 1])].view(B, self.widths[w])
                     for w in range(W) if self.widths[w]}
            where = {(s.table, s.index): (w, s) for w in range(W) for s in lay.owned[w]}
            pieces, dp_pieces = [], []
            for t in range(self.T):
                if t in self.dp_cols:
                    dp_pieces.append(tbe.Piece(sc["dp_out"], pooled, self.dp_cols[t], lay.model_cols[t], lay.dims[t]))
                    continue
                for k, i in enumerate(sorted(i for (tt, i) in where if tt == t)):
                    w, s = where[(t, i)]
                    pieces.append(tbe.Piece(views[w], pooled, s.chunk_col, lay.model_cols[t] + s.cols[0], s.dim,
                                            s.kind == "row_wise" and k > 0))
            packed = [(pl, tbe.pack_pieces(pl, self.device) if pl else None) for pl in (pieces, dp_pieces)]
            st.cache[key] = packed
        for pl, dev_tab in packed:
            if pl:
                tbe.copy_pieces(B, pl, dev_tab)
        return pooled

    def _pack_grad_sym(self, st: RankState, grad: torch.Tensor) -> None:
        """Upstream columns of every owner's shards stored straight into the
        owner's receive buffer (peer stores over NVLink)."""
        lay, W, B = self.lay, self.W, self.B
        sc = st.sc
        grad = grad.contiguous()
        g_dp = None
        if st.dp_group is not None:
            g_dp = self._buf(st, "dp_grad", B * self.dp_width, self.acc)[:B * self.dp_width].view(B, self.dp_width)
            sc["dp_grad"] = g_dp
        key = ("grad_sym", grad.data_ptr(), 0 if g_dp is None else g_dp.data_ptr())
        packed = st.cache.get(key)
        if packed is None:
            pieces = []
            for v in range(W):
                for s in lay.owned[v]:
                    pieces.append(tbe.Piece(grad, self.grad_peer[v], lay.model_cols[s.table] + s.cols[0],
                                            s.chunk_col, s.dim))
            dp_pieces = [tbe.Piece(grad, g_dp, lay.model_cols[t], self.dp_cols[t], lay.dims[t])
                         for t in lay.dp_tables] if g_dp is not None else []
            packed = [(pl, tbe.pack_pieces(pl, self.device) if pl else None) for pl in (pieces, dp_pieces)]
            if len(st.cache) > 64:
                st.cache.clear()
            st.cache[key] = packed
        for pl, dev_tab in packed:
            if pl:
                tbe.copy_pieces(B, pl, dev_tab)

    # -- byte contract ---------------------------------------------------
    def pooled_send_bytes(self, rank: int, elem_bytes: Optional[int] = None) -> int:
        """Per-rank pooled all-to-all send bytes excluding self: sum over
        local shards of width x (n - B) x elem (comms.py:366-392 for TW/CW;
        row-wise partial pools ride the same exchange, (k-1)/k n D for k=W)."""
        e = elem_bytes or _dtype_bytes(self.fwd_comm)
        return self.widths[rank] * (self.n - self.B) * e

    # -- the step --------------------------------------------------------
    def _exchange_inputs(self, batches: Sequence) -> None:
        W, B = self.W, self.B
        S = self.states
        for st, bt in zip(S, batches):
            self._pack_lengths(st, bt)
        self.comm.all_to_all([st.sc["recv_len"] for st in S], [st.sc["send_len"] for st in S],
                             [[len(self.lay.owned[st.rank]) * B] * W for st in S],
                             [[len(self.lay.owned[v]) * B for v in range(W)] for st in S], label="lengths")
        cnts = []
        Smax = max(len(self.lay.owned[st.rank]) for st in S)
        for st in S:
            nS = len(self.lay.owned[st.rank])
            if nS:
                rl = st.sc["recv_len"][:W * nS * B].view(W, nS, B)
                recv = rl.sum(dim=(1, 2))
                per_shard = rl.sum(dim=(0, 2))
            else:
                recv = torch.zeros(W, dtype=torch.int64, device=self.device)
                per_shard = torch.zeros(0, dtype=torch.int64, device=self.device)
            pad = torch.zeros(Smax - nS, dtype=torch.int64, device=self.device)
            cnts.append(torch.cat([st.sc["send_counts"], recv, per_shard, pad, st.cache["err"].buf]))
        host = torch.stack(cnts).cpu().numpy()  # the one host sync of the step
        for st, h in zip(S, host):
            pos, val, tab = (int(x) for x in h[-3:])
            if pos != np.iinfo(np.int64).max:  # IndexOutOfRange before any table is touched
                table = int(np.int32(tab & 0xFFFFFFFF))
                raise IndexOutOfRange(self.model.tables[table].id if 0 <= table < self.T else "", val)
        for st, h in zip(S, host):
            nS = len(self.lay.owned[st.rank])
            st.sc["idx_in_splits"] = h[:W].tolist()
            st.sc["idx_out_splits"] = h[W:2 * W].tolist()
            st.sc["shard_counts"] = h[2 * W:2 * W + nS].tolist()
            self._pack_ids(st)
        self.comm.all_to_all([st.sc["recv_ids"] for st in S], [st.sc["send_ids"] for st in S],
                             [st.sc["idx_out_splits"] for st in S], [st.sc["idx_in_splits"] for st in S], label="ids")

    def step(self, batches: Sequence, lr: float, eps: float = 0.0,
             upstream_fn: Optional[Callable] = None, timers: Optional[dict] = None):
        """One training step.  batches[i] = (lengths (T, B) int64 host array,
        ids (table-major, device), optional lengths already on the device)
        for local rank slot i.  Returns the pooled (B, sum D) outputs per
        local rank (model table order).  upstream_fn(pooled) -> gradient
        (default: ones, the reference's sum-of-outputs loss).  timers: dict
        receiving CUDA event pairs for "inputs", "fwd", "a2a_fwd", "a2a_bwd", "bwd", "dp"."""
        W, B = self.W, self.B
        S = self.states
        ev = _Timers(timers)
        ev.start("inputs")
        self._exchange_inputs(batches)
        ev.stop("inputs")
        for st in S:
            self._route_backward(st)
        if self.transport == "nvlink":
            p0, dp_handle = self._step_nvlink(S[0], lr, eps, upstream_fn, ev)
            if self.lay.dp_tables:
                ev.start("dp")
                if dp_handle is not None:
                    dp_handle.wait()
                for st in S:
                    self._dp_update(st, lr, eps)
                ev.stop("dp")
            return [p0]
        ev.start("fwd")
        for st in S:
            self._prepare_forward(st)
        handles = []
        for g in range(self.G):  # TBE of group g, then its exchange (async) while group g+1 computes
            for st in S:
                self._forward_group(st, g)
            handles.append(self.comm.all_to_all(
                [st.sc["recv_pool"][g] for st in S], [st.sc["send_pool"][g] for st in S],
                [[B * self.gwidth[w][g] for w in range(W)] for st in S],
                [[B * self.gwidth[st.rank][g]] * W for st in S], async_op=True, label="pooled"))
        ev.stop("fwd")
        ev.start("a2a_fwd")
        for h in handles:
            if h is not None:
                h.wait()
        ev.stop("a2a_fwd")
        pooled = [self._assemble(st) for st in S]
        for st, p in zip(S, pooled):
            if upstream_fn is not None:
                g = upstream_fn(p)
            else:
                g = self._ones_like(st, p)
            self._pack_grad(st, g)
        ev.start("bwd")
        handles = [self.comm.all_to_all(
            [st.sc["recv_grad"][g] for st in S], [st.sc["send_grad"][g] for st in S],
            [[B * self.gwidth[st.rank][g]] * W for st in S],
            [[B * self.gwidth[v][g] for v in range(W)] for st in S], async_op=True, label="grad")
            for g in range(self.G)]
        dp_handle = None
        if self.lay.dp_tables:  # the DP all-reduce follows the gradient exchanges, under the sharded updates
            for st in S:
                self._backward_dp(st)
            dp_handle = self.comm.all_reduce_sum([st.dp_dense for st in S], label="dp", async_op=True)
        for g, h in enumerate(handles):  # update of group g while group g+1's gradients arrive
            if h is not None:
                h.wait()
            for st in S:
                self._backward_group(st, g, lr, eps)
        ev.stop("bwd")
        if self.lay.dp_tables:
            ev.start("dp")
            if dp_handle is not None:
                dp_handle.wait()
            for st in S:
                self._dp_update(st, lr, eps)
            ev.stop("dp")
        return pooled

    def redistribute(self, batches: Sequence) -> list:
        """Run only the input exchange (+ permute) and return, per local rank,
        {"shards": {(table, shard index): (lengths, ids)}, "dp": {table:
        (lengths, ids)}} as host arrays (comms.py:292-353)."""
        W, B = self.W, self.B
        self._exchange_inputs(batches)
        res = []
        for st, bt in zip(self.states, batches):
            lengths = bt[0]
            sc = st.sc
            shards = self.lay.owned[st.rank]
            nS = len(shards)
            out = {"shards": {}, "dp": {}}
            if nS:
                pl, pi, _ = self._permute_local(st)
                pl = pl.cpu().numpy().reshape(nS, W * B)
                pi = pi.cpu().numpy()
                pos = 0
                for k, s in enumerate(shards):
                    c = int(pl[k].sum())
                    out["shards"][(s.table, s.index)] = (pl[k].copy(), pi[pos:pos + c].astype(np.int64))
                    pos += c
            ids_h = sc["ids"].cpu().numpy()
            tab_off = sc["tab_off"]
            for t in self.lay.dp_tables:
                out["dp"][t] = (np.asarray(lengths[t], dtype=np.int64).copy(),
                                ids_h[int(tab_off[t]):int(tab_off[t + 1])].astype(np.int64))
            res.append(out)
        return res

    # -- phase helpers ---------------------------------------------------
    def _pack_lengths(self, st: RankState, bt) -> None:
        lay, W, B, T = self.lay, self.W, self.B, self.T
        dev = self.device
        lengths = np.asarray(bt[0], dtype=np.int64)
        ids = bt[1]
        if lengths.shape != (T, B):
            raise LayoutMismatch(f"rank {st.rank}: lengths must be ({T}, {B})")
        if int(ids.numel()) != int(lengths.sum()):
            raise LayoutMismatch("lengths do not cover the index buffer")
        if ids.dtype != self.index_dtype:
            raise LayoutMismatch("ids dtype must match the engine's index dtype")
        sc = st.sc
        ids = ids.to(dev)
        sc["ids"] = ids
        cnt = lengths.sum(axis=1)
        tab_off = np.concatenate(([0], np.cumsum(cnt)))
        sc["tab_off"] = tab_off
        L_dev = bt[2] if len(bt) > 2 and bt[2] is not None else torch.from_numpy(lengths.reshape(-1)).to(dev)
        sc["L_dev"] = L_dev
        # ids outside their table are caught here, before anything moves: the
        # first bad position rides the step's one host read (_exchange_inputs)
        err = st.cache.get("err")
        if err is None:
            err = tbe.ErrorRecord(dev)
            st.cache["err"] = err
            st.cache["rows_dev"] = torch.tensor([t.num_rows for t in self.model.tables], dtype=torch.int64,
                                                device=dev)
        err.reset()
        g_off = tbe.lengths_to_offsets(L_dev)
        if ids.numel():
            tbe.check_indices(st.cache["rows_dev"], g_off, ids, B, err)
        es = ids.element_size()
        nb = len(self.send_blocks)
        nS = len(lay.owned[st.rank])
        sc["recv_len"] = self._buf(st, "recv_len", W * nS * B, torch.int64)
        sc["send_len"] = self._buf(st, "send_len", nb * B, torch.int64)
        R, kmax = len(self.rw_tables), self.rw_kmax
        if R:  # bucketise this rank's block of every row-wise table, one launch
            meta = st.cache.get("rw_meta")
            if meta is None:
                meta = (torch.tensor(self.rw_tables, dtype=torch.int32, device=dev),
                        torch.from_numpy(self.rw_starts.reshape(-1)).to(dev),
                        torch.from_numpy(self.rw_k).to(dev))
                st.cache["rw_meta"] = meta
            rw_len = self._buf(st, "rw_len", R * kmax * B, torch.int64)[:R * kmax * B]
            rw_off = self._buf(st, "rw_off", R * kmax * B + 1, torch.int64)[:R * kmax * B + 1]
            n_rw = int(sum(cnt[t] for t in self.rw_tables))
            rw_idx = self._buf(st, "rw_idx", max(n_rw, 1), ids.dtype)
            ws = tbe.WORKSPACE.get("bucketize", tbe.capi.lib().neo_bucketize_workspace_bytes(R * B, kmax), dev)
            tbe.capi.check(tbe.capi.lib().neo_bucketize_rowwise_multi(
                R, B, meta[0].data_ptr(), g_off.data_ptr(), ids.data_ptr(), tbe.INDEX_CODE[ids.dtype], kmax,
                meta[1].data_ptr(), meta[2].data_ptr(), rw_len.data_ptr(), rw_off.data_ptr(), rw_idx.data_ptr(),
                ws.data_ptr(), ws.numel(), tbe._stream()), "neo_bucketize_rowwise_multi")
        if not nb:
            sc["send_counts"] = torch.zeros(W, dtype=torch.int64, device=dev)
            sc["blk"] = None
            return
        rwm, tabs = self.blk_rw, self.blk_table
        len_ptr = np.where(rwm, (rw_len.data_ptr() if R else 0) + self.blk_flat * B * 8, L_dev.data_ptr() + tabs * B * 8)
        ptr = np.where(rwm, rw_idx.data_ptr() if R else 0, ids.data_ptr() + tab_off[tabs] * es)
        cnt_h = np.where(rwm, 0, cnt[tabs])
        meta = torch.from_numpy(np.stack([len_ptr, np.full(nb, B, np.int64), np.arange(nb, dtype=np.int64) * B,
                                          ptr, cnt_h]).astype(np.int64)).to(dev, non_blocking=False)
        tbe.gather_blocks_dev(meta[0], meta[1], meta[2], sc["send_len"])
        ptr_dev, cnt_dev = meta[3].clone(), meta[4].clone()
        if R and rwm.any():  # row-wise block sizes / starts live on the device
            sel = st.cache.get("rw_sel")
            if sel is None:
                pos_h = np.nonzero(rwm)[0]
                sel = (torch.from_numpy(pos_h).to(dev), torch.from_numpy(self.blk_flat[pos_h] * B).to(dev),
                       torch.from_numpy((self.blk_flat[pos_h] + 1) * B).to(dev))
                st.cache["rw_sel"] = sel
            lo = rw_off.index_select(0, sel[1])
            hi = rw_off.index_select(0, sel[2])
            ptr_dev.index_add_(0, sel[0], lo * es)
            cnt_dev.index_copy_(0, sel[0], hi - lo)
        dst_dev = torch.cumsum(cnt_dev, 0) - cnt_dev
        dest = self._dest_index(st)
        sc["send_counts"] = torch.zeros(W, dtype=torch.int64, device=dev).index_add_(0, dest, cnt_dev)
        sc["blk"] = (ptr_dev, cnt_dev, dst_dev)

    def _dest_index(self, st: RankState) -> torch.Tensor:
        d = st.cache.get("dest")
        if d is None:
            d = torch.tensor([v for v, _ in self.send_blocks], dtype=torch.int64, device=self.device)
            st.cache["dest"] = d
        return d

    def _pack_ids(self, st: RankState) -> None:
        sc = st.sc
        total_send = int(sum(sc["idx_in_splits"]))
        total_recv = int(sum(sc["idx_out_splits"]))
        sc["send_ids"] = self._buf(st, "send_ids", total_send, self.index_dtype)
        sc["recv_ids"] = self._buf(st, "recv_ids", total_recv, self.index_dtype)
        if sc["blk"] is not None and total_send:
            tbe.gather_blocks_dev(*sc["blk"], sc["send_ids"])

    def _permute_local(self, st: RankState):
        """(W, S, B) received blocks -> (S, W, B): each local shard sees the
        global batch in sample order (comms.py:248-252)."""
        W, B = self.W, self.B
        sc = st.sc
        nS = len(self.lay.owned[st.rank])
        total = int(sum(sc["idx_out_splits"]))
        rl = sc["recv_len"][:W * nS * B]
        ri = sc["recv_ids"][:max(total, 1)]
        perm_len = self._buf(st, "perm_len", W * nS * B, torch.int64)[:W * nS * B]
        perm_ids = self._buf(st, "perm_ids", total, self.index_dtype)[:max(total, 1)]
        ws_bytes = tbe.capi.lib().neo_permute_workspace_bytes(W, nS)
        ws = tbe.WORKSPACE.get("permute", ws_bytes, self.device)
        tbe.capi.check(tbe.capi.lib().neo_permute_blocks(
            W, nS, B, rl.data_ptr(), ri.data_ptr(), tbe.INDEX_CODE[self.index_dtype], perm_len.data_ptr(),
            perm_ids.data_ptr(), ws.data_ptr(), ws.numel(), tbe._stream()), "neo_permute_blocks")
        off = tbe.lengths_to_offsets(perm_len)
        return perm_len, perm_ids, off

    def _prepare_forward(self, st: RankState) -> None:
        W, B, n = self.W, self.B, self.n
        sc = st.sc
        sc["send_pool"] = [self._buf(st, f"send_pool{g}", n * self.gwidth[st.rank][g], self.fwd_comm)
                           for g in range(self.G)]
        sc["recv_pool"] = [self._buf(st, f"recv_pool{g}", B * sum(self.gwidth[w][g] for w in range(W)),
                                     self.fwd_comm) for g in range(self.G)]
        if st.group is not None:
            _, perm_ids, off = self._permute_local(st)
            sc["perm_ids"], sc["perm_off"] = perm_ids, off
        if st.dp_group is not None:  # data-parallel tables: local batch only
            ids, tab_off, L_dev = sc["ids"], sc["tab_off"], sc["L_dev"]
            dp = self.lay.dp_tables
            cnts = [int(tab_off[t + 1] - tab_off[t]) for t in dp]
            dp_ids = self._buf(st, "dp_ids", sum(cnts), ids.dtype)
            tbe.gather_blocks([ids[int(tab_off[t]):] if cnts[i] else ids for i, t in enumerate(dp)], cnts, dp_ids)
            dp_len = self._buf(st, "dp_len", len(dp) * B, torch.int64)[:len(dp) * B]
            tbe.gather_blocks([L_dev[t * B:(t + 1) * B] for t in dp], [B] * len(dp), dp_len)
            sc["dp_ids"], sc["dp_off"] = dp_ids, tbe.lengths_to_offsets(dp_len)
            sc["dp_counts"] = cnts  # exact id counts: dp_ids is a grow-only buffer
            dp_out = self._buf(st, "dp_out", B * self.dp_width, self.acc)[:B * self.dp_width].view(B, self.dp_width)
            sc["dp_out"] = st.dp_group.forward(dp_ids, sc["dp_off"], B, out=dp_out)

    def _forward_group(self, st: RankState, g: int) -> None:
        grp = st.groups[g] if st.groups else None
        if grp is None:
            return
        n = self.n
        k0, _ = self.gbounds[st.rank][g]
        gw = self.gwidth[st.rank][g]
        sc = st.sc
        grp.forward(sc["perm_ids"], sc["perm_off"][k0 * n:], n, out=sc["send_pool"][g][:n * gw].view(n, gw))

    def _assemble(self, st: RankState) -> torch.Tensor:
        """Place received column blocks (TW copy, CW column placement, RW
        partial sums in shard order: comms.py:692-711) in model order."""
        lay, W, B = self.lay, self.W, self.B
        sc = st.sc
        pooled = self._buf(st, "pooled", B * lay.total_dim, self.acc)[:B * lay.total_dim].view(B, lay.total_dim)
        key = ("asm", tuple(b.data_ptr() for b in sc["recv_pool"]), pooled.data_ptr(),
               sc["dp_out"].data_ptr() if "dp_out" in sc else 0)
        packed = st.cache.get(key)
        if packed is None:
            views = {}
            for g in range(self.G):
                starts = np.concatenate(([0], np.cumsum([B * self.gwidth[w][g] for w in range(W)])))
                for w in range(W):
                    if self.gwidth[w][g]:
                        views[(w, g)] = sc["recv_pool"][g][int(starts[w]):int(starts[w + 1])].view(B, self.gwidth[w][g])
            where = {(s.table, s.index): (w, s) for w in range(W) for s in lay.owned[w]}
            pieces, dp_pieces = [], []
            for t in range(self.T):
                if t in self.dp_cols:
                    dp_pieces.append(tbe.Piece(sc["dp_out"], pooled, self.dp_cols[t], lay.model_cols[t], lay.dims[t]))
                    continue
                for k, i in enumerate(sorted(i for (tt, i) in where if tt == t)):
                    w, s = where[(t, i)]
                    pieces.append(tbe.Piece(views[(w, s.grp)], pooled, s.out_col, lay.model_cols[t] + s.cols[0],
                                            s.dim, s.kind == "row_wise" and k > 0))
            packed = [(pl, tbe.pack_pieces(pl, self.device) if pl else None) for pl in (pieces, dp_pieces)]
            st.cache[key] = packed
        for pl, dev_tab in packed:
            if pl:
                tbe.copy_pieces(B, pl, dev_tab)
        return pooled

    def _pack_grad(self, st: RankState, grad: torch.Tensor) -> None:
        lay, W, B, n = self.lay, self.W, self.B, self.n
        sc = st.sc
        grad = grad.contiguous()
        sends = [self._buf(st, f"send_grad{g}", B * sum(self.gwidth[v][g] for v in range(W)), self.bwd_comm)
                 for g in range(self.G)]
        sc["send_grad"] = sends
        sc["recv_grad"] = [self._buf(st, f"recv_grad{g}", n * self.gwidth[st.rank][g], self.bwd_comm)
                           for g in range(self.G)]
        g_dp = None
        if st.dp_group is not None:
            g_dp = self._buf(st, "dp_grad", B * self.dp_width, self.acc)[:B * self.dp_width].view(B, self.dp_width)
            sc["dp_grad"] = g_dp
        key = ("grad", grad.data_ptr(), tuple(x.data_ptr() for x in sends), 0 if g_dp is None else g_dp.data_ptr())
        packed = st.cache.get(key)
        if packed is None:
            pieces = []
            for g in range(self.G):
                starts = np.concatenate(([0], np.cumsum([B * self.gwidth[v][g] for v in range(W)])))
                for v in range(W):
                    gw = self.gwidth[v][g]
                    if not gw:
                        continue
                    chunk = sends[g][int(starts[v]):int(starts[v + 1])].view(B, gw)
                    k0, k1 = self.gbounds[v][g]
                    for s in lay.owned[v][k0:k1]:
                        pieces.append(tbe.Piece(grad, chunk, lay.model_cols[s.table] + s.cols[0], s.out_col, s.dim))
            dp_pieces = [tbe.Piece(grad, g_dp, lay.model_cols[t], self.dp_cols[t], lay.dims[t])
                         for t in lay.dp_tables] if g_dp is not None else []
            packed = [(pl, tbe.pack_pieces(pl, self.device) if pl else None) for pl in (pieces, dp_pieces)]
            if len(st.cache) > 64:
                st.cache.clear()
            st.cache[key] = packed
        for pl, dev_tab in packed:
            if pl:
                tbe.copy_pieces(B, pl, dev_tab)

    def _backward_group(self, st: RankState, g: int, lr: float, eps: float) -> None:
        grp = st.groups[g] if st.groups else None
        if grp is None:
            return
        n = self.n
        sc = st.sc
        k0, k1 = self.gbounds[st.rank][g]
        gw = self.gwidth[st.rank][g]
        grp.backward(sc["perm_ids"], sc["perm_off"][k0 * n:], n, sc["recv_grad"][g][:n * gw].view(n, gw),
                     mode="update", optim=self.optim, lr=lr, eps=eps, table_counts=sc["shard_counts"][k0:k1])

    def _route_backward(self, st: RankState) -> None:
        """One backward path for all of a rank's shard groups (the bucketed
        sort when every shard qualifies, else the pipelined walk), so the
        per-group launches (NCCL transport, LocalComm) and the single
        all-shards launch (NVLink transport) compute the same bits."""
        shards = self.lay.owned[st.rank]
        counts = st.sc.get("shard_counts", [])
        ok = all(tbe.bucket_rule(s.num_rows, int(c)) and s.dim % 8 == 0 and s.dim <= 256
                 for s, c in zip(shards, counts))
        for grp in list(st.groups or []) + [st.all_group]:
            if grp is not None:
                grp.force_bucketed = ok

    def _backward_dp(self, st: RankState) -> None:
        sc = st.sc
        if st.dp_group is not None:
            st.dp_dense.zero_()
            st.dp_group.backward(sc["dp_ids"], sc["dp_off"], self.B, sc["dp_grad"], mode="dense",
                                 dense_grads=st.dp_dense_views, table_counts=sc["dp_counts"])

    def _backward_dp_start(self, st: RankState):
        """One rank's data-parallel dense gradient, then its all-reduce issued
        asynchronously (one process per GPU); the caller waits before the
        update."""
        if not self.lay.dp_tables:
            return None
        self._backward_dp(st)
        return self.comm.all_reduce_sum([st.dp_dense], label="dp", async_op=True)

    def _dp_update(self, st: RankState, lr: float, eps: float) -> None:
        for w, m, g in zip(st.dp_group.weights, st.dp_group.moments, st.dp_dense_views):
            tbe.apply_row_updates(w, m, None, g, self.optim, lr, eps)

    # -- state access ----------------------------------------------------
    def shard_tensors(self, rank_slot: int = 0):
        """[(LocalShard, weight, moment)] of a local rank."""
        st = self.states[rank_slot]
        out = []
        for (k0, k1), grp in zip(self.gbounds[st.rank], st.groups):
            if grp is not None:
                out += list(zip(self.lay.owned[st.rank][k0:k1], grp.weights, grp.moments))
        return out


class _Timers:
    """CUDA event pairs per phase on the current stream (no-op if unused)."""

    def __init__(self, d: Optional[dict]):
        self.d = d

    def start(self, name: str) -> None:
        if self.d is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.d.setdefault(name, []).append([e, None])

    def stop(self, name: str) -> None:
        if self.d is not None:
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            self.d[name][-1][1] = e
