"""DLRM training step around the sharded embedding engine.

The dense part stays in PyTorch, as the north star says; what this module
adds is the step's dependency structure from the reference's cost model
(perf.py:110-145):

  fwd = max(bottom-MLP fwd, embedding lookup + pooled all-to-all)
        + interaction + top-MLP fwd
  bwd = top-MLP bwd + interaction bwd
        + max(grad all-to-all + embedding update, bottom-MLP bwd)
  dense all-reduce overlapped with the embedding backward.

Realisation on one GPU per rank:
* the bottom MLP runs on a side stream, launched before the embedding step,
  so it overlaps the TBE forward and the pooled exchange;
* the top of the model (interaction + top MLP + BCE loss) runs inside the
  engine's ``upstream_fn`` — it receives the pooled embeddings and returns
  their gradient, and autograd also queues the bottom MLP's backward on the
  side stream, which then overlaps the engine's gradient exchange and fused
  TBE backward/AdaGrad;
* the dense gradients of all ranks are summed by one bucketed NCCL
  all-reduce issued as soon as the dense backward is queued;
* dense SGD via ``torch._foreach`` ops.  The dense MLP + interaction are
  captured as CUDA graphs (``torch.cuda.make_graphed_callables``) when
  ``graphs=True`` — the embedding step itself has a host-side count exchange
  per step and is not captured.

Interaction: "dot" (DLRM pairwise dot products of the bottom output and every
table's pooled vector, plus the bottom output) when every table dim equals the
bottom MLP's output width, else "cat" (concatenation).
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch
from torch import nn

from .dist import Comm, NcclComm, ShardedEmbedding


def mlp(widths: Sequence[int], final_act: bool = True) -> nn.Sequential:
    layers = []
    for i in range(len(widths) - 1):
        layers.append(nn.Linear(widths[i], widths[i + 1]))
        if i < len(widths) - 2 or final_act:
            layers.append(nn.ReLU())
    return nn.Sequential(*layers)


class Interaction(nn.Module):
    def __init__(self, num_tables: int, kind: str):
        super().__init__()
        self.T, self.kind = num_tables, kind
        if kind == "dot":
            F = num_tables + 1
            li, lj = torch.tril_indices(F, F, offset=-1)
            self.register_buffer("li", li, persistent=False)
            self.register_buffer("lj", lj, persistent=False)

    def out_dim(self, bottom_dim: int, total_emb_dim: int) -> int:
        if self.kind == "dot":
            F = self.T + 1
            return bottom_dim + F * (F - 1) // 2
        return bottom_dim + total_emb_dim

    def forward(self, x: torch.Tensor, pooled: torch.Tensor) -> torch.Tensor:
        if self.kind == "cat":
            return torch.cat([x, pooled], dim=1)
        B, d = x.shape
        z = torch.cat([x.unsqueeze(1), pooled.view(B, self.T, d)], dim=1)  # (B, T+1, d)
        zz = torch.bmm(z, z.transpose(1, 2))
        return torch.cat([x, zz[:, self.li, self.lj]], dim=1)


class DLRM:
    """Sharded-embedding DLRM on one rank (one process per GPU).

    model: ModelSpec (tables; the MLP widths come from bottom/top here);
    plan: ShardingPlan; comm: NcclComm (or a single-rank LocalComm);
    dense_in: dense feature width; bottom: hidden widths of the bottom MLP
    (its output width is appended automatically when the interaction is
    "dot"); top: hidden widths of the top MLP (a final 1-wide logit layer is
    appended)."""

    def __init__(self, model, plan, comm: Comm, local_batch: int, dense_in: int = 13,
                 bottom: Sequence[int] = (512, 256), top: Sequence[int] = (512, 256), device=None,
                 emb_dtype=torch.float32, emb_lr: float = 0.05, emb_eps: float = 1e-8, dense_lr: float = 0.05,
                 fwd_comm: Optional[torch.dtype] = None, bwd_comm: Optional[torch.dtype] = None,
                 transport: str = "nccl", graphs: bool = False, index_dtype=torch.int32, seed: int = 0,
                 init=None):
        self.device = torch.device(device or "cuda")
        self.comm = comm
        self.B = local_batch
        dims = [t.dim for t in model.tables]
        self.T = len(dims)
        d0 = dims[0] if dims else 0
        kind = "dot" if dims and all(d == d0 for d in dims) else "cat"
        bw = list(bottom) + ([d0] if kind == "dot" else [])
        torch.manual_seed(seed)  # identical dense replicas on every rank
        self.bottom = mlp([dense_in] + bw).to(self.device)
        self.inter = Interaction(self.T, kind).to(self.device)
        ti = self.inter.out_dim(bw[-1], sum(dims))
        self.top = mlp([ti] + list(top) + [1], final_act=False).to(self.device)
        self.params = list(self.bottom.parameters()) + list(self.top.parameters())
        self.emb = ShardedEmbedding(model, plan, comm, local_batch, device=self.device, dtype=emb_dtype,
                                    optim="rowwise_adagrad", fwd_comm=fwd_comm, bwd_comm=bwd_comm,
                                    index_dtype=index_dtype, transport=transport, init=init)
        self.emb_lr, self.emb_eps, self.dense_lr = emb_lr, emb_eps, dense_lr
        self.side = torch.cuda.Stream(device=self.device)
        self.flat_grad = torch.zeros(sum(p.numel() for p in self.params), device=self.device)
        self.loss = torch.zeros((), device=self.device)
        self.graphs = graphs
        self._graphed = None
        self.total_dim = sum(dims)
        self.bottom_out = bw[-1]
        self.world = comm.world
        if not isinstance(comm, NcclComm) and len(comm.ranks) != 1:
            raise ValueError("DLRM drives one rank per process (NcclComm, or a 1-rank LocalComm)")

    # -- dense pieces ------------------------------------------------------
    def _make_graphed(self, dense: torch.Tensor) -> None:
        """CUDA-graph the bottom MLP and the top (interaction + MLP)."""
        pooled_like = torch.zeros((self.B, self.total_dim), device=self.device, requires_grad=True)
        x_like = torch.zeros((self.B, self.bottom_out), device=self.device, requires_grad=True)
        top_mod = _Top(self.inter, self.top)
        self._g_bottom = torch.cuda.make_graphed_callables(self.bottom, (dense.detach().clone(),))
        self._g_top = torch.cuda.make_graphed_callables(top_mod, (x_like, pooled_like))
        self._graphed = True

    def step(self, lengths, ids, dense: torch.Tensor, labels: torch.Tensor, lengths_dev=None) -> torch.Tensor:
        """One training step on this rank's local batch: lengths (T, B)
        host int64, ids (device, table-major), dense (B, dense_in), labels
        (B,) in {0, 1}.  Returns the (device) mean BCE loss of the batch."""
        if self.graphs and self._graphed is None:
            self._make_graphed(dense)
        bottom = self._g_bottom if self.graphs else self.bottom
        main = torch.cuda.current_stream(self.device)
        self.side.wait_stream(main)
        with torch.cuda.stream(self.side):  # overlaps the TBE forward + pooled exchange
            x = bottom(dense)
        state = {}

        def upstream(pooled: torch.Tensor) -> torch.Tensor:
            main.wait_stream(self.side)
            p = pooled.detach().requires_grad_(True)
            if self.graphs:
                logit = self._g_top(x, p)
            else:
                logit = self.top(self.inter(x, p))
            loss = nn.functional.binary_cross_entropy_with_logits(logit.view(-1), labels)
            for q in self.params:
                q.grad = None
            loss.backward()  # bottom-MLP backward is queued on the side stream
            state["loss"] = loss.detach()
            return p.grad

        self.emb.step([(lengths, ids, lengths_dev)], lr=self.emb_lr, eps=self.emb_eps, upstream_fn=upstream)
        main.wait_stream(self.side)
        self._dense_update()
        return state["loss"]

    def _dense_update(self) -> None:
        grads = [p.grad for p in self.params]
        if self.world > 1:
            off = 0
            for g in grads:
                n = g.numel()
                self.flat_grad[off:off + n].copy_(g.view(-1))
                off += n
            self.emb.comm.all_reduce_sum([self.flat_grad])
            self.flat_grad.div_(self.world)
            off = 0
            for g in grads:
                n = g.numel()
                g.view(-1).copy_(self.flat_grad[off:off + n])
                off += n
        with torch.no_grad():
            torch._foreach_add_(self.params, grads, alpha=-self.dense_lr)


class _Top(nn.Module):
    def __init__(self, inter: Interaction, top: nn.Module):
        super().__init__()
        self.inter, self.top = inter, top

    def forward(self, x, pooled):
        return self.top(self.inter(x, pooled))
