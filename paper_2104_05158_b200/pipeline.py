"""Host-facing training pipeline for one TBE table group.

``TrainPipeline.run`` takes host (pinned) batches in the reference's
lengths format — per-table lengths (T*B,) and the table-major id buffer —
and for each batch: copies it to HBM on a side stream (overlapping the
previous step's compute), builds offsets on device, runs the fused TBE
forward, the loss (sum of pooled outputs, the reference's train-step loss,
embedding.py:319-327), the fused backward + optimizer, and reads the loss
back to pinned host memory.  Two device slots double-buffer the inputs.
"""
from __future__ import annotations

from typing import Optional, Sequence

import torch

from . import tbe


class TrainPipeline:
    def __init__(self, group: tbe.TableGroup, batch: int, optim: str = "rowwise_adagrad",
                 lr: float = 0.05, eps: float = 1e-8, pooling: str = "sum",
                 upstream: Optional[torch.Tensor] = None):
        self.g = group
        self.B = batch
        self.optim, self.lr, self.eps, self.pooling = optim, lr, eps, pooling
        dev = group.device
        od = torch.float64 if group.dtype == torch.float64 else torch.float32
        self.out = torch.empty((batch, group.total_dim), dtype=od, device=dev)
        # d(sum of outputs)/d(outputs) = 1: the reference loss's upstream
        self.upstream = upstream if upstream is not None else torch.ones_like(self.out)
        self.copy_stream = torch.cuda.Stream(device=dev)
        self.slots = [dict(ids=None, lengths=None, copied=torch.cuda.Event(), free=torch.cuda.Event())
                      for _ in range(2)]
        for s in self.slots:
            s["free"].record()

    def _stage(self, slot, lengths: torch.Tensor, ids: torch.Tensor) -> None:
        dev = self.g.device
        if slot["ids"] is None or slot["ids"].numel() != ids.numel() or slot["ids"].dtype != ids.dtype:
            slot["ids"] = torch.empty(ids.shape, dtype=ids.dtype, device=dev)
        if slot["lengths"] is None or slot["lengths"].numel() != lengths.numel():
            slot["lengths"] = torch.empty(lengths.shape, dtype=torch.int64, device=dev)
        slot["counts"] = lengths.view(self.g.T, -1).sum(dim=1).tolist()  # host data: no device sync
        with torch.cuda.stream(self.copy_stream):
            self.copy_stream.wait_event(slot["free"])
            slot["ids"].copy_(ids, non_blocking=True)
            slot["lengths"].copy_(lengths, non_blocking=True)
            slot["copied"].record(self.copy_stream)

    def run(self, batches: Sequence) -> list:
        """batches: sequence of (lengths (T*B,) int64, ids) host tensors
        (pinned for asynchronous copies).  Returns the per-step losses."""
        if not batches:
            return []
        losses = torch.empty(len(batches), dtype=self.out.dtype, pin_memory=True)
        compute = torch.cuda.current_stream(self.g.device)
        self._stage(self.slots[0], *batches[0])
        for i in range(len(batches)):
            slot = self.slots[i % 2]
            if i + 1 < len(batches):  # prefetch the next batch behind this step
                self._stage(self.slots[(i + 1) % 2], *batches[i + 1])
            compute.wait_event(slot["copied"])
            offsets = tbe.lengths_to_offsets(slot["lengths"])
            out = self.g.forward(slot["ids"], offsets, self.B, pooling=self.pooling, out=self.out)
            loss = out.sum()
            losses[i:i + 1].copy_(loss.reshape(1), non_blocking=True)
            self.g.backward(slot["ids"], offsets, self.B, self.upstream, mode="update", optim=self.optim,
                            lr=self.lr, eps=self.eps, pooling=self.pooling, table_counts=slot["counts"])
            slot["free"].record(compute)
        torch.cuda.current_stream(self.g.device).synchronize()
        return losses.tolist()
