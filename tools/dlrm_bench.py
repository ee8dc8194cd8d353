"""The whole DLRM training step around the embedding engine on one B200
(does the kernel work show up in samples/s once the dense
model is there?).  Config-2 tables (64 x 1,000,000 x 128 fp32, batch 65,536,
pooling 32, row-wise AdaGrad) under dlrm.DLRM: bottom MLP 13-512-256-128 on a
side stream overlapping the TBE forward, dot interaction (65 vectors -> 2,080
pairs + 128), top MLP 2208-1024-1024-512-256-1, BCE loss, dense SGD; dense
matmuls in fp32 with TF32 tensor cores.  Prints one JSON line with the step
time, the embedding-only step time of the same batch and the MLP share.

  python tools/dlrm_bench.py [--steps 10] [--warmup 3] [--graphs]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--graphs", action="store_true", help="CUDA-graph the dense MLPs")
    a = ap.parse_args()
    import paper_2104_05158_b200 as pkg
    from paper_2104_05158_b200 import dist, dlrm
    from paper_2104_05158_b200 import plan as P

    pkg.load()
    torch.backends.cuda.matmul.allow_tf32 = True
    dev = torch.device("cuda", 0)
    T, H, D, B, L = 64, 1_000_000, 128, 65536, 32
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=H, dim=D, avg_pooling=float(L)) for i in range(T)]
    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    plan = P.ShardingPlan(1, 1, tuple(P.TableAssignment(t.id, P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(0),))
                                      for t in specs))
    m = dlrm.DLRM(model, plan, dist.LocalComm(1), B, dense_in=13, bottom=(512, 256), top=(1024, 1024, 512, 256),
                  device=dev, graphs=a.graphs, index_dtype=torch.int32, dense_lr=1e-3)
    for st in m.emb.states:
        for grp in list(st.groups) + [st.dp_group]:
            if grp is not None:
                for w in grp.weights:
                    w.uniform_(-1.0 / H ** 0.5, 1.0 / H ** 0.5)  # DLRM-style init (keeps the logits finite)
    lengths = np.full((T, B), L, dtype=np.int64)
    L_dev = torch.from_numpy(lengths.reshape(-1)).to(dev)
    g = torch.Generator(device=dev).manual_seed(3)
    ids = [torch.randint(0, H, (T * B * L,), generator=g, device=dev, dtype=torch.int32) for _ in range(2)]
    dense = torch.randn((B, 13), generator=g, device=dev)
    labels = (torch.rand(B, generator=g, device=dev) < 0.5).float()

    def timed(fn):
        for i in range(a.warmup):
            fn(i)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(a.steps):
            fn(i)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.steps

    losses = []

    def full_step(i):
        losses.append(m.step(lengths, ids[i % 2], dense, labels, lengths_dev=L_dev))

    ms = timed(full_step)
    emb_ms = timed(lambda i: m.emb.step([(lengths, ids[i % 2], L_dev)], lr=0.05, eps=1e-8))
    loss = [float(x) for x in losses[-3:]]
    print(json.dumps({
        "metric": "DLRM training samples/sec (embedding engine + dense MLPs)", "unit": "samples/s", "n_gpus": 1,
        "value": B / (ms * 1e-3), "ms_per_step": ms, "embedding_only_ms_per_step": emb_ms,
        "dense_share_ms": ms - emb_ms, "steps": a.steps, "warmup": a.warmup, "graphs": a.graphs,
        "config": {"tables": "64 x 1,000,000 x 128 fp32 (config 2)", "batch": B, "pooling": L,
                   "bottom": "13-512-256-128", "interaction": "dot (65 vectors)",
                   "top": "2208-1024-1024-512-256-1", "dense_dtype": "fp32 (TF32 matmuls)",
                   "optimizers": "row-wise AdaGrad (tables), SGD (dense)"},
        "last_losses": loss, "data": "synthetic (random ids, dense features and labels)"}))


if __name__ == "__main__":
    main()
