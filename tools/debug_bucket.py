"""Diagnostics: one bucketed backward step with progress prints (run with
NEO_BKT_DEBUG=1 to trace every launch)."""
import sys

import numpy as np
import torch

import paper_2104_05158_b200 as neo
from paper_2104_05158_b200 import tbe

neo.load()
case = sys.argv[1] if len(sys.argv) > 1 else "adagrad"
rows, dims, B = [3000, 7000], [64, 32], 2048
rng = np.random.default_rng(302)
lengths = rng.integers(0, 40, size=(2, B))
idx = np.concatenate([rng.integers(0, r, size=int(lengths[t].sum())) for t, r in enumerate(rows)])
off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
ix = torch.from_numpy(idx.astype(np.int32)).cuda()
up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
for optim in (case, "sgd", "rowwise_adagrad", "adagrad"):
    grp = tbe.TableGroup(rows, dims, dtype=torch.float32, optim=optim)
    print("group", optim, flush=True)
    grp.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8)
    print("issued", flush=True)
    torch.cuda.synchronize()
    print("done", optim, flush=True)
