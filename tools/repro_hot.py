"""Reproduce the skewed-row backward in isolation (development tool)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_05158_b200 import tbe  # noqa: E402

rng = np.random.default_rng(11)
dims = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [64, 128, 32, 8, 100]
rows = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [3000, 5000, 40, 2000, 700]
B = 1024
lengths = rng.integers(0, 25, size=(len(dims), B))
idx = np.concatenate([rng.integers(0, rows[t], size=int(lengths[t].sum())) for t in range(len(dims))])
grp = tbe.TableGroup(rows, dims, dtype=torch.float32, optim="rowwise_adagrad")
grp._storage.normal_()
off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
g = torch.randn((B, grp.total_dim), device="cuda")
t0 = time.time()
grp.backward(torch.from_numpy(idx).int().cuda(), off, B, g, mode="update", optim="rowwise_adagrad", lr=0.05, eps=1e-8)
torch.cuda.synchronize()
print("ok", dims, rows, f"{time.time() - t0:.3f}s", flush=True)
