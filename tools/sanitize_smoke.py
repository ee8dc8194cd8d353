"""Small end-to-end exercise of the round-1b kernels for compute-sanitizer
(memcheck): pipelined backward (uniform + skewed, update + dense), row-cache
replay, HBM tier.  Sizes are tiny so the instrumented run stays short."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2104_05158_b200 as neo  # noqa: E402
from paper_2104_05158_b200 import cache, tbe, tier  # noqa: E402


def main():
    neo.load()
    rng = np.random.default_rng(0)
    rows, dims, B = [3000, 1000], [128, 64], 256
    T = len(rows)
    for zipf in (0.0, 1.2):
        lengths = rng.integers(0, 20, size=(T, B))
        parts = [np.minimum(rng.zipf(zipf, int(lengths[t].sum())) - 1, rows[t] - 1) if zipf
                 else rng.integers(0, rows[t], int(lengths[t].sum())) for t in range(T)]
        ix = torch.from_numpy(np.concatenate(parts).astype(np.int32)).cuda()
        off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
        up = torch.randn((B, sum(dims)), device="cuda")
        counts = [int(c) for c in lengths.sum(axis=1)]
        for optim in ("rowwise_adagrad", "sgd", "adagrad"):
            g = tbe.TableGroup(rows, dims, optim=optim)
            g.forward(ix, off, B)
            g.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8, table_counts=counts)
        dense = [torch.zeros((r, d), device="cuda") for r, d in zip(rows, dims)]
        g.backward(ix, off, B, up, mode="dense", dense_grads=dense, table_counts=counts)
    cache.access_trace(cache.CacheConfig(num_sets=16, ways=8), rng.integers(0, 500, 5000))
    cache.access_trace(cache.CacheConfig(num_sets=4, ways=32, policy=cache.ReplacementPolicy.LFU),
                       np.minimum(rng.zipf(1.1, 5000) - 1, 10**6))
    tg = tier.TieredTableGroup([5000, 3000], [128, 64], num_sets=[64, 64], ways=16)
    off = torch.arange(0, 2 * 64 + 1, dtype=torch.int64, device="cuda") * 4
    for _ in range(3):
        ix = torch.from_numpy(np.concatenate([rng.integers(0, 5000, 256), rng.integers(0, 3000, 256)])
                              .astype(np.int32)).cuda()
        tg.forward(ix, off, 64, [256, 256])
        tg.backward(off, 64, torch.randn((64, 192), device="cuda"), [256, 256], lr=0.05, eps=1e-8)
    tg.flush()
    torch.cuda.synchronize()
    print("sanitize smoke done")


if __name__ == "__main__":
    main()
