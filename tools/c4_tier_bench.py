"""Config 4 in fp32 at 2 GPUs through the HBM + host-memory tier (SURVEY.md
8d: 205.6 GB of tables per GPU, more than HBM; the reference classifies such a
worker "hbm+dram", planner.py:512-522, and prices it with cache.py:129-136).

One rank's step of the row-wise plan (4 tables x 100,000,000 rows x dim 256
fp32, rank 0 owns rows [0, 50M) of every table): the global batch of 65,536
samples at pooling 32, the ids that fall into rank 0's rows routed to it
(about 16 per bag and table), fused forward + backward + row-wise AdaGrad.
Rows [0, hbm_rows) of each shard stay in HBM, the rest in pinned host memory
behind a set-associative slot cache (tier.HybridTableGroup).  Rank 1's step is
the mirror image on its own GPU, so the 2-GPU throughput is 65,536 samples per
slowest-rank step; the pooled row-wise exchange is not part of this step (it is
in bench.py's c4 line).

  python tools/c4_tier_bench.py [--hbm-rows 36000000] [--sets 16384] [--steps 5]
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

T, H_GLOBAL, D, B, L, W = 4, 100_000_000, 256, 65536, 32, 2
H = H_GLOBAL // W  # rank 0's rows of each table


def rank0_batch(gen, dev):
    """ids (table-major, int32, rebased to rank 0's shard) + lengths (T, B) of
    the global batch's lookups that rank 0 owns."""
    full = torch.randint(0, H_GLOBAL, (T, B, L), generator=gen, device=dev, dtype=torch.int64)
    mask = full < H
    lengths = mask.sum(dim=2)
    ids = full[mask].to(torch.int32)
    return ids, lengths


def build(hbm_rows: int, sets: int, dev):
    from paper_2104_05158_b200 import tier

    hy = tier.HybridTableGroup([H] * T, [D] * T, [hbm_rows] * T, num_sets=sets, ways=32, optim="rowwise_adagrad",
                               device=dev)
    g = torch.Generator(device=dev).manual_seed(5)
    for w in hy.hbm.weights:
        w.normal_(generator=g)
    chunk = torch.empty((1 << 20, D), dtype=torch.float32, device=dev)
    for hw in hy.host.host_w:  # host rows from device-generated chunks (a CPU RNG pass over 49 GB is slow)
        for r0 in range(0, hw.shape[0], chunk.shape[0]):
            n = min(chunk.shape[0], hw.shape[0] - r0)
            chunk[:n].normal_(generator=g)
            hw[r0:r0 + n].copy_(chunk[:n])
    return hy


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--hbm-rows", type=int, default=36_000_000)
    ap.add_argument("--sets", type=int, default=16384)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    import paper_2104_05158_b200 as neo

    neo.load()
    dev = torch.device("cuda", 0)
    t0 = time.time()
    hy = build(a.hbm_rows, a.sets, dev)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    gen = torch.Generator(device=dev).manual_seed(7)
    batches = []
    for _ in range(a.warmup + a.steps):
        ids, lengths = rank0_batch(gen, dev)
        off = torch.zeros(T * B + 1, dtype=torch.int64, device=dev)
        torch.cumsum(lengths.reshape(-1), 0, out=off[1:])
        batches.append((ids, off))
    up = torch.ones((B, T * D), dtype=torch.float32, device=dev)
    out = torch.empty((B, T * D), dtype=torch.float32, device=dev)
    for i in range(a.warmup):
        hy.forward(batches[i][0], batches[i][1], B, out=out)
        hy.backward(B, up, lr=0.05, eps=1e-8)
    torch.cuda.synchronize()
    st0 = dict(hy.host.stats)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    ev[0].record()
    for i in range(a.steps):
        ids, off = batches[a.warmup + i]
        hy.forward(ids, off, B, out=out)
        hy.backward(B, up, lr=0.05, eps=1e-8)
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[-1]) / a.steps
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.steps)]
    d = {k: (hy.host.stats[k] - st0[k]) / a.steps for k in st0}
    ids_step = float(np.mean([int(b[0].numel()) for b in batches[a.warmup:]]))
    host_frac = 1.0 - a.hbm_rows / H
    row_b = D * 4 + 4
    res = {
        "metric": "embedding-training samples/sec", "unit": "samples/s", "n_gpus": W,
        "value": B / (ms * 1e-3), "ms_per_step": ms, "steps": a.steps, "warmup": a.warmup,
        "step_ms": [round(x, 3) for x in per], "dtype": "f32", "data": "synthetic",
        "config": {"workload": "c4: 4 tables x 100,000,000 rows x dim 256 fp32, row-wise over 2 GPUs, global batch "
                               "65,536, pooling 32 (rank 0's step; rank 1 mirrors it on its GPU)",
                   "tier": f"rows [0, {a.hbm_rows:,}) of each 50M-row shard in HBM, the other "
                           f"{H - a.hbm_rows:,} in pinned host memory behind {a.sets:,} sets x 32 ways "
                           f"(+{hy.host.spill} spill slots) per table",
                   "hbm_gb": round(sum(w.numel() * 4 for w in hy.hbm.weights) / 1e9, 1),
                   "host_gb": round(sum(w.numel() * 4 for w in hy.host.host_w) / 1e9, 1),
                   "l2": "inputs larger than L2"},
        "ids_per_step": ids_step, "host_part_ids_per_step": d["accesses"],
        "host_part_hit_rate": 1.0 - d["misses"] / max(d["accesses"], 1),
        "row_fetches_per_step": d["misses"], "write_backs_per_step": d["writebacks"], "spills_per_step": d["spills"],
        "host_link_gb_per_step": (d["misses"] + d["writebacks"] + d["spills"]) * row_b / 1e9,
        "host_fraction_of_rows": host_frac, "setup_s": round(setup_s, 1),
    }
    print(json.dumps(res))


if __name__ == "__main__":
    main()
