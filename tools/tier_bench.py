"""Measure the HBM tier over host-resident tables (tier.TieredTableGroup) on
one GPU and compare with the reference's analytical model of that tier
(cache.py:129-136 effective_row_bandwidth: 1 / (h / hbm + (1-h) / backing)).

  python tools/tier_bench.py --tables 4 --rows 10000000 --dim 128 --batch 16384 --pooling 32 --sets 32768
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

import paper_2104_05158_b200 as neo  # noqa: E402
from paper_2104_05158_b200 import cache, tier  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", type=int, default=4)
    ap.add_argument("--rows", type=int, default=10_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--pooling", type=int, default=32)
    ap.add_argument("--sets", type=int, default=32768)
    ap.add_argument("--zipf", type=float, default=1.05)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    a = ap.parse_args()
    neo.load()
    dev = torch.device("cuda", 0)
    T, H, D, B, L = a.tables, a.rows, a.dim, a.batch, a.pooling
    t0 = time.time()
    tg = tier.TieredTableGroup([H] * T, [D] * T, num_sets=a.sets, ways=32, optim="rowwise_adagrad", device=dev)
    for w in tg.host_w:
        w.normal_()
    setup_s = time.time() - t0
    counts = [B * L] * T
    off = torch.arange(0, T * B + 1, dtype=torch.int64, device=dev) * L
    up = torch.ones((B, T * D), dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)

    def ids():
        u = torch.rand(T * B * L, generator=g, device=dev, dtype=torch.float64)
        if a.zipf > 0:
            al = a.zipf
            r = (1.0 - u * (1.0 - H ** (1.0 - al))) ** (1.0 / (1.0 - al)) - 1.0
        else:
            r = u * H
        return torch.clamp(r, 0, H - 1).to(torch.int32)

    batches = [ids() for _ in range(a.warmup + a.steps)]
    for i in range(a.warmup):
        tg.forward(batches[i], off, B, counts)
        tg.backward(off, B, up, counts, lr=0.05, eps=1e-8)
    torch.cuda.synchronize()
    m0, w0, acc0 = tg.stats["misses"], tg.stats["writebacks"], tg.stats["accesses"]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(a.warmup, a.warmup + a.steps):
        tg.forward(batches[i], off, B, counts)
        tg.backward(off, B, up, counts, lr=0.05, eps=1e-8)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.steps
    misses = (tg.stats["misses"] - m0) / a.steps
    wbs = (tg.stats["writebacks"] - w0) / a.steps
    accesses = (tg.stats["accesses"] - acc0) / a.steps
    row_b = D * 4 + 4
    pcie_bytes = (misses + wbs) * row_b
    hit = 1.0 - misses / accesses
    res = {"workload": f"{T} tables x {H:,} rows x dim {D} fp32 in pinned host memory, HBM cache {a.sets:,} sets x 32 "
                       f"ways per table ({a.sets * 32 / H:.1%} of rows), batch {B:,}, pooling {L}, "
                       f"ids {'Zipf(%g)' % a.zipf if a.zipf > 0 else 'uniform'}, row-wise AdaGrad",
           "samples_per_s": B / (ms * 1e-3), "ms_per_step": ms, "lookup_hit_rate": hit,
           "misses_per_step": misses, "writebacks_per_step": wbs,
           "host_link_gbs": pcie_bytes / (ms * 1e-3) / 1e9, "host_bytes_per_step": pcie_bytes,
           "setup_s": setup_s}
    # the reference's model of this tier at the measured hit rate, with this box's measured HBM
    # copy bandwidth and the host link bandwidth measured by this run
    res["reference_model_row_gbs"] = cache.effective_row_bandwidth(hit, 6544.3, max(res["host_link_gbs"], 1e-9))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
