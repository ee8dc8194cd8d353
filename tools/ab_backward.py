"""A/B of the fused backward fast-path variants on one GPU (diagnostic).

Runs the same UPDATE backward (row-wise AdaGrad unless --optim) on two copies
of a table group, once through NEO_BWD_VARIANT=stream (single-warp walk) and
once through the warp-specialised pipeline, checks the updated weights and
moments agree (bitwise on uniform ids: same accumulation order), then times
each variant's backward with CUDA events.

  python tools/ab_backward.py --tables 64 --rows 1000000 --dim 128 --batch 65536 --pooling 32
"""
from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2104_05158_b200 import tbe  # noqa: E402
import paper_2104_05158_b200 as neo  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tables", type=int, default=64)
    ap.add_argument("--rows", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--pooling", type=int, default=32)
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--optim", default="rowwise_adagrad")
    ap.add_argument("--zipf", type=float, default=0.0, help="power-law ids (alpha) instead of uniform")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--randn-upstream", action="store_true")
    ap.add_argument("--only", default="", help="run one variant only (stream|pipe)")
    a = ap.parse_args()
    neo.load()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    T, H, D, B, L = a.tables, a.rows, a.dim, a.batch, a.pooling
    N = B * L
    dt = getattr(torch, a.dtype)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    grps = []
    for _ in range(2):
        grp = tbe.TableGroup([H] * T, [D] * T, dtype=dt, optim=a.optim, device=dev)
        grps.append(grp)
    grps[0]._storage.normal_(generator=g)
    grps[1]._storage.copy_(grps[0]._storage)
    offsets = torch.arange(0, T * B + 1, dtype=torch.int64, device=dev) * L
    if a.zipf > 0:
        rng = np.random.default_rng(0)
        ids = np.minimum(rng.zipf(a.zipf, size=T * N) - 1, H - 1).astype(np.int32)
        ix = torch.from_numpy(ids).to(dev)
    else:
        ix = torch.randint(0, H, (T * N,), dtype=torch.int32, device=dev, generator=g)
    if a.randn_upstream:
        up = torch.randn((B, T * D), dtype=torch.float32, device=dev, generator=g)
    else:
        up = torch.ones((B, T * D), dtype=torch.float32, device=dev)
    counts = [N] * T
    res = {}
    for name, grp in (("stream", grps[0]), ("pipe", grps[1])):
        if a.only and name != a.only:
            continue
        os.environ["NEO_BWD_VARIANT"] = name
        grp.backward(ix, offsets, B, up, mode="update", optim=a.optim, lr=0.05, eps=1e-8, table_counts=counts)
        torch.cuda.synchronize()
        print(name, "ok", flush=True)
    if a.only:
        return
    w0, w1 = grps[0]._storage, grps[1]._storage
    diff = (w0.float() - w1.float()).abs()
    res["weights_bitwise_equal"] = bool(torch.equal(w0, w1))
    res["weights_max_abs_diff"] = float(diff.max())
    if grps[0].moments[0] is not None:
        m0 = torch.cat([m.flatten() for m in grps[0].moments])
        m1 = torch.cat([m.flatten() for m in grps[1].moments])
        res["moments_bitwise_equal"] = bool(torch.equal(m0, m1))
        res["moments_max_rel_diff"] = float(((m0 - m1).abs() / m0.abs().clamp_min(1e-30)).max())
    del diff
    for name, grp in (("stream", grps[0]), ("pipe", grps[1])):
        os.environ["NEO_BWD_VARIANT"] = name
        timers = {}
        for _ in range(2):
            grp.backward(ix, offsets, B, up, mode="update", optim=a.optim, lr=0.05, eps=1e-8, table_counts=counts)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.iters):
            grp.backward(ix, offsets, B, up, mode="update", optim=a.optim, lr=0.05, eps=1e-8, table_counts=counts,
                         timers=timers)
        e1.record()
        torch.cuda.synchronize()
        aps = [x.elapsed_time(y) for x, y, _, _ in timers.get("apply", [])]
        res[name] = {"bwd_ms": e0.elapsed_time(e1) / a.iters, "apply_ms_mean": float(np.mean(aps)) if aps else None,
                     "applies_per_bwd": len(aps) // a.iters}
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
