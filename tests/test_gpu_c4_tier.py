"""Config 4 in fp32 at 2 GPUs (205.6 GB of tables per GPU: more than HBM)
through the HBM + host tier (tier.HybridTableGroup), rank 0's full-size step
(tools/c4_tier_bench.py): one step with a random upstream, then table 0's
touched rows (HBM part and host part) against the f64 C oracle
(embedding.py:175-192 aggregate, :212-232 row-wise AdaGrad), untouched rows
unchanged.  Needs ~150 GB of HBM and ~57 GB of host memory."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))
from oracle import tbe_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
LR, EPS = 0.05, 1e-8


def test_c4_fp32_w2_rank0_step_through_tier_matches_oracle():
    import paper_2104_05158_b200 as neo
    import c4_tier_bench as C

    assert torch.cuda.is_available()
    neo.load()
    torch.cuda.empty_cache()
    dev = torch.device("cuda", 0)
    hbm_rows = 36_000_000
    hy = C.build(hbm_rows, 16384, dev)
    gen = torch.Generator(device=dev).manual_seed(11)
    ids, lengths = C.rank0_batch(gen, dev)
    off = torch.zeros(C.T * C.B + 1, dtype=torch.int64, device=dev)
    torch.cumsum(lengths.reshape(-1), 0, out=off[1:])
    up = torch.randn((C.B, C.T * C.D), generator=gen, device=dev)
    n0 = int(lengths[0].sum())
    part = ids[:n0].cpu().numpy().astype(np.int64)
    uniq, remap = np.unique(part, return_inverse=True)
    in_hbm = uniq < hbm_rows
    u_h = torch.from_numpy(uniq[in_hbm]).to(dev)
    before = np.empty((len(uniq), C.D))
    before[in_hbm] = hy.hbm.weights[0][u_h].double().cpu().numpy()
    before[~in_hbm] = hy.host.host_w[0][torch.from_numpy(uniq[~in_hbm] - hbm_rows)].double().numpy()
    rng = np.random.default_rng(3)
    untouched = np.setdiff1d(rng.integers(0, C.H, 20000), uniq)
    ut_h, ut_c = untouched[untouched < hbm_rows], untouched[untouched >= hbm_rows] - hbm_rows
    keep_h = hy.hbm.weights[0][torch.from_numpy(ut_h).to(dev)].cpu()
    keep_c = hy.host.host_w[0][torch.from_numpy(ut_c)].clone()
    hy.forward(ids, off, C.B)
    hy.backward(C.B, up, lr=LR, eps=EPS)
    hy.flush()
    torch.cuda.synchronize()
    ids_a, gr = O.backward_aggregate_c(lengths[0].cpu().numpy().astype(np.int64), remap,
                                       np.ascontiguousarray(up[:, :C.D].double().cpu().numpy()))
    w = before.copy()
    m = np.zeros(len(uniq))
    O.apply_c("rowwise_adagrad", w, m, ids_a, gr, LR, EPS)
    got = np.empty_like(w)
    got_m = np.empty(len(uniq))
    got[in_hbm] = hy.hbm.weights[0][u_h].double().cpu().numpy()
    got_m[in_hbm] = hy.hbm.moments[0][u_h].double().cpu().numpy()
    hc = torch.from_numpy(uniq[~in_hbm] - hbm_rows)
    got[~in_hbm] = hy.host.host_w[0][hc].double().numpy()
    got_m[~in_hbm] = hy.host.host_m[0][hc].double().numpy()
    assert (np.abs(got - w) <= 1e-5 * (np.abs(w) + np.abs(w - before)) + 1e-7).all(), "touched rows"
    assert np.allclose(got_m, m, rtol=1e-5, atol=1e-9), "row-wise AdaGrad state"
    assert (~in_hbm).sum() > 100_000 and in_hbm.sum() > 100_000  # both parts exercised
    assert torch.equal(hy.hbm.weights[0][torch.from_numpy(ut_h).to(dev)].cpu(), keep_h)
    assert torch.equal(hy.host.host_w[0][torch.from_numpy(ut_c)], keep_c)
