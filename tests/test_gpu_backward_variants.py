"""The warp-specialised backward (tbe_pipe.cuh, default) against the
single-warp streamed walk (NEO_BWD_VARIANT=stream) and the CPU oracle.

Both kernels accumulate each row's upstream rows in sorted (= buffer) order
and fold hot-chunk partials identically, so their updated weights and
moments must be BITWISE equal; the oracle check bounds both against the
reference arithmetic (embedding.py:175-254) at the f32 tolerance."""
import os

import numpy as np
import pytest
import torch

from oracle import tbe_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tbe():
    import paper_2104_05158_b200 as p
    from paper_2104_05158_b200 import tbe as t

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    p.load()
    return t


def _run(tbe, variant, rows, dims, dtype, optim, ix, off, B, up, counts):
    grp = tbe.TableGroup(rows, dims, dtype=dtype, optim=optim)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    for w in grp.weights:
        w.copy_(torch.randn(w.shape, generator=g, device="cuda").to(dtype))
    if grp.moments[0] is not None:
        for m in grp.moments:
            m.copy_(torch.rand(m.shape, generator=g, device="cuda"))
    init_w = [w.double().cpu().numpy() for w in grp.weights]
    init_m = [None if m is None else m.double().cpu().numpy() for m in grp.moments]
    old = os.environ.get("NEO_BWD_VARIANT")
    os.environ["NEO_BWD_VARIANT"] = variant
    try:
        grp.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8, table_counts=counts)
        torch.cuda.synchronize()
    finally:
        if old is None:
            os.environ.pop("NEO_BWD_VARIANT", None)
        else:
            os.environ["NEO_BWD_VARIANT"] = old
    w = [x.clone() for x in grp.weights]
    m = [None if x is None else x.clone() for x in grp.moments]
    return w, m, init_w, init_m


CASES = [
    # rows, dims, weight dtype, grad dtype, optimizer, zipf alpha (0 = uniform)
    ([20000, 5000, 30000], [128, 128, 128], torch.float32, torch.float32, "rowwise_adagrad", 0.0),
    ([20000, 5000, 30000], [128, 128, 128], torch.float32, torch.float32, "sgd", 1.1),
    ([3000, 7000], [64, 32], torch.float32, torch.float32, "adagrad", 0.0),
    ([4000, 4000, 900], [256, 128, 256], torch.float32, torch.float32, "rowwise_adagrad", 1.2),
    ([8000, 2000], [256, 64], torch.float16, torch.float32, "rowwise_adagrad", 0.0),
    ([8000, 2000], [128, 96], torch.float32, torch.bfloat16, "rowwise_adagrad", 1.05),
    ([500, 800], [128, 128], torch.float32, torch.float16, "adagrad", 1.3),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_pipe_matches_stream_bitwise_and_oracle(tbe, case):
    rows, dims, wdt, gdt, optim, alpha = CASES[case]
    T, B = len(rows), 2048
    rng = np.random.default_rng(100 + case)
    lengths = rng.integers(0, 40, size=(T, B))
    parts = []
    for t in range(T):
        n = int(lengths[t].sum())
        if alpha > 0:
            parts.append(np.minimum(rng.zipf(alpha, size=n) - 1, rows[t] - 1))
        else:
            parts.append(rng.integers(0, rows[t], size=n))
    idx = np.concatenate(parts)
    counts = [int(c) for c in lengths.sum(axis=1)]
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    ix = torch.from_numpy(idx.astype(np.int32)).cuda()
    up = torch.from_numpy(rng.standard_normal((B, sum(dims)))).to(gdt).cuda()
    ws, ms, init_w, init_m = _run(tbe, "stream", rows, dims, wdt, optim, ix, off, B, up, counts)
    wp, mp, _, _ = _run(tbe, "pipe", rows, dims, wdt, optim, ix, off, B, up, counts)
    for t in range(T):
        assert torch.equal(ws[t], wp[t]), f"weights differ (table {t})"
        if ms[t] is not None:
            assert torch.equal(ms[t], mp[t]), f"moments differ (table {t})"
    # oracle: f64 restatement of aggregate + optimizer on the same (rounded) inputs
    tab_off = O.offsets_of(lengths.sum(axis=1))
    upd = up.double().cpu().numpy()
    col = 0
    for t, D in enumerate(dims):
        part = idx[tab_off[t]:tab_off[t + 1]]
        ids, gr = O.backward_aggregate_c(lengths[t], part, np.ascontiguousarray(upd[:, col:col + D]))
        w = init_w[t].copy()
        m = np.zeros(rows[t]) if init_m[t] is None else init_m[t].copy()
        O.apply_c(optim, w, m, ids, gr, 0.05, 1e-8)
        got = wp[t].double().cpu().numpy()
        ulp = 2.0 ** -10 if wdt == torch.float16 else 0.0
        bound = 1e-4 * (np.abs(w) + np.abs(w - init_w[t])) + ulp * np.abs(w) + 1e-6
        assert (np.abs(got - w) <= bound).all(), f"table {t}: max err {np.abs(got - w).max()}"
        col += D


def test_prepare_backward_on_side_stream_matches(tbe):
    """prepare_backward (key build + sort issued early on a side stream, here
    under a residency-capped forward) + backward == backward alone, bitwise."""
    rows, dims, B, L = [300000, 200000, 250000], [128, 128, 128], 4096, 16
    T = len(rows)
    rng = np.random.default_rng(5)
    idx = np.concatenate([rng.integers(0, r, size=B * L) for r in rows]).astype(np.int32)
    ix = torch.from_numpy(idx).cuda()
    off = torch.arange(0, T * B + 1, dtype=torch.int64, device="cuda") * L
    up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
    counts = [B * L] * T
    outs = []
    for prepared in (False, True):
        grp = tbe.TableGroup(rows, dims, dtype=torch.float32, optim="rowwise_adagrad")
        g = torch.Generator(device="cuda")
        g.manual_seed(3)
        grp._storage.copy_(torch.randn(grp._storage.shape, generator=g, device="cuda"))
        if prepared:
            tbe.set_forward_residency(3)
            try:
                assert grp.prepare_backward(ix, off, B, up, counts, optim="rowwise_adagrad")
                pooled = grp.forward(ix, off, B)
            finally:
                tbe.set_forward_residency(0)
        else:
            pooled = grp.forward(ix, off, B)
        grp.backward(ix, off, B, up, mode="update", optim="rowwise_adagrad", lr=0.05, eps=1e-8, table_counts=counts)
        torch.cuda.synchronize()
        outs.append((pooled.clone(), grp._storage.clone(), torch.cat([m.flatten() for m in grp.moments])))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("zipf", [0.0, 1.1])
def test_dense_mode_pipe_matches_oracle(tbe, zipf):
    """mode="dense" (the data-parallel tables' gradient) on the pipelined walk
    and on the warp-per-segment kernel (NEO_BWD_VARIANT=stream routes dense
    there) against the f64 oracle aggregate: |got - ref| <= 1e-5 * sum|terms|."""
    rows, dims, B = [30000, 8000, 12000], [128, 64, 256], 2048
    T = len(rows)
    rng = np.random.default_rng(21)
    lengths = rng.integers(0, 40, size=(T, B))
    parts = []
    for t in range(T):
        n = int(lengths[t].sum())
        parts.append(np.minimum(rng.zipf(zipf, n) - 1, rows[t] - 1) if zipf else rng.integers(0, rows[t], n))
    idx = np.concatenate(parts)
    ix = torch.from_numpy(idx.astype(np.int32)).cuda()
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    up_np = rng.standard_normal((B, sum(dims))).astype(np.float32)
    up = torch.from_numpy(up_np).cuda()
    counts = [int(c) for c in lengths.sum(axis=1)]
    grp = tbe.TableGroup(rows, dims, dtype=torch.float32, optim="sgd")
    tab_off = O.offsets_of(lengths.sum(axis=1))
    for variant in ("stream", "pipe"):
        dense = [torch.zeros((r, d), dtype=torch.float32, device="cuda") for r, d in zip(rows, dims)]
        os.environ["NEO_BWD_VARIANT"] = variant
        try:
            grp.backward(ix, off, B, up, mode="dense", dense_grads=dense, table_counts=counts)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("NEO_BWD_VARIANT", None)
        col = 0
        for t, D in enumerate(dims):
            part = idx[tab_off[t]:tab_off[t + 1]]
            u = np.ascontiguousarray(up_np[:, col:col + D].astype(np.float64))
            ids, gr = O.backward_aggregate_c(lengths[t], part, u)
            _, ga = O.backward_aggregate_c(lengths[t], part, np.abs(u))
            got = dense[t].double().cpu().numpy()[ids]
            assert (np.abs(got - gr) <= 1e-5 * ga + 1e-30).all(), f"{variant}: table {t}"
            col += D


def test_tma_gather4_producer_bitwise(tbe):
    """NEO_PIPE_TMA=1: the producer stages full 4-entry stages of upstream rows
    with one TMA tile::gather4 each; results stay bitwise equal to the walk."""
    old = os.environ.get("NEO_PIPE_TMA")
    os.environ["NEO_PIPE_TMA"] = "1"
    try:
        for case in (0, 3):
            test_pipe_matches_stream_bitwise_and_oracle(tbe, case)
    finally:
        if old is None:
            os.environ.pop("NEO_PIPE_TMA", None)
        else:
            os.environ["NEO_PIPE_TMA"] = old
