"""The bucketed backward (csrc/tbe_bucket.cu, the default UPDATE / DENSE fast
path: hand-written stable two-level counting sort + fused sub-warp-per-row
reduce and optimizer) against the CPU oracle, for determinism, and at the
edges the reference tests touch: empty bags, single-row tables, hot rows
split across the CTA, buckets larger than shared memory (global passes),
multi-pass row sorts, invalid ids (embedding.py:175-254)."""
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


def _ids(rng, rows, n, alpha):
    if alpha > 0:
        return np.minimum(rng.zipf(alpha, size=n) - 1, rows - 1)
    return rng.integers(0, rows, size=n)


def _group(tbe, rows, dims, wdt, optim, seed=7):
    grp = tbe.TableGroup(rows, dims, dtype=wdt, optim=optim)
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    for w in grp.weights:
        w.copy_(torch.randn(w.shape, generator=g, device="cuda").to(wdt))
    if grp.moments[0] is not None:
        for m in grp.moments:
            m.copy_(torch.rand(m.shape, generator=g, device="cuda"))
    return grp


def _check_oracle(grp, init_w, init_m, lengths, idx, upd, rows, dims, optim, wdt, tag=""):
    tab_off = O.offsets_of(lengths.sum(axis=1))
    col = 0
    for t, D in enumerate(dims):
        part = idx[tab_off[t]:tab_off[t + 1]]
        ids, gr = O.backward_aggregate_c(lengths[t], part, np.ascontiguousarray(upd[:, col:col + D]))
        w = init_w[t].copy()
        m = np.zeros(rows[t]) if init_m[t] is None else init_m[t].copy()
        O.apply_c(optim, w, m, ids, gr, 0.05, 1e-8)
        got = grp.weights[t].double().cpu().numpy()
        ulp = 2.0 ** -10 if wdt == torch.float16 else 0.0
        bound = 1e-4 * (np.abs(w) + np.abs(w - init_w[t])) + ulp * np.abs(w) + 1e-6
        err = np.abs(got - w)
        assert (err <= bound).all(), f"{tag} table {t}: max err {err.max()} at {np.unravel_index(err.argmax(), err.shape)}"
        if optim == "rowwise_adagrad":
            gm = grp.moments[t].double().cpu().numpy()
            assert np.allclose(gm, m, rtol=1e-4, atol=1e-6), f"{tag} moment table {t}"
        col += D


CASES = [
    # rows, dims, weight dtype, grad dtype, optimizer, zipf alpha (0 = uniform), B, max length
    ([20000, 5000, 30000], [128, 128, 128], torch.float32, torch.float32, "rowwise_adagrad", 0.0, 2048, 40),
    ([20000, 5000, 30000], [128, 128, 128], torch.float32, torch.float32, "sgd", 1.1, 2048, 40),
    ([3000, 7000], [64, 32], torch.float32, torch.float32, "adagrad", 0.0, 2048, 40),
    ([4000, 4000, 900], [256, 128, 256], torch.float32, torch.float32, "rowwise_adagrad", 1.2, 2048, 40),
    ([8000, 2000], [256, 64], torch.float16, torch.float32, "rowwise_adagrad", 0.0, 2048, 40),
    ([8000, 2000], [128, 96], torch.float32, torch.bfloat16, "rowwise_adagrad", 1.05, 2048, 40),
    ([500, 800], [128, 128], torch.float32, torch.float16, "adagrad", 1.3, 2048, 40),
    # multi-pass row sort (large sparse table: bucket bits > 9) and tiny tables
    ([5_000_000, 1, 17], [128, 16, 8], torch.float32, torch.float32, "rowwise_adagrad", 0.0, 3000, 12),
    # big buckets (> 4096 entries, global passes) + hot rows split across the CTA
    ([1_000_000, 50000], [128, 64], torch.float32, torch.float32, "rowwise_adagrad", 1.6, 4096, 64),
    ([2_000_000], [64], torch.float16, torch.bfloat16, "sgd", 2.5, 8192, 50),
    # B = 1 and empty bags
    ([1000, 300], [32, 48], torch.float32, torch.float32, "rowwise_adagrad", 0.0, 1, 30),
]


@pytest.mark.parametrize("case", range(len(CASES)))
def test_bucket_matches_oracle_and_is_deterministic(tbe, case):
    rows, dims, wdt, gdt, optim, alpha, B, lmax = CASES[case]
    T = len(rows)
    rng = np.random.default_rng(300 + case)
    lengths = rng.integers(0, lmax, size=(T, B))
    idx = np.concatenate([_ids(rng, rows[t], int(lengths[t].sum()), alpha) for t in range(T)])
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    ix = torch.from_numpy(idx.astype(np.int32)).cuda()
    up = torch.from_numpy(rng.standard_normal((B, sum(dims)))).to(gdt).cuda()
    results = []
    for rep in range(2):
        grp = _group(tbe, rows, dims, wdt, optim)
        assert grp._bucketed("update", B, up, up.stride(0), "sum")
        init_w = [w.double().cpu().numpy() for w in grp.weights]
        init_m = [None if m is None else m.double().cpu().numpy() for m in grp.moments]
        grp.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8)
        torch.cuda.synchronize()
        results.append(([w.clone() for w in grp.weights], [None if m is None else m.clone() for m in grp.moments]))
    for t in range(T):  # bitwise deterministic
        assert torch.equal(results[0][0][t], results[1][0][t]), f"weights nondeterministic (table {t})"
        if results[0][1][t] is not None:
            assert torch.equal(results[0][1][t], results[1][1][t])
    _check_oracle(grp, init_w, init_m, lengths, idx, up.double().cpu().numpy(), rows, dims, optim, wdt, f"case {case}")


def test_bucket_int64_ids_and_table_counts(tbe, monkeypatch):
    """int64 ids; the call with host table counts takes the same path (forced:
    with counts, tables whose buckets span > 2^9 rows route to the pipelined
    walk by default)."""
    monkeypatch.setenv("NEO_BWD_VARIANT", "bucket")
    rows, dims, B = [70000, 90000], [128, 64], 4096
    rng = np.random.default_rng(11)
    lengths = rng.integers(0, 30, size=(2, B))
    idx = np.concatenate([rng.integers(0, r, size=int(lengths[t].sum())) for t, r in enumerate(rows)])
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
    outs = []
    for dt, counts in ((torch.int64, None), (torch.int32, [int(c) for c in lengths.sum(axis=1)])):
        grp = _group(tbe, rows, dims, torch.float32, "rowwise_adagrad")
        init_w = [w.double().cpu().numpy() for w in grp.weights]
        init_m = [m.double().cpu().numpy() for m in grp.moments]
        grp.backward(torch.from_numpy(idx).to(dt).cuda(), off, B, up, mode="update", optim="rowwise_adagrad",
                     lr=0.05, eps=1e-8, table_counts=counts)
        torch.cuda.synchronize()
        outs.append(grp._storage.clone())
        _check_oracle(grp, init_w, init_m, lengths, idx, up.double().cpu().numpy(), rows, dims, "rowwise_adagrad",
                      torch.float32)
    assert torch.equal(outs[0], outs[1])


def test_bucket_invalid_ids_recorded_and_skipped(tbe):
    """An out-of-range id is recorded (first position in buffer order) and
    skipped; every valid row is still updated exactly once."""
    rows, dims, B, L = [1000, 2000], [64, 64], 512, 8
    rng = np.random.default_rng(3)
    idx = np.concatenate([rng.integers(0, r, size=B * L) for r in rows]).astype(np.int64)
    bad_pos = [B * L + 77, B * L + 900, 100]
    idx[B * L + 77] = 2000
    idx[B * L + 900] = -3
    idx[100] = 1000
    lengths = np.full((2, B), L)
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    up = torch.from_numpy(rng.standard_normal((B, 128)).astype(np.float32)).cuda()
    grp = _group(tbe, rows, dims, torch.float32, "sgd")
    init_w = [w.double().cpu().numpy() for w in grp.weights]
    err = tbe.ErrorRecord("cuda").reset()
    grp.backward(torch.from_numpy(idx).cuda(), off, B, up, mode="update", optim="sgd", lr=0.05, err=err)
    pos, value, table = err.read()
    assert (pos, value, table) == (min(bad_pos), 1000, 0)
    keep = np.ones(idx.shape, bool)
    keep[bad_pos] = False
    tab_off = O.offsets_of(lengths.sum(axis=1))
    upd = up.double().cpu().numpy()
    for t in range(2):
        sl = slice(tab_off[t], tab_off[t + 1])
        part, k = idx[sl], keep[sl]
        bags = np.repeat(np.arange(B), L)[k]
        w = init_w[t].copy()
        np.add.at(w, part[k], -0.05 * upd[bags, 64 * t:64 * t + 64])
        assert np.allclose(grp.weights[t].double().cpu().numpy(), w, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("zipf", [0.0, 1.1, 2.0])
def test_bucket_dense_mode_matches_oracle(tbe, zipf):
    """mode="dense" (data-parallel tables' gradient): |got - ref| <= 1e-5 * sum|terms|."""
    rows, dims, B = [30000, 8000, 12000], [128, 64, 256], 2048
    T = len(rows)
    rng = np.random.default_rng(21)
    lengths = rng.integers(0, 40, size=(T, B))
    idx = np.concatenate([_ids(rng, rows[t], int(lengths[t].sum()), zipf) for t in range(T)])
    ix = torch.from_numpy(idx.astype(np.int32)).cuda()
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    up_np = rng.standard_normal((B, sum(dims))).astype(np.float32)
    up = torch.from_numpy(up_np).cuda()
    grp = tbe.TableGroup(rows, dims, dtype=torch.float32, optim="sgd")
    dense = [torch.zeros((r, d), dtype=torch.float32, device="cuda") for r, d in zip(rows, dims)]
    assert grp._bucketed("dense", B, up, up.stride(0), "sum", dense)
    grp.backward(ix, off, B, up, mode="dense", dense_grads=dense)
    torch.cuda.synchronize()
    tab_off = O.offsets_of(lengths.sum(axis=1))
    col = 0
    for t, D in enumerate(dims):
        part = idx[tab_off[t]:tab_off[t + 1]]
        u = np.ascontiguousarray(up_np[:, col:col + D].astype(np.float64))
        ids, gr = O.backward_aggregate_c(lengths[t], part, u)
        _, ga = O.backward_aggregate_c(lengths[t], part, np.abs(u))
        got = dense[t].double().cpu().numpy()
        assert (np.abs(got[ids] - gr) <= 1e-5 * ga + 1e-30).all(), f"table {t}"
        untouched = np.ones(rows[t], bool)
        untouched[ids] = False
        assert not got[untouched].any()
        col += D


def test_bucket_matches_stream_variant(tbe):
    """The bucketed path and the streamed walk (NEO_BWD_VARIANT=stream) agree
    to f32 rounding on the same step."""
    rows, dims, B = [50000, 20000], [128, 128], 4096
    rng = np.random.default_rng(2)
    lengths = rng.integers(0, 33, size=(2, B))
    idx = np.concatenate([rng.integers(0, r, size=int(lengths[t].sum())) for t, r in enumerate(rows)])
    off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
    ix = torch.from_numpy(idx.astype(np.int32)).cuda()
    up = torch.from_numpy(rng.standard_normal((B, 256)).astype(np.float32)).cuda()
    counts = [int(c) for c in lengths.sum(axis=1)]
    outs = []
    for variant in ("bucket", "stream"):
        grp = _group(tbe, rows, dims, torch.float32, "rowwise_adagrad")
        os.environ["NEO_BWD_VARIANT"] = variant
        try:
            grp.backward(ix, off, B, up, mode="update", optim="rowwise_adagrad", lr=0.05, eps=1e-8,
                         table_counts=counts)
            torch.cuda.synchronize()
        finally:
            os.environ.pop("NEO_BWD_VARIANT", None)
        outs.append(grp._storage.clone())
    assert torch.allclose(outs[0], outs[1], rtol=1e-5, atol=1e-6)
