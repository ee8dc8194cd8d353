"""GPU: training through the HBM tier over host-resident tables
(tier.TieredTableGroup: pinned host rows + HBM slot cache + neo_tier_prepare)
matches training the same tables fully in HBM: pooled outputs every step,
and the flushed host tables and optimizer state after the last step.
BITWISE on uniform ids; on skewed ids the backward folds hot rows through
128-entry chunk partials whose grouping follows the row's position in the
sorted stream (slot order vs row order), so there the bar is f32
summation-order tolerance (1e-4 relative after several steps).  The cache holds a small fraction of the rows, so rows are
evicted, written back and re-fetched across steps."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mods():
    import paper_2104_05158_b200 as p
    from paper_2104_05158_b200 import tbe, tier

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    p.load()
    return tbe, tier


@pytest.mark.parametrize("dtype,optim,zipf", [(torch.float32, "rowwise_adagrad", 0.0),
                                              (torch.float32, "rowwise_adagrad", 1.1),
                                              (torch.float16, "rowwise_adagrad", 0.0),
                                              (torch.float32, "sgd", 1.05),
                                              (torch.float32, "adagrad", 0.0)])
def test_tier_training_matches_full_hbm(mods, dtype, optim, zipf):
    tbe, tier = mods
    rows, dims, B, L, steps = [60000, 20000], [128, 64], 512, 8, 4
    T = len(rows)
    rng = np.random.default_rng(17)
    init = [rng.standard_normal((r, d)).astype(np.float32) for r, d in zip(rows, dims)]
    full = tbe.TableGroup(rows, dims, dtype=dtype, optim=optim)
    for w, v in zip(full.weights, init):
        w.copy_(torch.from_numpy(v).to(dtype))
    tg = tier.TieredTableGroup(rows, dims, num_sets=[512, 256], ways=32, dtype=dtype, optim=optim)
    for t in range(T):
        tg.host_w[t].copy_(torch.from_numpy(init[t]).to(dtype))
    counts = [B * L] * T
    off = torch.arange(0, T * B + 1, dtype=torch.int64, device="cuda") * L
    for s in range(steps):
        parts = []
        for r in rows:
            if zipf > 0:
                parts.append(np.minimum(rng.zipf(zipf, B * L) - 1, r - 1))
            else:
                parts.append(rng.integers(0, r, B * L))
        ix = torch.from_numpy(np.concatenate(parts).astype(np.int32)).cuda()
        up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
        a = full.forward(ix, off, B)
        b = tg.forward(ix, off, B, counts)
        if zipf == 0:
            assert torch.equal(a, b), f"pooled outputs differ at step {s}"
        else:
            # the weights entering this forward already carry the summation-order
            # differences of the previous steps' hot-row gradients
            assert torch.allclose(a, b, rtol=1e-4, atol=1e-5 * float(a.abs().max())), f"pooled outputs, step {s}"
        full.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8, table_counts=counts)
        tg.backward(off, B, up, counts, lr=0.05, eps=1e-8)
    tg.flush()
    assert tg.stats["misses"] > 0
    if zipf == 0:
        assert tg.stats["writebacks"] > 0  # uniform ids overflow the cache: rows were evicted and re-fetched
    for t in range(T):
        fw, hw = full.weights[t].cpu(), tg.host_w[t]
        if zipf == 0:
            assert torch.equal(fw, hw), f"table {t} values"
        else:
            assert torch.allclose(fw.float(), hw.float(), rtol=1e-4, atol=1e-5), f"table {t} values"
        if full.moments[t] is not None:
            fm, hm = full.moments[t].cpu(), tg.host_m[t]
            if zipf == 0:
                assert torch.equal(fm, hm), f"table {t} optimizer state"
            else:
                assert torch.allclose(fm, hm, rtol=1e-4, atol=1e-7), f"table {t} optimizer state"


def test_tier_errors(mods):
    tbe, tier = mods
    tg = tier.TieredTableGroup([1000], [32], num_sets=1, ways=2, spill=0)
    off = torch.tensor([0, 4], dtype=torch.int64, device="cuda")
    with pytest.raises(tier.InvalidValue):  # one set, 2 ways, 3 distinct rows in one batch, no spill slots
        tg.forward(torch.tensor([1, 2, 3, 1], dtype=torch.int32, device="cuda"), off, 1, [4])
    tg.spill_ok = tier.TieredTableGroup([1000], [32], num_sets=1, ways=2)  # default spill slots: served
    assert tg.spill_ok.forward(torch.tensor([1, 2, 3, 1], dtype=torch.int32, device="cuda"), off, 1, [4]).shape == (1, 32)
    assert tg.spill_ok.stats["spills"] == 1
    tg2 = tier.TieredTableGroup([1000], [32], num_sets=8, ways=4, table_ids=["emb"])
    import paper_2104_05158_b200 as p

    with pytest.raises(p.IndexOutOfRange):
        tg2.forward(torch.tensor([1, 2, 1000, 1], dtype=torch.int32, device="cuda"), off, 1, [4])


@pytest.mark.parametrize("optim", ["rowwise_adagrad", "adagrad"])
def test_tier_set_overflow_spills_and_matches_full_hbm(mods, optim):
    """A cache far too small for one batch (4 ways, 128 sets: every set sees
    ~15 distinct rows per batch): the overflowing rows take spill slots, are
    fetched, updated and written back; training stays bitwise equal to the
    full-HBM tables (uniform ids)."""
    tbe, tier = mods
    rows, dims, B, L, steps = [40000, 9000], [64, 32], 256, 8, 3
    T = len(rows)
    rng = np.random.default_rng(23)
    init = [rng.standard_normal((r, d)).astype(np.float32) for r, d in zip(rows, dims)]
    full = tbe.TableGroup(rows, dims, dtype=torch.float32, optim=optim)
    for w, v in zip(full.weights, init):
        w.copy_(torch.from_numpy(v))
    tg = tier.TieredTableGroup(rows, dims, num_sets=128, ways=4, optim=optim, spill=4096)
    for t in range(T):
        tg.host_w[t].copy_(torch.from_numpy(init[t]))
    counts = [B * L] * T
    off = torch.arange(0, T * B + 1, dtype=torch.int64, device="cuda") * L
    for s in range(steps):
        ix = torch.from_numpy(np.concatenate([rng.integers(0, r, B * L) for r in rows]).astype(np.int32)).cuda()
        up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
        a = full.forward(ix, off, B)
        b = tg.forward(ix, off, B, counts)
        assert torch.equal(a, b), f"pooled outputs differ at step {s}"
        full.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8, table_counts=counts)
        tg.backward(off, B, up, counts, lr=0.05, eps=1e-8)
    tg.flush()
    assert tg.stats["spills"] > 1000
    for t in range(T):
        assert torch.equal(full.weights[t].cpu(), tg.host_w[t]), f"table {t} values"
        assert torch.equal(full.moments[t].cpu(), tg.host_m[t]), f"table {t} optimizer state"


def test_tier_spill_exhausted_raises(mods):
    tbe, tier = mods
    tg = tier.TieredTableGroup([5000], [32], num_sets=2, ways=2, spill=8)
    ix = torch.arange(0, 2048, dtype=torch.int32, device="cuda")
    off = torch.tensor([0, 2048], dtype=torch.int64, device="cuda")
    from paper_2104_05158_b200.errors import InvalidValue
    with pytest.raises(InvalidValue):
        tg.forward(ix, off, 1, [2048])


@pytest.mark.parametrize("optim", ["rowwise_adagrad", "sgd"])
def test_hybrid_tables_match_full_hbm(mods, optim):
    """Tables split by rows between HBM and the host tier (HybridTableGroup):
    pooled outputs are the two part sums (row-wise-shard rounding, f32
    tolerance), updated weights and optimizer state bitwise equal to the
    whole tables in HBM; the host part spills when its sets overflow."""
    tbe, tier = mods
    rows, dims, hbm_rows, B, steps = [50000, 30000, 7000], [128, 64, 32], [30000, 8000, 6999], 384, 3
    T = len(rows)
    rng = np.random.default_rng(29)
    init = [rng.standard_normal((r, d)).astype(np.float32) for r, d in zip(rows, dims)]
    full = tbe.TableGroup(rows, dims, dtype=torch.float32, optim=optim)
    for w, v in zip(full.weights, init):
        w.copy_(torch.from_numpy(v))
    hy = tier.HybridTableGroup(rows, dims, hbm_rows, num_sets=256, ways=8, optim=optim)
    for t in range(T):
        hy.hbm.weights[t].copy_(torch.from_numpy(init[t][:hbm_rows[t]]))
        hy.host.host_w[t].copy_(torch.from_numpy(init[t][hbm_rows[t]:]))
    for s in range(steps):
        lengths = rng.integers(0, 20, size=(T, B))
        idx = np.concatenate([rng.integers(0, rows[t], int(lengths[t].sum())) for t in range(T)]).astype(np.int32)
        off = tbe.lengths_to_offsets(torch.from_numpy(lengths.reshape(-1)).cuda())
        ix = torch.from_numpy(idx).cuda()
        up = torch.from_numpy(rng.standard_normal((B, sum(dims))).astype(np.float32)).cuda()
        a = full.forward(ix, off, B)
        b = hy.forward(ix, off, B)
        assert torch.allclose(a, b, rtol=1e-5, atol=1e-5), f"pooled outputs, step {s}"
        full.backward(ix, off, B, up, mode="update", optim=optim, lr=0.05, eps=1e-8,
                      table_counts=[int(c) for c in lengths.sum(axis=1)])
        hy.backward(B, up, lr=0.05, eps=1e-8)
    hy.flush()
    assert hy.host.stats["spills"] > 0
    for t in range(T):
        h = hbm_rows[t]
        fw = full.weights[t].cpu()
        assert torch.equal(fw[:h], hy.hbm.weights[t].cpu()), f"table {t} HBM rows"
        assert torch.equal(fw[h:], hy.host.host_w[t]), f"table {t} host rows"
        if full.moments[t] is not None:
            fm = full.moments[t].cpu()
            assert torch.equal(fm[:h], hy.hbm.moments[t].cpu()) and torch.equal(fm[h:], hy.host.host_m[t])
