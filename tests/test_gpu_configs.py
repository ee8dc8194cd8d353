"""The BASELINE configs 3-5 as parity cases, on one GPU.

* c4 index bucketisation at FULL size: 4 tables x 100M rows, 65,536 bags
  x 32 ids per table, row bounds from the committed c4_rw_w{2,4,8} plans;
  bit-exact against the oracle (comms.py:107-141).
* c4 row-wise / column-wise sharded steps (rows scaled 100x so the oracle
  and two copies of the tables fit), c3 table-wise over 256 tables, and
  c5's mixed TW/RW/CW/DP plan over 512 skewed tables with Zipf(1.05) ids
  and fp16/bf16 wires (rows scaled to [1e3, 1e5]; the committed c5s plan):
  the production engine on W logical ranks (dist.LocalComm) against the
  f64 C oracle run on the touched rows only (ids remapped monotonically, so
  the oracle's buffer-order sums and ascending-row updates are unchanged).
  Untouched rows must be bit-identical to their initial values.

Tolerances: pooled |got - ref| <= 1e-5 * sum|terms|, plus
2^-11 * sum|terms| for the fp16 wire; updated weights within 1e-5 of
|w| + |dw|; the bf16 wire is fed to the oracle as the bf16-rounded upstream.
"""
import json
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import tbe_oracle as O  # noqa: E402

pytestmark = pytest.mark.gpu
PLANS = ROOT / "configs" / "plans"


@pytest.fixture(scope="module")
def pkg():
    import paper_2104_05158_b200 as p

    assert torch.cuda.is_available()
    p.load()
    return p


# ---------------------------------------------------------------------------
# c4 bucketisation, full size


@pytest.mark.parametrize("k", [2, 4, 8])
def test_c4_bucketize_full_size_bitexact(pkg, k):
    from paper_2104_05158_b200 import tbe

    doc = json.loads((PLANS / f"c4_rw_w{k}.json").read_text())
    rng = np.random.default_rng(40 + k)
    B, L = 65536, 32
    for a in doc["tables"][:2]:  # two of the four tables per k (same bounds; keeps the suite fast)
        bounds = [s["rows"] for s in a["shards"]]
        starts = [b[0] for b in bounds] + [bounds[-1][1]]
        H = starts[-1]
        assert H == 100_000_000
        lens = np.full(B, L, dtype=np.int64)
        lens[rng.random(B) < 0.05] = 0  # empty bags
        lens[rng.random(B) < 0.05] = 64  # longer ones
        ids = rng.integers(0, H, size=int(lens.sum()), dtype=np.int64)
        ids[-5:] = [0, H - 1, starts[1] - 1, starts[1], starts[-2]]  # shard edges
        want = O.bucketize_c(lens, ids, starts)
        off = tbe.lengths_to_offsets(torch.from_numpy(lens).cuda())
        for dt in (torch.int32, torch.int64):
            gl, go, gi = tbe.bucketize_rowwise(off, torch.from_numpy(ids).to(dt).cuda(), starts)
            gl, go, gi = gl.cpu().numpy(), go.cpu().numpy(), gi.cpu().numpy()
            for s, (wl, wi) in enumerate(want):
                assert np.array_equal(gl[s], wl), (k, s, dt)
                assert np.array_equal(gi[go[s * B]:go[(s + 1) * B]].astype(np.int64), wi), (k, s, dt)


# ---------------------------------------------------------------------------
# sharded steps against the touched-row oracle


def _device_tables(specs, seed):
    g = torch.Generator(device="cuda").manual_seed(seed)
    return [torch.randn((t.num_rows, t.dim), generator=g, device="cuda") for t in specs]


def _run(pkg, specs, plan, W, B, optim, seed, fwd=None, bwd=None, lr=0.05, eps=1e-8):
    from paper_2104_05158_b200 import dist
    from paper_2104_05158_b200.comms import _local_batches

    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    lengths, indices = O.synthetic_batch(specs, W * B, seed)
    batch = pkg.CombinedBatch(lengths, indices)
    full = _device_tables(specs, seed + 1)
    eng = dist.ShardedEmbedding(model, plan, dist.LocalComm(W), B, dtype=torch.float32, optim=optim,
                                fwd_comm=fwd, bwd_comm=bwd, index_dtype=torch.int64,
                                init=lambda t, r, c: full[t][r[0]:r[1], c[0]:c[1]])
    rng = np.random.default_rng(seed + 2)
    up = rng.standard_normal((W * B, sum(t.dim for t in specs))).astype(np.float32)
    ups = iter([torch.from_numpy(up[w * B:(w + 1) * B]).cuda() for w in range(W)])
    pooled = eng.step(_local_batches(batch, W), lr=lr, eps=eps, upstream_fn=lambda p: next(ups))
    got = torch.cat([p.double() for p in pooled]).cpu().numpy()
    return eng, full, lengths, indices, up, got


def _check(eng, specs, full, lengths, indices, up, got, optim, fwd_q=False, bwd_q=False, lr=0.05, eps=1e-8):
    lay = eng.lay
    dp = set(lay.dp_tables)
    dcol = np.concatenate(([0], np.cumsum([t.dim for t in specs])))
    tab_off = O.offsets_of(lengths.sum(axis=1))
    cache = {}
    for t, spec in enumerate(specs):
        part = indices[tab_off[t]:tab_off[t + 1]]
        uniq, remap = np.unique(part, return_inverse=True)
        vals = full[t][torch.from_numpy(uniq).cuda()].double().cpu().numpy() if len(uniq) else \
            np.zeros((0, spec.dim))
        cache[t] = (uniq, remap.astype(np.int64), vals)
        want = O.forward_pooled_c(vals, lengths[t], remap)
        bound = O.forward_pooled_c(np.abs(vals), lengths[t], remap)
        q = fwd_q and t not in dp
        rel = 1e-5 + (2.0 ** -11 if q else 0.0)
        # fp16 wire: half an ulp per rounded partial (relative 2^-11), and at
        # most 2^-25 absolute for partials in fp16's subnormal range, per shard
        absq = len(eng.lay.owned) * 2.0 ** -25 if q else 1e-30
        err = np.abs(got[:, dcol[t]:dcol[t + 1]] - want)
        assert (err <= rel * bound + absq).all(), (spec.id, float((err - rel * bound - absq).max()))
    upq = up.astype(np.float64)
    if bwd_q:
        upb = O.bf16_roundtrip(upq)
        for t in range(len(specs)):
            if t not in dp:
                upq[:, dcol[t]:dcol[t + 1]] = upb[:, dcol[t]:dcol[t + 1]]
    shards = [(s.table, s.rows, s.cols, w) for slot in range(len(eng.states))
              for s, w, _ in eng.shard_tensors(slot)]
    st0 = eng.states[0]
    if st0.dp_group is not None:
        shards += [(t, (0, specs[t].num_rows), (0, specs[t].dim), w) for t, w in zip(lay.dp_tables,
                                                                                     st0.dp_group.weights)]
    seen = set()
    for t, (r0, r1), (c0, c1), w in shards:
        seen.add(t)
        uniq, remap, vals = cache[t]
        ids, g = O.backward_aggregate_c(lengths[t], remap,
                                        np.ascontiguousarray(upq[:, dcol[t] + c0:dcol[t] + c1]))
        keep = (uniq[ids] >= r0) & (uniq[ids] < r1)
        rows = uniq[ids[keep]]
        base = vals[ids[keep]][:, c0:c1]
        v = base.copy()
        mom = {"rowwise_adagrad": np.zeros(len(v)), "adagrad": np.zeros_like(v), "sgd": None}[optim]
        O.apply_c(optim, v, mom, np.arange(len(v), dtype=np.int64), np.ascontiguousarray(g[keep]), lr, eps)
        gw = w[torch.from_numpy(rows - r0).cuda()].double().cpu().numpy()
        # f32 gradient sums carry 1e-5 * sum|terms|; propagate it through the update
        _, gabs = O.backward_aggregate_c(lengths[t], remap,
                                         np.ascontiguousarray(np.abs(upq[:, dcol[t] + c0:dcol[t] + c1])))
        dg = 1e-5 * gabs[keep]
        gk = g[keep]
        if optim == "sgd":
            gtol = lr * dg
        elif optim == "adagrad":
            gtol = lr * np.minimum(2.0, 2.0 * dg / np.maximum(np.abs(gk), 1e-300))
        else:
            rms = np.sqrt((gk ** 2).mean(axis=1, keepdims=True)) if gk.size else np.zeros((0, 1))
            gtol = lr * np.minimum(2.0, 2.0 * dg.max(axis=1, keepdims=True) / np.maximum(rms, 1e-300)) \
                if gk.size else np.zeros_like(gk)
        tol = 1e-5 * (np.abs(v) + np.abs(v - base)) + 1e-6 + gtol
        assert (np.abs(gw - v) <= tol).all(), (specs[t].id, r0, c0, float((np.abs(gw - v) - tol).max()))
        changed = ((w != full[t][r0:r1, c0:c1]).any(dim=1).nonzero().flatten().cpu().numpy() + r0)
        assert np.isin(changed, rows).all(), (specs[t].id, "an untouched row changed")
    assert seen == set(range(len(specs)))


@pytest.mark.parametrize("W", [2, 4, 8])
def test_c4_rowwise_sharded_step(pkg, W):
    from paper_2104_05158_b200 import plan as P

    H = 1_000_000  # c4's 100M rows scaled 100x
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=H, dim=256, avg_pooling=32.0) for i in range(4)]
    plan = P.ShardingPlan(W, W, tuple(
        P.TableAssignment(t.id, P.Scheme(P.SchemeKind.ROW_WISE, num_row_shards=W),
                          tuple(P.Shard(i, rows=b) for i, b in enumerate(P.even_bounds(H, W)))) for t in specs))
    eng, full, lengths, indices, up, got = _run(pkg, specs, plan, W, 128, "rowwise_adagrad", seed=400 + W)
    _check(eng, specs, full, lengths, indices, up, got, "rowwise_adagrad")


def test_c4_columnwise_sharded_step(pkg):
    from paper_2104_05158_b200 import plan as P

    W, H = 4, 1_000_000
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=H, dim=256, avg_pooling=32.0) for i in range(4)]
    doc = json.loads((PLANS / "c4_cw_w4.json").read_text())  # the committed column split, rows scaled
    plan = P.plan_from_json(json.dumps(doc))
    eng, full, lengths, indices, up, got = _run(pkg, specs, plan, W, 128, "rowwise_adagrad", seed=44)
    _check(eng, specs, full, lengths, indices, up, got, "rowwise_adagrad")


def test_c3_tablewise_sharded_step(pkg):
    from paper_2104_05158_b200 import plan as P

    W = 8
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=20_000, dim=128, avg_pooling=32.0) for i in range(256)]
    plan = P.plan_from_json((PLANS / "c3_w8.json").read_text())  # reference plan_4d placement (TW)
    eng, full, lengths, indices, up, got = _run(pkg, specs, plan, W, 32, "rowwise_adagrad", seed=33)
    _check(eng, specs, full, lengths, indices, up, got, "rowwise_adagrad")


@pytest.mark.parametrize("optim", ["rowwise_adagrad", "sgd", "adagrad"])
def test_c5_mixed_plan_skewed_quantized(pkg, optim):
    from paper_2104_05158_b200 import plan as P
    from paper_2104_05158_b200 import spec

    W = 8
    model = spec.model_from_json((ROOT / "configs" / "models" / "c5s.json").read_text())
    plan = P.plan_from_json((PLANS / "c5s_w8.json").read_text())
    kinds = {a.scheme.kind.value for a in plan.assignments}
    assert kinds == {"table_wise", "row_wise", "column_wise", "data_parallel"}
    specs = list(model.tables)
    quant = optim == "rowwise_adagrad"
    eng, full, lengths, indices, up, got = _run(
        pkg, specs, plan, W, 4, optim, seed=55, fwd=torch.float16 if quant else None,
        bwd=torch.bfloat16 if quant else None)
    _check(eng, specs, full, lengths, indices, up, got, optim, fwd_q=quant, bwd_q=quant)
