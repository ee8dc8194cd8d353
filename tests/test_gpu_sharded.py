"""Sharded step on W logical ranks (dist.LocalComm, one GPU) through the
production engine, against the reference's own train_step_sharded /
alltoall_redistribute outputs (tests/golden/steps*.{npz,json}).  The f64
path reproduces the reference's order of operations, so outputs and
reassembled tables must be BIT-identical to the reference's sharded step
(and within 1e-9 of its single-worker step, cli.py:50)."""
import hashlib
import json

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import paper_2104_05158_b200 as p

    assert torch.cuda.is_available()
    p.load()
    return p


def _case(pkg, meta, z, c):
    tables = [pkg.TableSpec(id=d["id"], num_rows=d["num_rows"], dim=d["dim"], avg_pooling=d["avg_pooling"],
                            value_precision=pkg.Precision(d["value_precision"])) for d in meta["tables"]]
    model = pkg.ModelSpec(tables=tuple(tables), local_batch=meta["local_batch"])
    plan = pkg.plan_from_json(json.dumps(meta["plan"]))
    batch = pkg.CombinedBatch(z[f"s{c}_lengths"], z[f"s{c}_indices"])
    cfg = pkg.OptimizerConfig(pkg.OptimizerKind(meta["kind"]), lr=meta["lr"], eps=meta["eps"])
    return model, plan, batch, cfg


def test_sharded_step_bitwise_vs_reference(pkg, steps_golden):
    z, plans = steps_golden
    for c, meta in plans.items():
        model, plan, batch, cfg = _case(pkg, meta, z, c)
        out, state = pkg.train_step_sharded(model, plan, batch, cfg, seed=meta["seed"])
        assert np.array_equal(out, z[f"s{c}_sh_out"]), c
        assert np.max(np.abs(out - z[f"s{c}_ref_out"]), initial=0.0) <= 1e-9
        vals = pkg.reassemble_values(model, plan, state)
        for t, v in enumerate(vals):
            assert np.array_equal(v, z[f"s{c}_sh_t{t}"]), (c, t)
            assert np.max(np.abs(v - z[f"s{c}_ref_t{t}"]), initial=0.0) <= 1e-9
        for tid, reps in state.dp_replicas.items():  # test_comms.py:341-361
            for r in reps[1:]:
                assert np.array_equal(r.values, reps[0].values)


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_alltoall_redistribute_bit_exact(pkg, steps_golden):
    z, plans = steps_golden
    for c, meta in plans.items():
        model, plan, batch, _ = _case(pkg, meta, z, c)
        W = plan.num_workers
        slices = pkg.alltoall_redistribute(pkg.to_wtb(batch, W), plan, model)
        got = {}
        for ws in slices:
            for si in ws.inputs:
                s = si.shard
                key = (ws.worker, si.table_id, tuple(s.rows) if s.rows else None, tuple(s.cols) if s.cols else None)
                got[key] = (si.sample_base, _sha(np.asarray(si.lengths, dtype=np.int64)),
                            _sha(np.asarray(si.indices, dtype=np.int64)))
        want = {}
        for r in meta["redistribute"]:
            key = (r["worker"], r["table_id"], tuple(r["rows"]) if r["rows"] else None,
                   tuple(r["cols"]) if r["cols"] else None)
            want[key] = (r["sample_base"], r["lengths_sha"], r["indices_sha"])
        assert got == want, c


def test_sharded_f32_engine_matches_oracle(pkg):
    """Production f32 engine on 4 logical ranks with a mixed TW/RW/CW/DP
    plan and random upstream: pooled outputs and updated shards vs the f64
    oracle within the stated tolerance."""
    from oracle import tbe_oracle as O
    from paper_2104_05158_b200 import dist, plan as P

    rng = np.random.default_rng(1)
    W, B = 4, 64
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=int(r), dim=int(d), avg_pooling=6.0)
             for i, (r, d) in enumerate([(500, 64), (900, 32), (300, 128), (50, 16), (700, 64), (400, 96)])]
    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    A = P.TableAssignment
    plan = P.ShardingPlan(W, W, (
        A("t0", P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(2),)),
        A("t1", P.Scheme(P.SchemeKind.ROW_WISE, num_row_shards=3),
          tuple(P.Shard(w, rows=b) for w, b in zip((1, 3, 0), P.even_bounds(900, 3)))),
        A("t2", P.Scheme(P.SchemeKind.COLUMN_WISE, col_splits=((0, 64), (64, 128))),
          (P.Shard(0, cols=(0, 64)), P.Shard(3, cols=(64, 128)))),
        A("t3", P.Scheme(P.SchemeKind.DATA_PARALLEL), (P.Shard(None),)),
        A("t4", P.Scheme(P.SchemeKind.ROW_WISE, num_row_shards=4),
          tuple(P.Shard(w, rows=b) for w, b in zip((0, 1, 2, 3), P.even_bounds(700, 4)))),
        A("t5", P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(1),)),
    ))
    batch = pkg.gen_synthetic_batch(model, W * B, seed=3)
    full = [rng.standard_normal((t.num_rows, t.dim)).astype(np.float32).astype(np.float64) for t in specs]

    def init(t, rows, cols):
        return torch.from_numpy(full[t][rows[0]:rows[1], cols[0]:cols[1]].copy())

    eng = dist.ShardedEmbedding(model, plan, dist.LocalComm(W), B, dtype=torch.float32, optim="rowwise_adagrad",
                                init=init)
    from paper_2104_05158_b200.comms import _local_batches
    up_full = rng.standard_normal((W * B, sum(t.dim for t in specs))).astype(np.float32)
    ups = [torch.from_numpy(up_full[w * B:(w + 1) * B]).cuda() for w in range(W)]
    it = iter(range(W))
    pooled = eng.step(_local_batches(batch, W), lr=0.05, eps=1e-8, upstream_fn=lambda p: ups[next(it)])
    got = torch.cat(pooled).double().cpu().numpy()
    # oracle: unsharded forward; row-wise AdaGrad per shard slice (CW shards keep their own moments)
    L = np.asarray(batch.lengths)
    tab_off = O.offsets_of(L.sum(axis=1))
    col = 0
    for t, spec in enumerate(specs):
        part = np.asarray(batch.indices)[tab_off[t]:tab_off[t + 1]]
        want = O.forward_pooled_c(full[t], L[t], part)
        bound = O.forward_pooled_c(np.abs(full[t]), L[t], part)
        assert (np.abs(got[:, col:col + spec.dim] - want) <= 1e-5 * bound + 1e-30).all(), spec.id
        col += spec.dim
    for slot in range(W):
        for s, w, m in eng.shard_tensors(slot):
            t = s.table
            r0, r1 = s.rows
            c0, c1 = s.cols
            part = np.asarray(batch.indices)[tab_off[t]:tab_off[t + 1]]
            mc = sum(x.dim for x in specs[:t])
            ids, g = O.backward_aggregate_c(L[t], part, np.ascontiguousarray(up_full[:, mc + c0:mc + c1].astype(np.float64)))
            keep = (ids >= r0) & (ids < r1)
            v = full[t][r0:r1, c0:c1].copy()
            mom = np.zeros(r1 - r0)
            O.apply_c("rowwise_adagrad", v, mom, ids[keep] - r0, g[keep], 0.05, 1e-8)
            gw = w.double().cpu().numpy()
            base = full[t][r0:r1, c0:c1]
            assert (np.abs(gw - v) <= 1e-5 * (np.abs(v) + np.abs(v - base)) + 1e-6).all(), (s.table_id, s.index)


def test_quantized_alltoall_fp16_fwd_bf16_bwd(pkg):
    """Paper-style quantized communication: pooled rows cross
    the all-to-all as fp16 (written by the TBE epilogue), gradients as bf16.
    Received pooled values equal the fp16 rounding of the f32 result
    (comms oracle: quantize_fp16_roundtrip, embedding.py:288-299); the update
    sees the bf16-rounded upstream (restated RNE, parity unpinned)."""
    from oracle import tbe_oracle as O
    from paper_2104_05158_b200 import dist, plan as P
    from paper_2104_05158_b200.comms import _local_batches

    rng = np.random.default_rng(4)
    W, B = 2, 128
    specs = [pkg.TableSpec(id=f"t{i}", num_rows=2000, dim=128, avg_pooling=8.0) for i in range(3)]
    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    plan = P.ShardingPlan(W, W, tuple(P.TableAssignment(t.id, P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(i % W),))
                                      for i, t in enumerate(specs)))
    full = [rng.standard_normal((2000, 128)).astype(np.float32) for _ in specs]
    batch = pkg.gen_synthetic_batch(model, W * B, seed=11)

    def run(fwd, bwd):
        eng = dist.ShardedEmbedding(model, plan, dist.LocalComm(W), B, dtype=torch.float32, optim="sgd",
                                    fwd_comm=fwd, bwd_comm=bwd,
                                    init=lambda t, r, c: torch.from_numpy(full[t][r[0]:r[1], c[0]:c[1]].copy()))
        up = torch.from_numpy(rng.standard_normal((B, 384)).astype(np.float32)).cuda()
        pooled = [p.clone() for p in eng.step(_local_batches(batch, W), lr=0.1, upstream_fn=lambda p: up)]
        return eng, torch.cat(pooled).double().cpu().numpy(), up

    eng32, p32, _ = run(None, None)
    engq, pq, up = run(torch.float16, torch.bfloat16)
    assert np.array_equal(pq, O.fp16_roundtrip(p32)[0])  # one fp16 rounding of the same f32 sums
    # the bf16 wire rounds the upstream once: check the SGD update of every shard
    upb = O.bf16_roundtrip(up.double().cpu().numpy())
    L = np.asarray(batch.lengths)
    tab_off = O.offsets_of(L.sum(axis=1))
    for slot in range(W):
        for s, w, _ in engq.shard_tensors(slot):
            t = s.table
            part = np.asarray(batch.indices)[tab_off[t]:tab_off[t + 1]]
            ups = np.concatenate([upb] * W)[:, 128 * t:128 * (t + 1)]  # every worker used the same upstream
            ids, g = O.backward_aggregate_c(L[t], part, np.ascontiguousarray(ups))
            v = full[t].astype(np.float64)
            O.apply_c("sgd", v, None, ids, g, 0.1, 0.0)
            got = w.double().cpu().numpy()
            assert (np.abs(got - v) <= 1e-5 * (np.abs(v) + np.abs(v - full[t])) + 1e-6).all()
    # byte contract: fp16 payload is exactly half of fp32 (criterion 8, test_acceptance.py:318-343)
    assert engq.pooled_send_bytes(0) * 2 == eng32.pooled_send_bytes(0)


@pytest.mark.parametrize("bad_table", [0, 1])
def test_sharded_step_raises_index_out_of_range_before_any_update(pkg, bad_table):
    """An id outside its table raises the reference's IndexOutOfRange (table
    id, value) from ShardedEmbedding.step before any shard is touched
    (model.py:344-348; forward_pooled / bucketize_rowwise raise, embedding.py:
    144-146, comms.py:127-129) — for a table-wise and a row-wise table."""
    from paper_2104_05158_b200 import dist, plan as P
    from paper_2104_05158_b200.comms import _local_batches
    from paper_2104_05158_b200.errors import IndexOutOfRange

    W, B = 2, 64
    specs = [pkg.TableSpec(id="tw", num_rows=500, dim=32, avg_pooling=4.0),
             pkg.TableSpec(id="rw", num_rows=900, dim=32, avg_pooling=4.0)]
    model = pkg.ModelSpec(tables=tuple(specs), local_batch=B)
    plan = P.ShardingPlan(W, W, (
        P.TableAssignment("tw", P.Scheme(P.SchemeKind.TABLE_WISE), (P.Shard(0),)),
        P.TableAssignment("rw", P.Scheme(P.SchemeKind.ROW_WISE),
                          (P.Shard(0, rows=(0, 450)), P.Shard(1, rows=(450, 900))))))
    batch = pkg.gen_synthetic_batch(model, W * B, seed=5)
    L = np.asarray(batch.lengths)
    idx = np.asarray(batch.indices).copy()
    tab_off = np.concatenate(([0], np.cumsum(L.sum(axis=1))))
    bad_pos = int(tab_off[bad_table]) + 3
    idx[bad_pos] = specs[bad_table].num_rows + 7
    full = [torch.randn((t.num_rows, t.dim)) for t in specs]
    eng = dist.ShardedEmbedding(model, plan, dist.LocalComm(W), B, dtype=torch.float32, optim="sgd",
                                index_dtype=torch.int64,
                                init=lambda t, r, c: full[t][r[0]:r[1], c[0]:c[1]].contiguous())
    before = [w.clone() for slot in range(W) for _, w, _ in eng.shard_tensors(slot)]
    with pytest.raises(IndexOutOfRange) as e:
        eng.step(_local_batches(pkg.CombinedBatch(L, idx), W), lr=0.1)
    assert e.value.table_id == specs[bad_table].id and e.value.index == specs[bad_table].num_rows + 7
    after = [w for slot in range(W) for _, w, _ in eng.shard_tensors(slot)]
    assert all(torch.equal(a, b) for a, b in zip(before, after))
