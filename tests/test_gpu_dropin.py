"""Drop-in integration: the reference package itself (installed offline into
oracle/_ref by oracle/make_ref.py, which travels with the repo snapshot) is patched with
dropin.install(); every patched call must return exactly what the
unpatched reference returns on the same inputs (the reference's numpy code
runs on the host as the checker).  Includes an acceptance-criterion-5 style
sweep of seeded random plans (all schemes incl. hierarchical row-wise, all
three optimizers) and the reference CLI's `verify` command end to end."""
import json
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

# the reference package as copied by oracle/make_ref.py (git-ignored, shipped
# with the snapshot); baseline/_ref (a pip --target install) also works
_ROOT = Path(__file__).resolve().parent.parent
REF = _ROOT / "oracle" / "_ref" if (_ROOT / "oracle" / "_ref" / "neosim").exists() else _ROOT / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "neosim").exists():
        pytest.fail("reference package missing: run __graft_entry__.build() (oracle/make_ref.py copies it into "
                    "oracle/_ref where /root/reference exists)")
    sys.path.insert(0, str(REF))
    import neosim
    from neosim import cli, comms, embedding

    originals = {
        "train_step_reference": embedding.train_step_reference,
        "train_step_sharded": comms.train_step_sharded,
        "forward_pooled": embedding.forward_pooled,
        "backward_sort_aggregate": embedding.backward_sort_aggregate,
        "bucketize_rowwise": comms.bucketize_rowwise,
        "alltoall_redistribute": comms.alltoall_redistribute,
        "reassemble_values": comms.reassemble_values,
    }
    from paper_2104_05158_b200 import dropin

    dropin.install(neosim)
    yield neosim, originals
    dropin.uninstall()


def _desk_model(neosim, tables, B):
    return neosim.ModelSpec(tables=tuple(tables), bottom_mlp_layers=(), top_mlp_layers=(), local_batch=B,
                            mflops_per_sample=1.0, interaction_flops_per_sample=0.0, dense_param_bytes=0)


def _random_plan(neosim, rng, model, W, gpn):
    """Seeded scheme mix over TW / RW / CW / DP / hierarchical RW."""
    from neosim.planner import even_bounds

    S, K = neosim.Scheme, neosim.SchemeKind
    out = []
    for t in model.tables:
        c = int(rng.integers(0, 5))
        if c == 4 and W > gpn:
            node = int(rng.integers(0, W // gpn))
            k = min(gpn, t.num_rows)
            sh = tuple(neosim.Shard(worker=node * gpn + i % gpn, rows=b) for i, b in enumerate(even_bounds(t.num_rows, k)))
            out.append(neosim.TableAssignment(t.id, S(K.ROW_WISE, num_row_shards=k, hierarchical=(K.TABLE_WISE, K.ROW_WISE)), sh))
        elif c == 3:
            out.append(neosim.TableAssignment(t.id, S(K.DATA_PARALLEL), (neosim.Shard(worker=None),)))
        elif c == 2 and t.dim % 2 == 0:
            sp = ((0, t.dim // 2), (t.dim // 2, t.dim))
            st = int(rng.integers(0, W))
            out.append(neosim.TableAssignment(t.id, S(K.COLUMN_WISE, col_splits=sp),
                                              tuple(neosim.Shard(worker=(st + i) % W, cols=x) for i, x in enumerate(sp))))
        elif c == 1 and min(W, t.num_rows) >= 2:
            k = int(rng.integers(2, min(W, t.num_rows, 4) + 1))
            st = int(rng.integers(0, W))
            out.append(neosim.TableAssignment(t.id, S(K.ROW_WISE, num_row_shards=k), tuple(
                neosim.Shard(worker=(st + i) % W, rows=b) for i, b in enumerate(even_bounds(t.num_rows, k)))))
        else:
            out.append(neosim.TableAssignment(t.id, S(K.TABLE_WISE), (neosim.Shard(worker=int(rng.integers(0, W))),)))
    return neosim.ShardingPlan(W, gpn, tuple(out))


def test_patched_ops_equal_reference(ref):
    neosim, orig = ref
    rng = np.random.default_rng(0)
    for _ in range(10):
        H, D, n = int(rng.integers(3, 60)), int(rng.integers(1, 9)), int(rng.integers(1, 20))
        lengths = rng.integers(0, 7, size=n)
        idx = rng.integers(0, H, size=int(lengths.sum()))
        spec = neosim.TableSpec(id="t", num_rows=H, dim=D, avg_pooling=1.0)
        table = neosim.EmbeddingTable(spec, rng.standard_normal((H, D)))
        assert np.array_equal(neosim.forward_pooled(table, lengths, idx), orig["forward_pooled"](table, lengths, idx))
        up = rng.standard_normal((n, D))
        a, b = neosim.backward_sort_aggregate(lengths, idx, up), orig["backward_sort_aggregate"](lengths, idx, up)
        assert np.array_equal(a.ids, b.ids) and np.array_equal(a.grads, b.grads)
    with pytest.raises(neosim.IndexOutOfRange):  # the reference's own exception class
        neosim.forward_pooled(neosim.EmbeddingTable(neosim.TableSpec("x", 2, 2, 1.0), np.ones((2, 2))), [1], [5])
    with pytest.raises(neosim.LayoutMismatch):
        neosim.comms.bucketize_rowwise([2], [1], [(0, 5)])


def test_random_plans_criterion5_style(ref):
    neosim, orig = ref
    rng = np.random.default_rng(2024)
    kinds = [neosim.OptimizerKind.SGD, neosim.OptimizerKind.ROWWISE_ADAGRAD, neosim.OptimizerKind.ADAGRAD]
    for trial in range(60):
        tables = [neosim.TableSpec(id=f"t{i}", num_rows=int(rng.integers(8, 33)), dim=int(rng.integers(1, 4)) * 2,
                                   avg_pooling=float(rng.uniform(1.0, 3.5))) for i in range(int(rng.integers(1, 9)))]
        model = _desk_model(neosim, tables, int(rng.integers(1, 4)))
        W = int(rng.choice([1, 2, 4]))
        gpn = 2 if W == 4 and trial % 2 else W
        plan = _random_plan(neosim, rng, model, W, gpn)
        cfg = neosim.OptimizerConfig(kinds[trial % 3], lr=0.1, eps=1e-8)
        seed = int(rng.integers(10_000))
        batch = neosim.gen_synthetic_batch(model, W * model.local_batch, seed)
        want_out, want_state = orig["train_step_sharded"](model, plan, batch, cfg, seed=seed)
        got_out, got_state = neosim.train_step_sharded(model, plan, batch, cfg, seed=seed)
        assert np.array_equal(got_out, want_out), trial
        for g, w in zip(neosim.comms.reassemble_values(model, plan, got_state),
                        orig["reassemble_values"](model, plan, want_state)):
            assert np.array_equal(g, w), trial
        r_out, r_tabs = neosim.train_step_reference(model, batch, cfg, seed=seed)
        o_out, o_tabs = orig["train_step_reference"](model, batch, cfg, seed=seed)
        assert np.array_equal(r_out, o_out)
        for a, b in zip(r_tabs, o_tabs):
            assert np.array_equal(a.values, b.values)


def test_reference_cli_verify_through_dropin(ref, tmp_path):
    neosim, _ = ref
    from neosim import cli, model as M

    tables = [neosim.TableSpec(id=f"t{i}", num_rows=200 + 37 * i, dim=8 * (1 + i % 3), avg_pooling=3.0 + i)
              for i in range(6)]
    spec = _desk_model(neosim, tables, 16)
    path = tmp_path / "model.json"
    path.write_text(M.serialize_model_spec(spec))
    for W in (1, 2, 4):
        out = tmp_path / f"w{W}"
        rc = cli.main(["verify", "--model", str(path), "--workers", str(W), "--optimizer", "rowwise_adagrad",
                       "--out", str(out)])
        assert rc == 0
        body = json.loads((out / "verify.json").read_text())["body"]
        assert body["passed"] and body["max_deviation"] <= 1e-9


def test_cache_simulate_trace_patched(ref):
    """neosim.cache.simulate_trace (and its by-name bindings in cli.py and the
    package) route to the GPU replay and return the reference's TraceStats."""
    neosim, _ = ref
    from neosim import cache as rc, cli

    from paper_2104_05158_b200 import cache as ours

    assert rc.simulate_trace is ours.simulate_trace and cli.simulate_trace is ours.simulate_trace
    rng = np.random.default_rng(9)
    for pol in (rc.ReplacementPolicy.LRU, rc.ReplacementPolicy.LFU):
        cfg = rc.CacheConfig(num_sets=8, ways=4, policy=pol)
        tr = rng.integers(0, 200, 5000).tolist()
        st = rc.simulate_trace(cfg, tr)
        state = rc.CacheState(cfg)  # the reference's own sequential loop as the checker
        for r in tr:
            rc.access(state, r)
        assert isinstance(st, rc.TraceStats)
        assert (st.hits, st.misses, st.evictions) == (state.hits, state.misses, state.evictions)
    with pytest.raises(neosim.EmptyTrace):
        rc.simulate_trace(rc.CacheConfig(num_sets=2), [])
    shipped = rc.make_scan_hot_trace()
    lru = rc.simulate_trace(rc.CacheConfig(num_sets=4, ways=8, policy=rc.ReplacementPolicy.LRU), shipped)
    lfu = rc.simulate_trace(rc.CacheConfig(num_sets=4, ways=8, policy=rc.ReplacementPolicy.LFU), shipped)
    assert lfu.hit_rate > lru.hit_rate  # test_cache.py:97-106
