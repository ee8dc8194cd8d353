"""Host-side plan ingest and exchange layout (CPU): the reference's plan
JSON parses, validates, and each rank's pooled all-to-all volume equals the
reference's byte contract (comms.py:366-392)."""
import json
import os

import numpy as np
import pytest

from paper_2104_05158_b200 import plan as P
from paper_2104_05158_b200.errors import InvalidScheme
from paper_2104_05158_b200.spec import ModelSpec, Precision, TableSpec


def _model(meta):
    return ModelSpec(tables=tuple(TableSpec(id=d["id"], num_rows=d["num_rows"], dim=d["dim"],
                                            avg_pooling=d["avg_pooling"],
                                            value_precision=Precision(d["value_precision"]))
                                  for d in meta["tables"]), local_batch=meta["local_batch"])


def test_plan_json_roundtrip_and_validate(steps_golden):
    _, plans = steps_golden
    for c, meta in plans.items():
        plan = P.plan_from_json(json.dumps(meta["plan"]))
        P.validate_plan(plan, _model(meta))
        again = P.plan_from_json(P.plan_to_json(plan))
        assert again == plan


def test_pooled_a2a_bytes_match_reference_contract(steps_golden):
    _, plans = steps_golden
    for c, meta in plans.items():
        model = _model(meta)
        plan = P.plan_from_json(json.dumps(meta["plan"]))
        lay = P.rank_layout(model, plan)
        W, B = plan.num_workers, model.local_batch
        for v in range(W):
            twcw = sum(s.dim for s in lay.owned[v] if s.kind != "row_wise")
            assert twcw * (W * B - B) * 4 == meta["vol_fwd"][v], (c, v)


def test_validate_rejects_bad_plans():
    model = ModelSpec(tables=(TableSpec("a", 10, 4, 1.0),))
    bad = P.ShardingPlan(2, 2, (P.TableAssignment("a", P.Scheme(P.SchemeKind.ROW_WISE, 2),
                                                  (P.Shard(0, rows=(0, 4)), P.Shard(1, rows=(5, 10)))),))
    with pytest.raises(InvalidScheme):
        P.validate_plan(bad, model)
    with pytest.raises(InvalidScheme):
        P.validate_plan(P.ShardingPlan(2, 2, ()), model)


def test_even_bounds():
    assert P.even_bounds(10, 3) == [(0, 4), (4, 7), (7, 10)]


def _gloo_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2104_05158_b200.dist import LocalComm, NcclComm

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = NcclComm()
    # uneven splits: rank w sends (w + v + 1) elements to v, valued 100*w + v
    ins = torch.cat([torch.full((rank + v + 1,), 100 * rank + v, dtype=torch.int64) for v in range(world)])
    in_splits = [rank + v + 1 for v in range(world)]
    out_splits = [w + rank + 1 for w in range(world)]
    out = torch.empty(sum(out_splits), dtype=torch.int64)
    comm.all_to_all([out], [ins], [out_splits], [in_splits])
    t = torch.full((3,), float(rank + 1))
    comm.all_reduce_sum([t])
    q.put((rank, out.tolist(), t.tolist()))
    dist.destroy_process_group()


def test_comm_split_semantics_gloo_world2():
    """NcclComm (over gloo on CPU) and LocalComm implement the same
    all-to-all split convention and all-reduce."""
    import multiprocessing as mp

    import torch
    from paper_2104_05158_b200.dist import LocalComm

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 2000)
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r, (o, t)) for r, o, t in (q.get(timeout=120) for _ in procs))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    W = 2
    lc = LocalComm(W)
    ins = [torch.cat([torch.full((w + v + 1,), 100 * w + v, dtype=torch.int64) for v in range(W)]) for w in range(W)]
    outs = [torch.empty(sum(w + v + 1 for w in range(W)), dtype=torch.int64) for v in range(W)]
    lc.all_to_all(outs, ins, [[w + v + 1 for w in range(W)] for v in range(W)],
                  [[w + v + 1 for v in range(W)] for w in range(W)])
    for v in range(W):
        assert res[v][0] == outs[v].tolist()
        assert res[v][1] == [3.0, 3.0, 3.0]
