"""Table checkpoints (NEOT, embedding.py:334-377).

CPU: the oracle's reader/writer reproduces the files the REFERENCE's
dump_table wrote (tests/golden/neot, made by make_golden.py) byte for byte.
GPU: dump from / load into HBM tables through paper_2104_05158_b200.checkpoint:
bitwise equal to the reference's files (f64 tables), RNE-narrowed on load
(f32/f16), resume reproduces an uninterrupted run, malformed records raise
the reference's error types."""
import io
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import tbe_oracle as O  # noqa: E402

GOLD = ROOT / "tests" / "golden" / "neot"
CASES = {"rowwise": (37, 8, 0, 1), "elementwise": (21, 5, 0, 2), "nomoment": (16, 12, 1, 0)}


def _read(name):
    with open(GOLD / f"{name}.bin", "rb") as fh:
        return O.neot_read(fh)


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_neot_matches_reference_files(name):
    H, D, prec, mcode = CASES[name]
    values, moment, p = _read(name)
    assert values.shape == (H, D) and p == prec
    assert (moment is None) == (mcode == 0)
    buf = io.BytesIO()
    O.neot_write(buf, values, moment, prec)
    assert buf.getvalue() == (GOLD / f"{name}.bin").read_bytes()


gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def ck():
    import paper_2104_05158_b200 as p

    assert torch.cuda.is_available()
    p.load()
    return p.checkpoint


def _dev(a, dtype):
    return None if a is None else torch.from_numpy(np.asarray(a, dtype=np.float64)).cuda().to(dtype)


@gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_load_then_dump_f64_is_bitwise(ck, name):
    values, moment, prec = _read(name)
    w = torch.empty(values.shape, dtype=torch.float64, device="cuda")
    m = None if moment is None else torch.empty(moment.shape, dtype=torch.float64, device="cuda")
    with open(GOLD / f"{name}.bin", "rb") as fh:
        assert ck.load_tensor(fh, w, m, chunk_bytes=64) == prec  # tiny chunks: exercise the staging ring
    assert np.array_equal(w.cpu().numpy(), values)
    if m is not None:
        assert np.array_equal(m.cpu().numpy(), moment)
    buf = io.BytesIO()
    ck.dump_tensor(buf, w, m, precision=prec, chunk_bytes=72)
    assert buf.getvalue() == (GOLD / f"{name}.bin").read_bytes()


@gpu
@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
def test_load_narrows_rne_and_dump_widens_exactly(ck, dtype):
    values, moment, _ = _read("rowwise")
    w = torch.empty(values.shape, dtype=dtype, device="cuda")
    m = torch.empty(moment.shape, dtype=torch.float32, device="cuda")
    with open(GOLD / "rowwise.bin", "rb") as fh:
        ck.load_tensor(fh, w, m, chunk_bytes=40)
    npd = np.float32 if dtype == torch.float32 else np.float16
    assert np.array_equal(w.cpu().numpy(), values.astype(npd))
    assert np.array_equal(m.cpu().numpy(), moment.astype(np.float32))
    buf = io.BytesIO()
    ck.dump_tensor(buf, w, m)
    buf.seek(0)
    v2, m2, p2 = O.neot_read(buf)
    assert p2 == (1 if dtype == torch.float16 else 0)
    assert np.array_equal(v2, values.astype(npd).astype(np.float64))
    assert np.array_equal(m2, moment.astype(np.float32).astype(np.float64))


@gpu
def test_malformed_records_raise(ck):
    from paper_2104_05158_b200.errors import InvalidValue, MalformedDocument

    raw = (GOLD / "rowwise.bin").read_bytes()
    w = torch.empty((37, 8), dtype=torch.float64, device="cuda")
    m = torch.empty(37, dtype=torch.float64, device="cuda")
    with pytest.raises(MalformedDocument):
        ck.load_tensor(io.BytesIO(b"XEOT" + raw[4:]), w, m)
    with pytest.raises(MalformedDocument):
        ck.load_tensor(io.BytesIO(raw[:-8]), w, m)
    with pytest.raises(InvalidValue):
        ck.load_tensor(io.BytesIO(raw), torch.empty((36, 8), dtype=torch.float64, device="cuda"), m)
    with pytest.raises(InvalidValue):  # record has a row-wise moment, table has none
        ck.load_tensor(io.BytesIO(raw), w, None)


@gpu
def test_group_resume_matches_uninterrupted_run(ck, tmp_path):
    from paper_2104_05158_b200 import tbe

    rng = np.random.default_rng(3)
    rows, dims, B = [300, 50, 1000], [64, 13, 128], 64

    def batch():
        lens = rng.integers(0, 9, size=len(rows) * B)
        ids = np.concatenate([rng.integers(0, rows[t], size=int(lens[t * B:(t + 1) * B].sum()))
                              for t in range(len(rows))])
        return (torch.from_numpy(ids.astype(np.int32)).cuda(),
                tbe.lengths_to_offsets(torch.from_numpy(lens).cuda()))

    init = [rng.standard_normal((r, d)).astype(np.float32) for r, d in zip(rows, dims)]

    def group():
        g = tbe.TableGroup(rows, dims, torch.float32, "rowwise_adagrad", "cuda", table_ids=["a", "b", "c"])
        for w, x in zip(g.weights, init):
            w.copy_(torch.from_numpy(x))
        return g

    def step(g, ids, off):
        out = g.forward(ids, off, B)
        g.backward(ids, off, B, torch.ones_like(out), mode="update", optim="rowwise_adagrad", lr=0.05, eps=1e-8)

    b1, b2 = batch(), batch()
    a = group()
    step(a, *b1)
    ck.dump_group(a, tmp_path)
    step(a, *b2)
    r = group()
    for w in r.weights:
        w.zero_()
    ck.load_group(r, tmp_path)
    step(r, *b2)
    torch.cuda.synchronize()
    for x, y in zip(a.weights + a.moments, r.weights + r.moments):
        assert torch.equal(x, y)
    assert sorted(p.name for p in tmp_path.iterdir()) == ["a.bin", "b.bin", "c.bin"]


@gpu
def test_sharded_dump_load_roundtrip(ck, tmp_path, steps_golden):
    import json

    import paper_2104_05158_b200 as pkg
    from paper_2104_05158_b200 import dist
    from paper_2104_05158_b200.comms import _local_batches

    z, plans = steps_golden
    c, meta = next((c, m) for c, m in plans.items() if m["plan"]["num_workers"] > 1)
    tables = [pkg.TableSpec(id=d["id"], num_rows=d["num_rows"], dim=d["dim"], avg_pooling=d["avg_pooling"])
              for d in meta["tables"]]
    model = pkg.ModelSpec(tables=tuple(tables), local_batch=meta["local_batch"])
    plan = pkg.plan_from_json(json.dumps(meta["plan"]))
    W, B = plan.num_workers, meta["local_batch"]
    batch = pkg.CombinedBatch(z[f"s{c}_lengths"], z[f"s{c}_indices"])
    rng = np.random.default_rng(0)
    full = [rng.standard_normal((t.num_rows, t.dim)) for t in tables]

    def engine():
        return dist.ShardedEmbedding(model, plan, dist.LocalComm(W), B, dtype=torch.float64,
                                     optim="rowwise_adagrad",
                                     init=lambda t, r, cc: torch.from_numpy(full[t][r[0]:r[1], cc[0]:cc[1]].copy()))

    e1 = engine()
    e1.step(_local_batches(batch, W), lr=0.05, eps=1e-8)
    ck.dump_sharded(e1, tmp_path)
    e2 = engine()
    ck.load_sharded(e2, tmp_path)
    for slot in range(W):
        for (s1, w1, m1), (s2, w2, m2) in zip(e1.shard_tensors(slot), e2.shard_tensors(slot)):
            assert s1 == s2 and torch.equal(w1, w2) and (m1 is None or torch.equal(m1, m2))
    o1 = torch.cat([p.clone() for p in e1.step(_local_batches(batch, W), lr=0.05, eps=1e-8)])
    o2 = torch.cat([p.clone() for p in e2.step(_local_batches(batch, W), lr=0.05, eps=1e-8)])
    assert torch.equal(o1, o2)
