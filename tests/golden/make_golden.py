"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/ops.npz (small op-level cases), tests/golden/steps.npz
(small train-step / sharded-step cases with their plans) and
tests/golden/c1_digest.json (sha256 of the reference's config-1 step
outputs/tables).  The GPU box never reads /root/reference; tests use only
these committed files.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REF.parent / "tests"))
sys.dont_write_bytecode = True

import neosim  # noqa: E402
from neosim import comms, embedding, planner  # noqa: E402
from neosim.model import GlobalBatchLayout, LayoutTag  # noqa: E402

OUT = Path(__file__).resolve().parent


def desk_model(tables, local_batch=4):
    return neosim.ModelSpec(tables=tuple(tables), bottom_mlp_layers=(), top_mlp_layers=(),
                            local_batch=local_batch, mflops_per_sample=1.0,
                            interaction_flops_per_sample=0.0, dense_param_bytes=0)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def op_cases() -> dict:
    rng = np.random.default_rng(20260418)
    z = {}
    # forward / backward / optimizer cases over odd and vector-friendly dims
    dims = [1, 2, 3, 5, 8, 13, 64, 100, 128, 200, 256]
    for i, D in enumerate(dims):
        H = int(rng.integers(4, 120))
        n = int(rng.integers(1, 40))
        lengths = rng.integers(0, 70, size=n)
        lengths[rng.random(n) < 0.2] = 0  # empty bags
        idx = rng.integers(0, H, size=int(lengths.sum()))
        if len(idx) > 4:  # force duplicates inside bags
            idx[1::3] = idx[0]
        values = rng.standard_normal((H, D)) * 10.0 ** rng.uniform(-3, 3, size=(H, 1))
        spec = neosim.TableSpec(id=f"f{i}", num_rows=H, dim=D, avg_pooling=1.0)
        table = embedding.EmbeddingTable(spec, values.copy())
        z[f"fwd{i}_values"] = values
        z[f"fwd{i}_lengths"] = lengths
        z[f"fwd{i}_indices"] = idx
        z[f"fwd{i}_out"] = embedding.forward_pooled(table, lengths, idx)
        upstream = rng.standard_normal((n, D))
        g = embedding.backward_sort_aggregate(lengths, idx, upstream)
        z[f"bwd{i}_upstream"] = upstream
        z[f"bwd{i}_ids"] = g.ids
        z[f"bwd{i}_grads"] = g.grads
        for kind in ("sgd", "rowwise_adagrad", "adagrad"):
            cfg = embedding.OptimizerConfig(embedding.OptimizerKind(kind), lr=0.05, eps=1e-8)
            if kind == "rowwise_adagrad":
                m0 = np.abs(rng.standard_normal(H))
            elif kind == "adagrad":
                m0 = np.abs(rng.standard_normal((H, D)))
            else:
                m0 = None
            t = embedding.EmbeddingTable(spec, values.copy(), None if m0 is None else m0.copy())
            embedding.fused_backward_update(t, lengths, idx, upstream, cfg)
            z[f"upd{i}_{kind}_m0"] = np.zeros(0) if m0 is None else m0
            z[f"upd{i}_{kind}_values"] = t.values
            z[f"upd{i}_{kind}_moment"] = np.zeros(0) if t.moment is None else t.moment
    z["ndims"] = np.array(len(dims))
    # fp16 round trip
    x = np.concatenate([rng.standard_normal(500) * 10.0 ** rng.uniform(-8, 5, 500),
                        [2049.0, 1e6, -1e6, 65504.0, 65520.0, 6e-8, 0.0, -0.0]])
    q, ovf = embedding.quantize_fp16_roundtrip(x)
    z["fp16_x"], z["fp16_q"], z["fp16_ovf"] = x, q, ovf
    # bucketize
    for i in range(8):
        H = int(rng.integers(2, 5000))
        k = int(rng.integers(1, min(H, 9) + 1))
        bounds = planner.even_bounds(H, k)
        n = int(rng.integers(1, 50))
        lengths = rng.integers(0, 40, size=n)
        idx = rng.integers(0, H, size=int(lengths.sum()))
        parts = comms.bucketize_rowwise(lengths, idx, bounds)
        z[f"bkt{i}_starts"] = np.array([b[0] for b in bounds] + [H])
        z[f"bkt{i}_lengths"] = lengths
        z[f"bkt{i}_indices"] = idx
        z[f"bkt{i}_out_lengths"] = np.stack([p[0] for p in parts])
        z[f"bkt{i}_out_indices"] = np.concatenate([p[1] for p in parts])
    # block permute (WTB -> TWB)
    for i in range(6):
        W, T, B = (int(v) for v in rng.integers(1, 5, size=3))
        lengths = rng.integers(0, 5, size=W * T * B)
        idx = rng.integers(0, 1000, size=int(lengths.sum()))
        laid = comms.LaidOutBatch(GlobalBatchLayout(W, T, B, LayoutTag.WTB), lengths, idx)
        out = comms.permute_WTB_to_TWB(laid)
        z[f"perm{i}_wtb"] = np.array([W, T, B])
        z[f"perm{i}_lengths"] = lengths
        z[f"perm{i}_indices"] = idx
        z[f"perm{i}_out_lengths"] = out.lengths
        z[f"perm{i}_out_indices"] = out.indices
    return z


def random_plan(rng, model, workers, gpn):
    from test_acceptance import _random_plan

    return _random_plan(rng, model, workers, gpn)


def step_cases() -> tuple[dict, dict]:
    """train_step_reference / train_step_sharded on small random models."""
    rng = np.random.default_rng(2024)
    z, plans = {}, {}
    kinds = ["sgd", "rowwise_adagrad", "adagrad"]
    for c in range(24):
        T = int(rng.integers(1, 7))
        tables = [neosim.TableSpec(id=f"t{i}", num_rows=int(rng.integers(8, 200)),
                                   dim=int(rng.integers(1, 5)) * 2, avg_pooling=float(rng.uniform(1, 6)),
                                   value_precision=neosim.Precision.FP16 if rng.random() < 0.2
                                   else neosim.Precision.FP32)
                  for i in range(T)]
        model = desk_model(tables, local_batch=int(rng.integers(1, 9)))
        W = int(rng.choice([1, 2, 4]))
        gpn = 2 if W == 4 and c % 2 else W
        plan = random_plan(rng, model, W, gpn)
        kind = kinds[c % 3]
        cfg = embedding.OptimizerConfig(embedding.OptimizerKind(kind), lr=0.1, eps=1e-8)
        seed = int(rng.integers(10_000))
        batch = neosim.gen_synthetic_batch(model, W * model.local_batch, seed)
        ref_out, ref_tables = embedding.train_step_reference(model, batch, cfg, seed=seed)
        sh_out, state = comms.train_step_sharded(model, plan, batch, cfg, seed=seed)
        vals = comms.reassemble_values(model, plan, state)
        z[f"s{c}_lengths"] = batch.lengths
        z[f"s{c}_indices"] = batch.indices
        z[f"s{c}_ref_out"] = ref_out
        z[f"s{c}_sh_out"] = sh_out
        for t in range(T):
            z[f"s{c}_ref_t{t}"] = ref_tables[t].values
            z[f"s{c}_sh_t{t}"] = vals[t]
            if ref_tables[t].moment is not None:
                z[f"s{c}_ref_m{t}"] = ref_tables[t].moment
        plans[str(c)] = {
            "tables": [dict(id=t.id, num_rows=t.num_rows, dim=t.dim, avg_pooling=t.avg_pooling,
                            value_precision=t.value_precision.value) for t in tables],
            "local_batch": model.local_batch, "kind": kind, "lr": 0.1, "eps": 1e-8, "seed": seed,
            "plan": json.loads(planner.plan_to_json(plan)),
            # byte contract of every collective on the path (comms.py:366-518)
            "vol_fwd": list(comms.volume_forward_alltoall(plan, model, W).per_worker_send_bytes),
            "vol_input": list(comms.volume_input_alltoall(plan, model, W).per_worker_send_bytes),
        }
        # redistribution (comms.py:292-353): per worker, per shard input
        slices = comms.alltoall_redistribute(comms.to_wtb(batch, W), plan, model)
        red = []
        for ws in slices:
            for si in ws.inputs:
                shard = si.shard
                red.append(dict(worker=ws.worker, table_id=si.table_id, shard_worker=shard.worker,
                                rows=list(shard.rows) if shard.rows else None,
                                cols=list(shard.cols) if shard.cols else None,
                                sample_base=si.sample_base, lengths_sha=sha(si.lengths),
                                indices_sha=sha(si.indices)))
        plans[str(c)]["redistribute"] = red
    return z, plans


def c1_digest() -> dict:
    """Config 1 (8 x 100k x 64, B=2048, L=20, row-wise AdaGrad): digests of
    the reference step, for a bitwise check of the f64 GPU path."""
    tables = [neosim.TableSpec(id=f"t{i}", num_rows=100_000, dim=64, avg_pooling=20.0) for i in range(8)]
    model = desk_model(tables, local_batch=2048)
    cfg = embedding.OptimizerConfig(embedding.OptimizerKind.ROWWISE_ADAGRAD, lr=0.05, eps=1e-8)
    batch = neosim.gen_synthetic_batch(model, 2048, seed=0)
    out, tabs = embedding.train_step_reference(model, batch, cfg, seed=0)
    return {"batch_indices": sha(batch.indices), "batch_lengths": sha(batch.lengths),
            "out": sha(out), "values": [sha(t.values) for t in tabs],
            "moment": [sha(t.moment) for t in tabs],
            "out_sum": float(out.sum()), "value_sums": [float(t.values.sum()) for t in tabs]}


def neot_cases() -> None:
    """Table checkpoints written by the reference's dump_table
    (embedding.py:341-360): one per moment kind, one FP16-precision spec."""
    rng = np.random.default_rng(7)
    d = OUT / "neot"
    d.mkdir(exist_ok=True)
    cases = [("rowwise", 37, 8, neosim.Precision.FP32, "rowwise"),
             ("elementwise", 21, 5, neosim.Precision.FP32, "elementwise"),
             ("nomoment", 16, 12, neosim.Precision.FP16, None)]
    for name, H, D, prec, kind in cases:
        spec = neosim.TableSpec(id=name, num_rows=H, dim=D, avg_pooling=1.0, value_precision=prec)
        values = rng.standard_normal((H, D))
        moment = None if kind is None else np.abs(rng.standard_normal(H if kind == "rowwise" else (H, D)))
        with open(d / f"{name}.bin", "wb") as fh:
            embedding.dump_table(embedding.EmbeddingTable(spec, values, moment), fh)


def main(parts=("ops", "steps", "c1", "neot")):
    if "ops" in parts:
        np.savez_compressed(OUT / "ops.npz", **op_cases())
    if "steps" in parts:
        z, plans = step_cases()
        np.savez_compressed(OUT / "steps.npz", **z)
        (OUT / "steps_plans.json").write_text(json.dumps(plans, indent=1, sort_keys=True))
    if "c1" in parts:
        (OUT / "c1_digest.json").write_text(json.dumps(c1_digest(), indent=1))
    if "neot" in parts:
        neot_cases()
    for p in sorted(OUT.glob("*")):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("ops", "steps", "c1", "neot"))
