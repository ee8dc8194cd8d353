"""Place the benchmark models with the REFERENCE planner (run where
/root/reference exists):  python configs/make_plans.py
Writes configs/plans/<workload>_w<W>.json (the reference's plan_to_json
document).  The build consumes these plans unchanged (plan.plan_from_json)."""
import json
import sys

import numpy as np
from pathlib import Path

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

import neosim  # noqa: E402
from neosim import planner  # noqa: E402

OUT = Path(__file__).resolve().parent / "plans"


def b200_node(workers: int) -> neosim.ClusterSpec:
    """One B200 box: 180 GB HBM3e at the measured 6,544 GB/s copy bandwidth,
    NVLink 5 at 900 GB/s per direction, 400 Gb/s scale-out NIC."""
    return neosim.ClusterSpec(
        num_nodes=1, gpus_per_node=workers, hbm_capacity_per_gpu=183_359 * 2**20, hbm_bw=6544e9,
        dram_capacity_per_node=2 * 2**40, dram_to_gpu_bw=55e9, scaleup_bw=900e9, scaleout_bw_per_gpu=50e9,
        peak_flops={"FP32": 80e12, "TF32": 1.1e15, "FP16": 2.25e15, "BF16": 2.25e15}, mlp_efficiency=0.7,
        alltoall_bw_points=((1 << 20, 5e9), (1 << 26, 30e9), (1 << 28, 45e9)),
        allreduce_bw_points=((1 << 23, 100e9), (1 << 28, 400e9), (1 << 32, 700e9)),
        fixed_latency_per_collective=1e-5)


def model(T, H, D, L, B):
    tabs = tuple(neosim.TableSpec(id=f"t{i}", num_rows=H, dim=D, avg_pooling=float(L)) for i in range(T))
    return neosim.ModelSpec(tables=tabs, bottom_mlp_layers=(), top_mlp_layers=(), local_batch=B,
                            mflops_per_sample=1.0, interaction_flops_per_sample=0.0, dense_param_bytes=0)


def rw_plan(m, W: int) -> neosim.ShardingPlan:
    """Config 4: every giant table row-wise over all W GPUs (even_bounds)."""
    A = [planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.ROW_WISE, num_row_shards=W),
                                 tuple(planner.Shard(worker=i, rows=b)
                                       for i, b in enumerate(planner.even_bounds(t.num_rows, W))))
         for t in m.tables]
    return planner.ShardingPlan(W, W, tuple(A))


def cw_plan(m, W: int) -> neosim.ShardingPlan:
    """Config 4, column-wise variant: each table in two column halves on two
    GPUs (table t's halves on workers 2t mod W, 2t+1 mod W)."""
    A = []
    for i, t in enumerate(m.tables):
        splits = ((0, t.dim // 2), (t.dim // 2, t.dim))
        A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.COLUMN_WISE, col_splits=splits),
                                         tuple(planner.Shard(worker=(2 * i + k) % W, cols=c)
                                               for k, c in enumerate(splits))))
    return planner.ShardingPlan(W, W, tuple(A))


def c5_model(max_rows: float, seed: int = 5):
    """Config 5: 512 tables, rows log-uniform in [1e3, max_rows], dims cycled
    {32, 64, 128, 256}, pooling uniform in [1, 64], Zipf(1.05) indices."""
    rng = np.random.default_rng(seed)
    dims = (32, 64, 128, 256)
    tabs = tuple(neosim.TableSpec(id=f"t{i}", num_rows=int(round(10 ** rng.uniform(3, np.log10(max_rows)))),
                                  dim=dims[i % 4], avg_pooling=float(rng.uniform(1, 64)),
                                  index_skew=neosim.IndexSkew(neosim.SkewKind.ZIPF, 1.05))
                 for i in range(512))
    return neosim.ModelSpec(tables=tabs, bottom_mlp_layers=(), top_mlp_layers=(), local_batch=8192,
                            mflops_per_sample=1.0, interaction_flops_per_sample=0.0, dense_param_bytes=0)


def mixed_plan(m, W: int, seed: int) -> neosim.ShardingPlan:
    """Config 5: a seeded TW / RW / CW / DP mix in the style of the
    reference's acceptance suite (test_acceptance.py:134-199); DP only for
    tables under 1e5 rows, RW for the largest."""
    rng = np.random.default_rng(seed)
    A = []
    for t in m.tables:
        c = int(rng.integers(0, 4))
        if t.num_rows > 2_000_000 and W >= 2:
            k = int(rng.integers(2, W + 1))
            start = int(rng.integers(0, W))
            A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.ROW_WISE, num_row_shards=k),
                                             tuple(planner.Shard(worker=(start + i) % W, rows=b)
                                                   for i, b in enumerate(planner.even_bounds(t.num_rows, k)))))
        elif c == 3 and t.num_rows < 100_000:
            A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.DATA_PARALLEL),
                                             (planner.Shard(worker=None),)))
        elif c == 2 and W >= 2:
            splits = ((0, t.dim // 2), (t.dim // 2, t.dim))
            start = int(rng.integers(0, W))
            A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.COLUMN_WISE,
                                                                  col_splits=splits),
                                             tuple(planner.Shard(worker=(start + i) % W, cols=s)
                                                   for i, s in enumerate(splits))))
        elif c == 1 and W >= 2:
            k = int(rng.integers(2, W + 1))
            start = int(rng.integers(0, W))
            A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.ROW_WISE, num_row_shards=k),
                                             tuple(planner.Shard(worker=(start + i) % W, rows=b)
                                                   for i, b in enumerate(planner.even_bounds(t.num_rows, k)))))
        else:
            A.append(planner.TableAssignment(t.id, planner.Scheme(planner.SchemeKind.TABLE_WISE),
                                             (planner.Shard(worker=int(rng.integers(0, W))),)))
    return planner.ShardingPlan(W, W, tuple(A))


def write(name: str, plan, m=None, W=None, flags=None) -> None:
    text = planner.plan_to_json(plan, m, b200_node(W), flags) if m is not None else planner.plan_to_json(plan)
    planner.validate_plan(plan, m) if m is not None else None
    (OUT / f"{name}.json").write_text(text)
    kinds = sorted({a.scheme.kind.value for a in plan.assignments})
    per = [sum(1 for a in plan.assignments for s in a.shards if s.worker == w) for w in range(plan.num_workers)]
    print(f"{name}: schemes {kinds}, shards per worker {per}")


def main():
    OUT.mkdir(exist_ok=True)
    (OUT.parent / "models").mkdir(exist_ok=True)
    flags = planner.CompressionFlags(rowwise_optimizer=True)
    for W in (2, 4, 8):
        # config 3: 256 x 2M x 128, 65,536 samples global, placed by the reference planner
        m3 = model(256, 2_000_000, 128, 32, 65536 // W)
        write(f"c3_w{W}", planner.plan_4d(m3, b200_node(W), planner.CostWeights(),
                                          planner.CandidatePolicy(flags=flags), "kk"), m3, W, flags)
        # config 4: 4 x 100M x 256, explicit row-wise (and a column-wise variant)
        m4 = model(4, 100_000_000, 256, 32, 65536 // W)
        write(f"c4_rw_w{W}", rw_plan(m4, W))
        write(f"c4_cw_w{W}", cw_plan(m4, W))
        # config 5 (full size) and its row-scaled single-GPU test variant
        for tag, mx in (("c5", 1e7), ("c5s", 1e5)):
            m5 = c5_model(mx)
            write(f"{tag}_w{W}", mixed_plan(m5, W, seed=100 + W))
    for tag, mx in (("c5", 1e7), ("c5s", 1e5)):
        (OUT.parent / "models" / f"{tag}.json").write_text(neosim.serialize_model_spec(c5_model(mx)))
    for W in (1, 2, 4, 8):
        # bench workload: config-2 tables, 65,536 samples per GPU (weak scaling)
        m = model(64, 1_000_000, 128, 32, 65536)
        p = planner.plan_4d(m, b200_node(W), planner.CostWeights(), planner.CandidatePolicy(flags=flags), "kk")
        (OUT / f"c2_w{W}.json").write_text(planner.plan_to_json(p, m, b200_node(W), flags))
        kinds = sorted({a.scheme.kind.value for a in p.assignments})
        per = [sum(1 for a in p.assignments for s in a.shards if s.worker == w) for w in range(W)]
        print(f"c2 W={W}: schemes {kinds}, shards per worker {per}")


if __name__ == "__main__":
    main()
