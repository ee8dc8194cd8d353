"""Place the benchmark models with the REFERENCE planner (run where
/root/reference exists):  python configs/make_plans.py
Writes configs/plans/<workload>_w<W>.json (the reference's plan_to_json
document).  The build consumes these plans unchanged (plan.plan_from_json)."""
import json
import sys
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


def main():
    OUT.mkdir(exist_ok=True)
    flags = planner.CompressionFlags(rowwise_optimizer=True)
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
