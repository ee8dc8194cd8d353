#!/usr/bin/env python
"""Benchmark: embedding-training samples/s of the fused TBE step on B200.

N=1 workload = BASELINE config 2 (the metric's HBM-roofline bench): 64
tables x 1,000,000 rows x dim 128 fp32, batch 65,536, pooling 32, row-wise
AdaGrad (lr 0.05, eps 1e-8), upstream gradient = ones (the reference's
sum-of-outputs loss, embedding.py:326).  A step = one fused TBE forward over
all tables + one fused backward/row-wise-AdaGrad over all tables.

N>1 (torchrun, one rank per GPU, NCCL): the sharded embedding step with the
same per-GPU work (weak scaling): the 64 tables are placed table-wise by the
reference planner's plan (configs/plans), global batch 65,536 x N, and
pooled rows / their gradients move through the all-to-all.

--impl reference times the reference's CPU implementation of the same step
(the oracle's port of the numpy code) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "embedding-training samples/sec"
UNIT = "samples/s"
LR, EPS = 0.05, 1e-8
FALLBACK_HBM_GBS = 6650.0


def parse_args(argv=None):
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["b200", "reference"], default="b200")
    p.add_argument("--tables", type=int, default=64)
    p.add_argument("--rows", type=int, default=1_000_000)
    p.add_argument("--dim", type=int, default=128)
    p.add_argument("--batch", type=int, default=65536, help="per-GPU batch (global = batch x N)")
    p.add_argument("--pooling", type=int, default=32)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--workload", choices=["c2", "c3", "c4", "c5"], default="c2",
                   help="N>1 only: c2 = config 2 per GPU (weak scaling, default); c3/c4/c5 = the BASELINE "
                        "multi-GPU configs at global batch 65,536")
    p.add_argument("--transport", choices=["nccl", "nvlink"], default="nvlink",
                   help="N>1 pooled exchange: NCCL all_to_all, or stores into peers' symmetric buffers")
    p.add_argument("--no-subgroups", action="store_true",
                   help="diagnostic: one backward call over all tables (no shorter sort keys)")
    p.add_argument("--upstream-broadcast", action="store_true",
                   help="diagnostic: one upstream row for every bag (stride 0); not a valid bench number")
    p.add_argument("--overlap-sort", type=int, default=-1,
                   help="N=1: issue the backward's key build + sort on a side stream under the forward, with the "
                        "forward capped at this many CTAs per SM (0 = uncapped; -1 = off)")
    p.add_argument("--no-cache-bench", action="store_true", help="skip the software row-cache replay line")
    p.add_argument("--cpu-sample-batch", type=int, default=0,
                   help="samples per step of the sampled CPU reference step (default 4096 of the batch)")
    return p.parse_args(argv)


def workload_name(a) -> str:
    return (f"c2: {a.tables} tables x {a.rows:,} rows x dim {a.dim} fp32, batch {a.batch:,}/GPU, "
            f"pooling {a.pooling}, row-wise AdaGrad")


def ncu_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu capture
    (profiles/r2_traffic.json), or None."""
    f = ROOT / "profiles" / "r2_traffic.json"
    if kernel is None or not f.exists():
        return None
    try:
        d = json.loads(f.read_text())[kernel]
        return float(d["dram_read_bytes"] + d["dram_write_bytes"])
    except Exception:
        return None


def hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    if f.exists():
        try:
            return float(json.loads(f.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


# ---------------------------------------------------------------------------
# clocks during the timed region


class Clocks:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.proc = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-i", str(index), "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out = ""
        sm, smax, reasons = [], [], set()
        for line in out.splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        busy = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# algorithmic bytes (SURVEY.md section 8d / DESIGN.md)


def fwd_bytes(T, N, D, B, e=4, i=4, o=8):
    """Compulsory bytes of one TBE forward: every lookup reads a row, ids,
    offsets, pooled write."""
    return T * (N * D * e + N * i + (B + 1) * o + B * D * 4)


def bwd_bytes(U_list, N, D, B, e=4, i=4, o=8):
    """Compulsory bytes of the fused backward + row-wise AdaGrad: upstream
    read, ids, offsets, read+write of every touched row and its moment."""
    return sum(B * D * 4 + N * i + (B + 1) * o + U * (2 * D * e + 2 * 4) for U in U_list)


# ---------------------------------------------------------------------------
# CPU legs: the reference's own numpy implementation — checker / baseline only
#
# One CPU "step" is a BOUNDED SAMPLE of the config-2 step: all 64 tables x
# `n` samples (L ids each), forward_pooled + fused_backward_update with
# row-wise AdaGrad and the reference's ones upstream, timed end to end.  The
# tables are spread over worker processes (one table-parallel process per
# host core, memory permitting); the step time is the wall time until every
# worker is done, so value = n / step time is measured, never extrapolated.
# The reference itself is sequential (cli.py:549): its one-core rate is n /
# (sum of the measured per-table times).  When oracle/_ref (a copy of the
# reference package) is present the REAL neosim functions run ("reference");
# otherwise the oracle's port of the same numpy primitives ("port").

REF_DIR = ROOT / "oracle" / "_ref"


def _ref_worker(conn, table_ids, H, D, L, seed):
    """Worker process: holds its tables, runs sampled steps on request."""
    use_ref = (REF_DIR / "neosim").is_dir()
    if use_ref:
        sys.path.insert(0, str(REF_DIR))
        from neosim import embedding as E
        from neosim import model as M

        specs = tuple(M.TableSpec(id=f"t{t}", num_rows=H, dim=D, avg_pooling=float(L)) for t in table_ids)
        model = M.ModelSpec(tables=specs, bottom_mlp_layers=(), top_mlp_layers=(), local_batch=1,
                            mflops_per_sample=1.0, interaction_flops_per_sample=0.0, dense_param_bytes=0)
        cfg = E.OptimizerConfig(E.OptimizerKind.ROWWISE_ADAGRAD, LR, EPS)
        tables = E.build_tables(model, cfg, seed=seed)
    else:
        from oracle import tbe_oracle as O

        rng0 = np.random.default_rng(seed)
        tables = [(rng0.standard_normal((H, D)), np.zeros(H)) for _ in table_ids]
    conn.send(("ready", "reference" if use_ref else "port"))
    while True:
        msg = conn.recv()
        if msg[0] == "stop":
            return
        _, step_seed, n = msg
        times = []
        if use_ref:
            batch = M.gen_synthetic_batch(model, n, seed=step_seed)
            ones = np.ones((n, D))
            for k, tab in enumerate(tables):
                lengths, idx = batch.table_slice(k)
                t0 = time.perf_counter()
                E.forward_pooled(tab, lengths, idx)
                E.fused_backward_update(tab, lengths, idx, ones, cfg)
                times.append(time.perf_counter() - t0)
        else:
            rng = np.random.default_rng(step_seed)
            lengths = np.full(n, L, dtype=np.int64)
            for values, moment in tables:
                idx = rng.integers(0, H, size=n * L, dtype=np.int64)
                t0 = time.perf_counter()
                O.np_forward_pooled(values, lengths, idx)
                ids, g = O.np_backward_sort_aggregate(lengths, idx, np.ones((n, D)))
                O.np_apply("rowwise_adagrad", values, moment, ids, g, LR, EPS)
                times.append(time.perf_counter() - t0)
        conn.send(("done", times))


class RefWorkers:
    """Table-parallel worker processes over the host cores."""

    def __init__(self, T, H, D, L, procs=None):
        import multiprocessing as mp

        per_table = H * D * 8 + H * 8
        try:
            import psutil

            avail = psutil.virtual_memory().available
        except Exception:
            avail = 16 << 30
        cores = os.cpu_count() or 1
        if procs is None:
            procs = max(1, min(cores, T, int(avail * 0.6 // (per_table * max(1, math.ceil(T / cores))))))
        self.procs = procs
        ctx = mp.get_context("spawn")
        self.conns, self.ps = [], []
        for w in range(procs):
            mine = list(range(w, T, procs))
            a, b = ctx.Pipe()
            proc = ctx.Process(target=_ref_worker, args=(b, mine, H, D, L, 1000 + w), daemon=True)
            proc.start()
            self.conns.append(a)
            self.ps.append(proc)
        kinds = {c.recv()[1] for c in self.conns}
        self.kind = kinds.pop()

    def step(self, seed, n):
        """Wall time of one sampled step over all tables and the per-table times."""
        t0 = time.perf_counter()
        for w, c in enumerate(self.conns):
            c.send(("step", seed * 1000 + w, n))
        per = [t for c in self.conns for t in c.recv()[1]]
        return time.perf_counter() - t0, per

    def close(self):
        for c in self.conns:
            c.send(("stop",))
        for p in self.ps:
            p.join(timeout=30)


def cpu_sample(a) -> int:
    return a.cpu_sample_batch or 4096


def cpu_baseline(a, T_total) -> dict:
    """The reference's CPU step on a bounded sample (see above), 2 steps."""
    n = cpu_sample(a)
    wk = RefWorkers(T_total, a.rows, a.dim, a.pooling)
    wk.step(1, n)  # warm-up
    walls, per = [], []
    for k in range(2):
        w, pt = wk.step(2 + k, n)
        walls.append(w)
        per.append(sum(pt))
    wk.close()
    wall, one = float(np.mean(walls)), float(np.mean(per))
    return {"value": n / wall, "unit": UNIT, "cores": wk.procs, "kind": wk.kind,
            "sample": f"each step: all {T_total} tables x {n:,} of {a.batch:,} samples x {a.pooling} ids, "
                      f"forward_pooled + fused_backward_update (row-wise AdaGrad, ones upstream), "
                      f"{'neosim (oracle/_ref)' if wk.kind == 'reference' else 'oracle numpy port'}; "
                      f"tables spread over {wk.procs} processes; wall time of the sampled step (not scaled)",
            "ms_per_sample_step": 1e3 * wall, "one_core": {"value": n / one, "unit": UNIT, "cores": 1,
                                                           "ms_per_sample_step": 1e3 * one,
                                                           "how": "sum of the measured per-table times "
                                                                  "(the reference runs tables sequentially)"},
            "nproc": os.cpu_count()}


def run_reference(a, rank, world):
    """--impl reference: the reference's own CPU implementation of the step,
    every table, on a bounded sample of the batch per step (measured wall
    time per step, all host cores; rank 0 only)."""
    if rank != 0:
        return
    n = cpu_sample(a)
    wk = RefWorkers(a.tables, a.rows, a.dim, a.pooling)
    for k in range(a.warmup):
        wk.step(100 + k, n)
    walls, ones = [], []
    for k in range(a.steps):
        w, pt = wk.step(1000 + k, n)
        walls.append(w)
        ones.append(sum(pt))
    wk.close()
    ms = 1e3 * float(np.mean(walls))
    value = n / (ms / 1e3)
    sample = (f"each step: all {a.tables} tables x {n:,} of {a.batch:,} samples x {a.pooling} ids "
              f"(a bounded sample of the config-2 step), "
              f"{'neosim forward_pooled + fused_backward_update from oracle/_ref' if wk.kind == 'reference' else 'oracle numpy port'}"
              f", row-wise AdaGrad, ones upstream; tables spread over {wk.procs} processes; ms_per_step is the "
              f"measured wall time of that sampled step")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": workload_name(a), "tables": a.tables, "rows": a.rows, "dim": a.dim,
                       "batch_per_gpu": a.batch, "pooling": a.pooling, "cpu_sample_samples_per_step": n},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": wk.procs, "kind": wk.kind, "sample": sample,
                             "one_core": {"value": n / float(np.mean(ones)), "unit": UNIT, "cores": 1,
                                          "how": "sum of the measured per-table times"},
                             "nproc": os.cpu_count()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cache_replay_bench(dev, cpu: bool = True) -> dict:
    """the software row cache (cache.py:68-126).  A Zipf
    (alpha 1.05) trace of 64 M row accesses over 100 M rows replayed through a
    1 M-set x 32-way LRU cache (32 M resident rows, the HBM tier of config 4)
    on the GPU, inputs resident; CPU: the oracle's C port of the reference's
    sequential access() loop on a 4 M-access prefix, one core."""
    import torch

    from paper_2104_05158_b200 import cache

    n, sets, ways = 64 << 20, 1 << 20, 32
    g = torch.Generator(device=dev)
    g.manual_seed(11)
    u = torch.rand(n, generator=g, device=dev, dtype=torch.float64)
    # inverse-CDF Zipf-like ranks over 1e8 rows (continuous approximation, alpha 1.05)
    alpha, H = 1.05, 1e8
    tr = torch.clamp((1.0 - u * (1.0 - H ** (1.0 - alpha))) ** (1.0 / (1.0 - alpha)) - 1.0, 0, H - 1).to(torch.int64)
    cfg = cache.CacheConfig(num_sets=sets, ways=ways)
    for _ in range(2):
        _, _, st = cache.access_trace(cfg, tr, with_results=False, device=dev)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        _, _, st = cache.access_trace(cfg, tr, with_results=True, device=dev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = {"workload": f"{n:,} Zipf(1.05) accesses over 1e8 rows, {sets:,} sets x {ways} ways LRU, per-access "
                       "AccessResult written (hit, evicted)", "value": n / (ms * 1e-3), "unit": "accesses/s",
           "ms": ms, "hit_rate": st.hit_rate, "gpu_kernels": "cache_keys_kernel + CUB radix sort + select + "
                                                              "cache_replay_kernel (warp per set)"}
    if cpu:
        from oracle import tbe_oracle as O

        m = 4 << 20
        sample = tr[:m].cpu().numpy()
        t0 = time.perf_counter()
        O.cache_simulate_c(sets, ways, "lru", sample)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": m / dt, "unit": "accesses/s", "cores": 1, "kind": "port",
                               "sample": f"first {m:,} accesses, oracle C port of cache.py access() (sequential)"}
    return out


# ---------------------------------------------------------------------------
# B200 arm


def count_launches(step_fn) -> int:
    """Kernels launched by one step, from a CUPTI trace of an untimed step."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step_fn()
        torch.cuda.synchronize()
    n = 0
    for ev in prof.events():
        if getattr(ev, "device_type", None) is not None and "CUDA" in str(ev.device_type):
            name = ev.name
            if "Memcpy" in name or "Memset" in name:
                continue
            n += 1
    return n


def run_b200(a, rank, world):
    import torch

    from paper_2104_05158_b200 import tbe
    import paper_2104_05158_b200 as neo

    neo.load()
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    if world > 1:
        return run_sharded(a, rank, world, dev)
    T, H, D, B, L = a.tables, a.rows, a.dim, a.batch, a.pooling
    N = B * L
    torch.manual_seed(0)
    grp = tbe.TableGroup([H] * T, [D] * T, dtype=torch.float32, optim="rowwise_adagrad", device=dev)
    grp._storage.normal_()
    offsets = torch.arange(0, T * B + 1, dtype=torch.int64, device=dev) * L
    batches = [torch.randint(0, H, (T * N,), dtype=torch.int32, device=dev) for _ in range(2)]
    out = torch.empty((B, T * D), dtype=torch.float32, device=dev)
    upstream = torch.ones((B, T * D), dtype=torch.float32, device=dev)
    if a.upstream_broadcast:
        upstream = torch.ones((1, T * D), dtype=torch.float32, device=dev).expand(B, T * D)
    U_list = [int(torch.unique(batches[0][t * N:(t + 1) * N]).numel()) for t in range(T)]

    counts = None if a.no_subgroups else [N] * T  # host-known per-table id counts (lengths are host data)

    overlap = a.overlap_sort >= 0 and counts is not None
    if overlap:
        tbe.set_forward_residency(a.overlap_sort)
        # the step runs on a high-priority stream: the block scheduler then
        # places the forward's CTAs first and the side-stream sort phase fills
        # the SM resources the capped forward leaves free
        torch.cuda.set_stream(torch.cuda.Stream(device=dev, priority=-1))

    def step(i):
        ix = batches[i % 2]
        if overlap:
            grp.prepare_backward(ix, offsets, B, upstream, counts, optim="rowwise_adagrad")
        grp.forward(ix, offsets, B, out=out)
        grp.backward(ix, offsets, B, upstream, mode="update", optim="rowwise_adagrad", lr=LR, eps=EPS,
                     table_counts=counts)

    # nvidia-smi starts before the warm-up: its start-up (NVML init) can stall
    # driver calls for tens of ms, which must not land inside the timed steps
    clocks = Clocks(dev.index)
    for i in range(a.warmup):
        step(i)
    launches_per_step = count_launches(lambda: step(0))
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    time.sleep(0.3)
    torch.cuda.synchronize()
    timers = {}
    for i in range(a.steps):
        e0, e1, e2 = ev[i]
        e0.record()
        ix = batches[i % 2]
        if overlap:
            grp.prepare_backward(ix, offsets, B, upstream, counts, optim="rowwise_adagrad")
        grp.forward(ix, offsets, B, out=out)
        e1.record()
        grp.backward(ix, offsets, B, upstream, mode="update", optim="rowwise_adagrad", lr=LR, eps=EPS,
                     table_counts=counts, timers=timers)
        e2.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = ev[0][0].elapsed_time(ev[-1][2])
    fwd_ms = float(np.mean([e0.elapsed_time(e1) for e0, e1, _ in ev]))
    bwd_ms = float(np.mean([e1.elapsed_time(e2) for _, e1, e2 in ev]))
    ms = total_ms / a.steps
    peak, peak_kind = hbm_peak()
    fb, bb = fwd_bytes(T, N, D, B), bwd_bytes(U_list, N, D, B)
    fwd_gbs = fb / (fwd_ms * 1e-3) / 1e9
    bwd_gbs = bb / (bwd_ms * 1e-3) / 1e9
    step_gbs = (fb + bb) / (ms * 1e-3) / 1e9
    applies = timers.get("apply", [])
    if applies:  # streamed segment-walk + optimizer launches (one per sort group)
        ap_ms = float(np.mean([x.elapsed_time(y) for x, y, _, _ in applies]))
        ap_bytes = float(np.mean([bwd_bytes(U_list[t0:t1], N, D, B) for _, _, t0, t1 in applies]))
        dominant = ("bkt_rows_kernel (APPLY of the bucketed backward: warp-specialised TMA producer + sub-warp-per-row "
                    f"reduce + row-wise AdaGrad, one launch over {applies[0][3] - applies[0][2]} tables; "
                    "plus the hot-row kernel)",
                    ap_bytes / (ap_ms * 1e-3) / 1e9, ap_bytes, ap_ms)
    else:
        dominant = ("tbe_backward (keys+sort+segments+row-wise AdaGrad)", bwd_gbs, bb, bwd_ms)
    line = {
        "metric": METRIC, "value": B / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(a), "tables": T, "rows": H, "dim": D, "batch_per_gpu": B,
                   "backward_sort": (f"side stream under the forward (forward capped at {a.overlap_sort} CTAs/SM)"
                                     if overlap else "in the backward, serial"),
                   "pooling": L, "index_dtype": "int32", "optimizer": "rowwise_adagrad",
                   "l2": "inputs larger than L2 (32.8 GB of tables, 537 MB of ids per step, 2 alternating batches)"},
        "roofline": {"bound": "hbm", "kernel": dominant[0], "achieved": dominant[1], "peak": peak,
                     "peak_kind": peak_kind, "unit": "GB/s", "frac": dominant[1] / peak,
                     "traffic": ncu_traffic("bkt_rows_kernel" if applies else None),
                     "traffic_source": "profiles/r2_traffic.json (ncu --set full, one launch)",
                     "algorithmic_bytes": dominant[2], "ms": dominant[3]},
        "roofline_fwd": {"kernel": "tbe_forward_kernel", "achieved": fwd_gbs, "frac": fwd_gbs / peak, "ms": fwd_ms,
                         "algorithmic_bytes": fb, "traffic": ncu_traffic("tbe_forward_kernel"),
                         "note": "algorithmic bytes count every lookup's row read; L2 serves the repeated rows, "
                                 "so achieved can exceed the copy peak (ncu DRAM bytes: profiles/)"},
        "roofline_step": {"achieved": step_gbs, "frac": step_gbs / peak, "fwd_gbs": fwd_gbs, "bwd_gbs": bwd_gbs,
                          "fwd_ms": fwd_ms, "bwd_ms": bwd_ms, "bytes": fb + bb,
                          "unique_rows_per_table": float(np.mean(U_list))},
        "gpu_launches": launches_per_step * a.steps,
        "clocks": clk,
    }
    if not a.no_e2e:
        line["e2e"] = e2e_b200(a, grp, dev)
    if not a.no_cache_bench:
        line["cache_replay"] = cache_replay_bench(dev, cpu=not a.no_cpu_baseline)
    if not a.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(a, T)
    print(json.dumps(line), flush=True)


def e2e_b200(a, grp, dev) -> dict:
    """Same step through the public pipeline API with host (pinned) inputs:
    every step copies its ids/offsets H2D and reads the loss back D2H."""
    import torch

    from paper_2104_05158_b200.pipeline import TrainPipeline

    T, H, D, B, L = a.tables, a.rows, a.dim, a.batch, a.pooling
    N = B * L
    g = torch.Generator().manual_seed(1)
    host = [torch.randint(0, H, (T * N,), dtype=torch.int32, generator=g).pin_memory() for _ in range(2)]
    lengths = torch.full((T * B,), L, dtype=torch.int64).pin_memory()
    pipe = TrainPipeline(grp, batch=B, optim="rowwise_adagrad", lr=LR, eps=EPS)
    batches = [(lengths, host[i % 2]) for i in range(a.warmup + a.steps)]
    pipe.run(batches[:a.warmup])
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    losses = pipe.run(batches[a.warmup:])
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.steps
    assert len(losses) == a.steps
    return {"value": B / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": host[0].numel() * 4 + lengths.numel() * 8, "d2h_bytes_per_step": 8,
            "api": "paper_2104_05158_b200.pipeline.TrainPipeline.run (pinned host ids/lengths, "
                   "H2D prefetch overlapped with the previous step, loss = sum of pooled outputs read back)"}


def expected_unique(H: int, N: int) -> float:
    return H * (1.0 - (1.0 - 1.0 / H) ** N)


class ShardedWorkload:
    """One BASELINE config as a sharded step: model, plan, per-rank batch,
    wire / storage dtypes and the id distribution (device-generated)."""

    def __init__(self, a, world: int):
        import torch

        from paper_2104_05158_b200 import plan as P
        from paper_2104_05158_b200 import spec

        self.key = a.workload
        self.fwd_comm = self.bwd_comm = None
        self.dtype = torch.float32
        self.zipf = False
        L = a.pooling
        if a.workload == "c2":
            T, H, D, self.B = a.tables, a.rows, a.dim, a.batch
            plan_name, self.scaling = f"c2_w{world}", "weak"
            self.name = workload_name(a)
        elif a.workload == "c3":
            T, H, D, self.B = 256, 2_000_000, 128, 65536 // world
            plan_name, self.scaling = f"c3_w{world}", "strong"
            self.name = "c3: 256 tables x 2,000,000 rows x dim 128 fp32, global batch 65,536, pooling 32"
        elif a.workload == "c4":
            T, H, D, self.B = 4, 100_000_000, 256, 65536 // world
            plan_name, self.scaling = f"c4_rw_w{world}", "strong"
            if world <= 2:
                self.dtype = torch.float16  # 205.6 GB/GPU in fp32
            self.name = (f"c4: 4 tables x 100,000,000 rows x dim 256 "
                         f"{'fp16' if world <= 2 else 'fp32'}, row-wise over {world} GPUs, global batch 65,536, "
                         "pooling 32")
        elif a.workload == "c5":
            self.B = 65536 // world
            plan_name, self.scaling = f"c5_w{world}", "strong"
            self.fwd_comm, self.bwd_comm = torch.float16, torch.bfloat16
            self.zipf = True
            self.name = ("c5: 512 tables (rows log-uniform 1e3..1e7, dims 32..256, pooling 1..64, Zipf 1.05), "
                         "mixed TW/RW/CW/DP plan, fp16 fwd / bf16 bwd all-to-all, global batch 65,536")
        else:
            raise SystemExit(f"unknown workload {a.workload}")
        if a.workload == "c5":
            self.model = spec.model_from_json((ROOT / "configs" / "models" / "c5.json").read_text())
        else:
            self.model = spec.ModelSpec(tables=tuple(spec.TableSpec(f"t{i}", H, D, float(L)) for i in range(T)),
                                        local_batch=self.B)
        self.plan_file = ROOT / "configs" / "plans" / f"{plan_name}.json"
        self.plan = P.plan_from_json(self.plan_file.read_text())
        self.rows = np.array([t.num_rows for t in self.model.tables], dtype=np.int64)
        self.pool = np.array([t.avg_pooling for t in self.model.tables])

    def table_bytes_per_rank(self, world: int) -> float:
        """Largest per-rank table + moment footprint under the plan."""
        import torch

        e = torch.empty(0, dtype=self.dtype).element_size()
        from paper_2104_05158_b200 import plan as P

        lay = P.rank_layout(self.model, self.plan)
        dp = sum(self.model.tables[t].num_rows * (self.model.tables[t].dim * e + 4) for t in lay.dp_tables)
        return dp + max(sum(s.num_rows * (s.dim * e + 4) for s in lay.owned[v]) for v in range(world))

    def lengths(self, seed: int) -> np.ndarray:
        """(T, B) bag lengths: floor(L) + Bernoulli(frac L) (model.py:396-401)."""
        rng = np.random.default_rng(seed)
        base = np.floor(self.pool).astype(np.int64)[:, None]
        frac = (self.pool - np.floor(self.pool))[:, None]
        return base + (rng.random((len(self.pool), self.B)) < frac)

    def ids(self, lengths: np.ndarray, gen, device, host: bool = False):
        """Table-major int32 ids: uniform, or a continuous Zipf(alpha) inverse
        CDF (bounded power law, floor) for the skewed config."""
        import torch

        counts = torch.from_numpy(lengths.sum(axis=1))
        dev = "cpu" if host else device
        H = torch.repeat_interleave(torch.from_numpy(self.rows), counts).to(dev)
        u = torch.rand(H.numel(), generator=gen, device=dev, dtype=torch.float64)
        if self.zipf:
            alpha = 1.05
            top = H.double().pow(1.0 - alpha)
            x = (1.0 + u * (top - 1.0)).pow(1.0 / (1.0 - alpha))
            ids = torch.minimum(x.floor().long() - 1, H - 1).clamp_(min=0)
        else:
            ids = torch.minimum((u * H).long(), H - 1)
        return ids.to(torch.int32)


def local_fwd_bytes(eng, wl, n, B) -> float:
    """Compulsory forward bytes of this rank's local shards for the last
    step's routed id counts (rows + ids + offsets + pooled write)."""
    import torch

    st = eng.states[0]
    e = torch.empty(0, dtype=eng.dtype).element_size()
    total = 0.0
    shards = eng.lay.owned[st.rank]
    for s, c in zip(shards, st.sc.get("shard_counts", [])):
        total += c * (s.dim * e + 4) + (n + 1) * 8 + n * s.dim * 4
    for t, c in zip(eng.lay.dp_tables, st.sc.get("dp_counts", [])):
        D = wl.model.tables[t].dim
        total += c * (D * e + 4) + (B + 1) * 8 + B * D * 4
    return total


def run_sharded(a, rank, world, dev):
    """N>1: sharded embedding step (one rank per GPU).  c2 (default): the
    single-GPU config's per-GPU work at every N (weak scaling); c3/c4/c5:
    the BASELINE multi-GPU configs at a fixed global batch (strong)."""
    import torch
    import torch.distributed as tdist

    from paper_2104_05158_b200 import dist as nd

    # stdout carries exactly one JSON line: anything the communicator setup
    # prints (NCCL's version banner) is sent to stderr
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    tdist.init_process_group("nccl", device_id=dev)
    wl = ShardedWorkload(a, world)
    B = wl.B
    need = wl.table_bytes_per_rank(world)
    have = torch.cuda.get_device_properties(dev).total_memory
    if need > 0.75 * have:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "unavailable": f"{a.workload} at {world} GPUs needs "
                              f"{need / 1e9:.0f} GB of tables per GPU (> 75% of {have / 1e9:.0f} GB); "
                              "run it on more GPUs"}), file=json_out, flush=True)
        tdist.destroy_process_group()
        return
    comm = nd.NcclComm()
    eng = nd.ShardedEmbedding(wl.model, wl.plan, comm, B, device=dev, dtype=wl.dtype, optim="rowwise_adagrad",
                              index_dtype=torch.int32, transport=a.transport, fwd_comm=wl.fwd_comm,
                              bwd_comm=wl.bwd_comm)
    torch.manual_seed(rank)
    for st in eng.states:
        for grp in list(st.groups) + [st.dp_group]:
            if grp is not None:
                for w in grp.weights:
                    w.normal_()
    lengths = wl.lengths(77 + rank)
    L_dev = torch.from_numpy(lengths.reshape(-1)).to(dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    ids = [wl.ids(lengths, g, dev) for _ in range(2)]

    def step(i, timers=None):
        return eng.step([(lengths, ids[i % 2], L_dev)], lr=LR, eps=EPS, timers=timers)

    clocks = Clocks(dev.index) if rank == 0 else None  # before the warm-up (see run_b200)
    for i in range(a.warmup):
        step(i)
    launches_per_step = count_launches(lambda: step(0))
    torch.cuda.synchronize()
    tdist.barrier()
    time.sleep(0.3)
    timers = {}
    torch.cuda.synchronize()
    tdist.barrier()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    evs[0].record()
    for i in range(a.steps):
        step(i, timers)
        evs[i + 1].record()
    torch.cuda.synchronize()
    tdist.barrier()
    clk = clocks.stop() if clocks else None
    ms_local = evs[0].elapsed_time(evs[-1]) / a.steps
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
    ph = {k: float(np.mean([x.elapsed_time(y) for x, y in v])) for k, v in timers.items()}
    n = B * world
    fb_local = local_fwd_bytes(eng, wl, n, B)
    fwd_gbs_local = fb_local / (ph.get("fwd", 1.0) * 1e-3) / 1e9
    t = torch.tensor([ms_local, ph.get("fwd", 0.0), ph.get("bwd", 0.0), ph.get("a2a_fwd", 0.0),
                      ph.get("a2a_bwd", 0.0), fb_local, ph.get("inputs", 0.0), ph.get("dp", 0.0)],
                     dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms, fwd_ms, bwd_ms, a2f_ms, a2b_ms, fb_max, in_ms, dp_ms = t.tolist()
    tmin = torch.tensor([fwd_gbs_local], dtype=torch.float64, device=dev)
    tdist.all_reduce(tmin, op=tdist.ReduceOp.MIN)
    busbw = alltoall_busbw(eng, dev, world)
    nvl = alltoall_nvlink_busbw(eng, dev, world) if a.transport == "nvlink" else None
    peak, peak_kind = hbm_peak()
    send = max(eng.pooled_send_bytes(v) for v in range(world))
    e2e = None if a.no_e2e else e2e_sharded(a, wl, eng, rank, world, dev, lengths, L_dev)
    if rank != 0:
        tdist.destroy_process_group()
        return
    fwd_gbs = fb_max / (fwd_ms * 1e-3) / 1e9
    kinds = sorted({x.scheme.kind.value for x in wl.plan.assignments})
    line = {
        "metric": METRIC, "value": n / (ms * 1e-3), "unit": UNIT, "n_gpus": world, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": wl.scaling,
        "vs_baseline": None, "dtype": "f16" if wl.dtype == torch.float16 else "f32", "data": "synthetic",
        "config": {"workload": wl.name + f", sharded over {world} GPUs ({wl.plan_file.name})",
                   "tables": wl.model.num_tables, "batch_per_gpu": B, "global_batch": n,
                   "lookups_per_step": int(lengths.sum()) * world, "schemes": kinds,
                   "parallelism": "+".join({"table_wise": "tw", "row_wise": "rw", "column_wise": "cw",
                                            "data_parallel": "dp"}[k] for k in kinds) + str(world),
                   "wire": {"fwd": str(eng.fwd_comm).replace("torch.", ""),
                            "bwd": str(eng.bwd_comm).replace("torch.", "")},
                   "l2": "inputs larger than L2"},
        "roofline": {"bound": "hbm", "kernel": "tbe_forward_kernel (local shards; slowest rank)", "achieved": fwd_gbs,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": fwd_gbs / peak, "traffic": None,
                     "algorithmic_bytes": fb_max, "ms": fwd_ms, "min_rank_gbs": float(tmin.item())},
        "phases_ms": {"fwd_incl_overlapped_a2a": fwd_ms, "a2a_fwd_tail": a2f_ms,
                      "bwd_incl_overlapped_a2a": bwd_ms, "input_exchange": in_ms, "dp_allreduce_update": dp_ms,
                      "overlap_groups": eng.G, "transport": a.transport,
                      "rank0_step_ms": [round(x, 3) for x in per_step]},
        "alltoall": {"send_bytes_per_gpu": send, "busbw_gbs": busbw["busbw_gbs"], "ms": busbw["ms"],
                     "peak_gbs": 900.0, "frac_of_nominal": busbw["busbw_gbs"] / 900.0,
                     "note": "pooled all-to-all payload of one step (per-GPU send bytes excluding self, "
                             "comms.py:366-392) through NCCL all_to_all_single, timed standalone with CUDA "
                             "events, max over ranks"},
        "gpu_launches": launches_per_step * a.steps,
        "clocks": clk,
    }
    if a.workload == "c2":
        U = expected_unique(a.rows, n * a.pooling)
        T_loc = max(len(eng.lay.owned[v]) for v in range(world))
        bb = bwd_bytes([U] * T_loc, n * a.pooling, a.dim, n)
        line["roofline_bwd"] = {"achieved": bb / (bwd_ms * 1e-3) / 1e9, "bytes_expected_U": bb, "ms": bwd_ms}
    if nvl is not None:
        line["alltoall_nvlink"] = {**nvl, "peak_gbs": 900.0, "frac_of_nominal": nvl["busbw_gbs"] / 900.0,
                                   "note": "the same payload stored by neo_copy_pieces straight into every "
                                           "peer's symmetric receive buffer + a symmetric-memory barrier "
                                           "(the transport the step uses), max over ranks"}
    if e2e is not None:
        line["e2e"] = e2e
    print(json.dumps(line), file=json_out, flush=True)
    tdist.destroy_process_group()


def alltoall_busbw(eng, dev, world) -> dict:
    """Pooled all-to-all bus bandwidth at this step's payload: per-GPU bytes
    sent to other GPUs / time (nccl-tests alltoall busbw definition)."""
    import torch
    import torch.distributed as tdist

    rank = tdist.get_rank()
    B = eng.B
    per_peer = B * eng.widths[rank]
    send = torch.empty(per_peer * world, dtype=eng.fwd_comm, device=dev)
    recv = torch.empty(sum(B * eng.widths[w] for w in range(world)), dtype=eng.fwd_comm, device=dev)
    osp = [B * eng.widths[w] for w in range(world)]
    for _ in range(3):
        tdist.all_to_all_single(recv, send, osp, [per_peer] * world)
    torch.cuda.synchronize()
    tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        tdist.all_to_all_single(recv, send, osp, [per_peer] * world)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes = per_peer * (world - 1) * send.element_size()
    return {"ms": ms, "busbw_gbs": nbytes / (ms * 1e-3) / 1e9}


def alltoall_nvlink_busbw(eng, dev, world) -> dict:
    """Peer-store all-to-all over NVLink at the same payload: each rank's
    (B x width) pooled block is written into every other rank's symmetric
    buffer by one neo_copy_pieces launch, then a symmetric-memory barrier."""
    import torch
    import torch.distributed as tdist

    from paper_2104_05158_b200 import tbe

    rank = tdist.get_rank()
    B, wd = eng.B, max(eng.widths[rank], 1)
    src = torch.zeros((B, wd), dtype=eng.fwd_comm, device=dev)
    off = int(eng.src_off[rank])
    pieces = [tbe.Piece(src, eng.hdl_pool.get_buffer(v, (B, wd), eng.fwd_comm, off), 0, 0, wd)
              for v in range(world) if v != rank]
    pdev = tbe.pack_pieces(pieces, dev)

    def once():
        tbe.copy_pieces(B, pieces, pdev)
        eng.hdl_pool.barrier(channel=0)

    for _ in range(3):
        once()
    torch.cuda.synchronize()
    tdist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        once()
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    nbytes = B * eng.widths[rank] * (world - 1) * src.element_size()
    return {"ms": ms, "busbw_gbs": nbytes / (ms * 1e-3) / 1e9}


def e2e_sharded(a, wl, eng, rank, world, dev, lengths, L_dev) -> dict:
    """Sharded step with host (pinned) ids copied H2D each step on a side
    stream (prefetch of the next batch overlaps the current step) and the
    loss read back D2H."""
    import torch
    import torch.distributed as tdist

    B = wl.B
    gen = torch.Generator().manual_seed(99 + rank)
    host = [wl.ids(lengths, gen, dev, host=True).pin_memory() for _ in range(2)]
    dev_ids = [torch.empty_like(h, device=dev) for h in host]
    copied = [torch.cuda.Event() for _ in range(2)]
    free = [torch.cuda.Event() for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)
    comp = torch.cuda.current_stream(dev)
    losses = torch.empty(a.warmup + a.steps, dtype=torch.float32, pin_memory=True)

    def stage(i):
        with torch.cuda.stream(cs):
            cs.wait_event(free[i % 2])
            dev_ids[i % 2].copy_(host[i % 2], non_blocking=True)
            copied[i % 2].record(cs)

    for e in free:
        e.record(comp)
    total = a.warmup + a.steps
    stage(0)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    for i in range(total):
        if i == a.warmup:
            torch.cuda.synchronize()
            tdist.barrier()
            e0.record(comp)
        if i + 1 < total:
            stage(i + 1)
        comp.wait_event(copied[i % 2])
        pooled = eng.step([(lengths, dev_ids[i % 2], L_dev)], lr=LR, eps=EPS)
        losses[i:i + 1].copy_(pooled[0].sum().reshape(1), non_blocking=True)
        free[i % 2].record(comp)
    e1.record(comp)
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1) / a.steps], dtype=torch.float64, device=dev)
    tdist.all_reduce(ms, op=tdist.ReduceOp.MAX)
    ms = float(ms.item())
    return {"value": B * world / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": host[0].numel() * 4 * world + lengths.size * 8 * world,
            "d2h_bytes_per_step": 4 * world,
            "api": "paper_2104_05158_b200.dist.ShardedEmbedding.step (pinned host ids per rank, H2D prefetch "
                   "overlapped, loss read back)"}


def main(argv=None):
    a = parse_args(argv)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != a.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} but --gpus {a.gpus}", file=sys.stderr)
    if a.impl == "reference":
        return run_reference(a, rank, world)
    return run_b200(a, rank, world)


if __name__ == "__main__":
    main()
