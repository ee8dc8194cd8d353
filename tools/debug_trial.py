"""Debug one criterion-5 style trial: drop-in vs reference, per table (development tool)."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))
sys.path.insert(0, str(ROOT / "tests"))
import neosim  # noqa: E402
from neosim import comms  # noqa: E402

from test_gpu_dropin import _desk_model, _random_plan  # noqa: E402

orig_sharded = comms.train_step_sharded
orig_reasm = comms.reassemble_values
from paper_2104_05158_b200 import dropin  # noqa: E402

dropin.install(neosim)
rng = np.random.default_rng(2024)
kinds = [neosim.OptimizerKind.SGD, neosim.OptimizerKind.ROWWISE_ADAGRAD, neosim.OptimizerKind.ADAGRAD]
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    tables = [neosim.TableSpec(id=f"t{i}", num_rows=int(rng.integers(8, 33)), dim=int(rng.integers(1, 4)) * 2,
                               avg_pooling=float(rng.uniform(1.0, 3.5))) for i in range(int(rng.integers(1, 9)))]
    model = _desk_model(neosim, tables, int(rng.integers(1, 4)))
    W = int(rng.choice([1, 2, 4]))
    gpn = 2 if W == 4 and trial % 2 else W
    plan = _random_plan(neosim, rng, model, W, gpn)
    cfg = neosim.OptimizerConfig(kinds[trial % 3], lr=0.1, eps=1e-8)
    seed = int(rng.integers(10_000))
    batch = neosim.gen_synthetic_batch(model, W * model.local_batch, seed)
    want_out, want_state = orig_sharded(model, plan, batch, cfg, seed=seed)
    got_out, got_state = neosim.train_step_sharded(model, plan, batch, cfg, seed=seed)
    print(f"trial {trial} W={W} B={model.local_batch} kind={cfg.kind.value} out_equal={np.array_equal(got_out, want_out)}")
    for a, g, w in zip(plan.assignments, neosim.comms.reassemble_values(model, plan, got_state),
                       orig_reasm(model, plan, want_state)):
        d = np.abs(g - w)
        bad = np.argwhere(d > 0)
        print(f"   {a.table_id} {a.scheme.kind.value:14s} shards={[(s.worker, s.rows, s.cols) for s in a.shards]} "
              f"maxdiff={d.max():.3g} bad_rows={sorted(set(bad[:, 0].tolist()))[:8]}")
