"""pytest plugin (``-p neo_dropin_plugin``, tests/ on PYTHONPATH) that routes the reference
package copied into oracle/_ref through the B200 operators before the
reference's own tests are collected: dropin.install(neosim) patches every
hot-path name, so pkg/tests exercise this implementation."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
REF = ROOT / "oracle" / "_ref"
for p in (str(ROOT), str(REF)):
    if p not in sys.path:
        sys.path.insert(0, p)

import neosim  # noqa: E402  (the copied reference)

import paper_2104_05158_b200 as _neo  # noqa: E402
from paper_2104_05158_b200 import dropin  # noqa: E402

dropin.install(neosim)
assert neosim.embedding.forward_pooled is _neo.embedding.forward_pooled
assert neosim.comms.train_step_sharded is _neo.comms.train_step_sharded


def pytest_report_header(config):
    return f"dropin: neosim from {Path(neosim.__file__).parent} routed through {Path(_neo.__file__).parent}"


def pytest_sessionfinish(session, exitstatus):
    import torch

    torch.cuda.synchronize()
    print(f"\ndropin: CUDA device used: {torch.cuda.get_device_name(0)}; "
          f"max memory allocated {torch.cuda.max_memory_allocated() / 2**20:.1f} MiB")
