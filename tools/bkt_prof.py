"""Row-kernel role breakdown from a NEO_BKT_PROF build (abv/libneob200_prof.so):
one c2-sized backward, then the clock64 sums per role."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("NEO_B200_LIB", str(ROOT / "abv" / "libneob200_prof.so"))
import paper_2104_05158_b200 as neo  # noqa: E402
from paper_2104_05158_b200 import _capi, tbe  # noqa: E402

neo.load()
T, H, D, B, L = int(os.environ.get("T", 16)), 1_000_000, 128, 65536, 32
grp = tbe.TableGroup([H] * T, [D] * T, dtype=torch.float32, optim="rowwise_adagrad")
grp._storage.normal_()
off = torch.arange(0, T * B + 1, dtype=torch.int64, device="cuda") * L
ix = torch.randint(0, H, (T * B * L,), dtype=torch.int32, device="cuda")
up = torch.randn((B, T * D), device="cuda")
lib = _capi.lib()
lib.neo_bkt_prof.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 12)()
for it in range(3):
    lib.neo_bkt_prof(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    timers = {}
    grp.backward(ix, off, B, up, mode="update", optim="rowwise_adagrad", lr=0.05, eps=1e-8, timers=timers)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b, _, _ in timers["apply"]][0]
    lib.neo_bkt_prof(buf, 0)
    v = list(buf)
    nb, nc = max(v[4], 1), max(v[7], 1)
    print(f"rows kernel {ms:.3f} ms; batches {v[4]}; producer cyc/batch: loop {v[0]/nb:.0f} "
          f"top->wait {v[2]/nb:.0f} wait-empty {v[1]/nb:.0f} issue {v[3]/nb:.0f}; consumer stages {v[7]} "
          f"cyc/stage: wait-full {v[5]/nc:.0f} work {v[6]/nc:.0f}; issue split: upstream {v[8]/nb:.0f} "
          f"weights+moments {v[9]/nb:.0f}; table consts {v[10]/nb:.0f}", flush=True)
