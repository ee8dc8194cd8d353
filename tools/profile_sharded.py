"""Per-kernel time breakdown of one sharded step (torch.profiler on rank 0).

  torchrun --nproc-per-node 4 tools/profile_sharded.py --workload c5 --gpus 4
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as tdist

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_2104_05158_b200 import dist as nd  # noqa: E402


def main():
    a = bench.parse_args(sys.argv[1:])
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    tdist.init_process_group("nccl", device_id=dev)
    wl = bench.ShardedWorkload(a, world)
    eng = nd.ShardedEmbedding(wl.model, wl.plan, nd.NcclComm(), wl.B, device=dev, dtype=wl.dtype,
                              optim="rowwise_adagrad", index_dtype=torch.int32, transport=a.transport,
                              fwd_comm=wl.fwd_comm, bwd_comm=wl.bwd_comm)
    for st in eng.states:
        for grp in list(st.groups) + [st.dp_group]:
            if grp is not None:
                for w in grp.weights:
                    w.normal_()
    lengths = wl.lengths(77 + rank)
    L_dev = torch.from_numpy(lengths.reshape(-1)).to(dev)
    g = torch.Generator(device=dev).manual_seed(1234 + rank)
    ids = wl.ids(lengths, g, dev)
    for _ in range(3):
        eng.step([(lengths, ids, L_dev)], lr=0.05, eps=1e-8)
    torch.cuda.synchronize()
    tdist.barrier()
    timers = {}
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA,
                                            torch.profiler.ProfilerActivity.CPU]) as prof:
        eng.step([(lengths, ids, L_dev)], lr=0.05, eps=1e-8, timers=timers)
        torch.cuda.synchronize()
    tdist.barrier()
    if rank == 0:
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
        ph = {k: float(np.mean([x.elapsed_time(y) for x, y in v])) for k, v in timers.items()}
        print("phases", ph)
        st = eng.states[0]
        print("groups", [None if gp is None else (gp.T, gp.total_rows, gp.max_dim) for gp in st.groups],
              "dp", None if st.dp_group is None else (st.dp_group.T, st.dp_group.total_rows))
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
