"""Multi-process put+signal ping-pong p50 for a few sizes (ranks 0 and 1),
next to the raw flag round trip in its four ordering variants
(ginsim_cuda_rtt_floor modes 0-5).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/pp_mp_probe.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))


def ag(blob):
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out


cells = int(os.environ.get("CELLS", "4096"))
sig = int(os.environ.get("SIG", "4001"))
comm = G.Comm.create(rank, world, local, ag, G.Config(signal_cells=cells))
sz = 1 << 20
sb, rb = comm.mem_alloc(sz), comm.mem_alloc(sz)
ws, wr = comm.window_register(sb, sz), comm.window_register(rb, sz)
rtt = torch.zeros(1000, dtype=torch.int64, device=torch.device("cuda", local))
warm = int(os.environ.get("WARMUP", "100"))
threads = int(os.environ.get("THREADS", "0"))
for mode in (0, 1, 2, 3, 4, 5):
    G.check(G.lib().ginsim_cuda_rtt_floor(G.comm_handles([comm]), 1, 0, 1, mode, 1000, warm, 4010, rtt.data_ptr(), None))
    dist.barrier()
    if rank == 0:
        t = np.sort(rtt.cpu().numpy())
        print(f"floor mode {mode} p50 {int(t[500])} p99 {int(t[990])}", flush=True)
for s in (0, 8, 64, 4096):
    G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles([comm]), 1, 0, 1, ws, wr, s, 1000, warm, sig, threads,
                                         rtt.data_ptr(), None))
    dist.barrier()
    if rank == 0:
        t = np.sort(rtt.cpu().numpy())
        print(f"put+signal bytes {s} threads {threads} p50 {int(t[500])} p99 {int(t[990])}", flush=True)
comm.destroy()
dist.destroy_process_group()
