"""Debug: multi-process ping-pong with the launch handshake."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import torch.distributed as dist
import paper_2511_15076_b200 as G

rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
def ag(blob):
    out = [None] * world
    dist.all_gather_object(out, blob)
    return out
comm = G.Comm.create(rank, world, local, ag, G.Config(signal_cells=512, timeout_ms=5000))
sz = 1 << 20
sb, rb = comm.mem_alloc(sz), comm.mem_alloc(sz)
ws, wr = comm.window_register(sb, sz), comm.window_register(rb, sz)
rtt = torch.zeros(1000, dtype=torch.int64, device=torch.device("cuda", local))
sig = int(os.environ.get("SIG", "401"))
for s in [8, 64, 4096]:
    print(rank, "before", s, comm.read_signal(sig), comm.read_signal(sig + 1), flush=True)
    try:
        G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles([comm]), 1, 0, 1, ws, wr, s, 50, 5, sig, 512, rtt.data_ptr(), None))
    except Exception as e:
        print(rank, "ERR", e, flush=True)
    print(rank, "after", s, comm.read_signal(sig), comm.read_signal(sig + 1), flush=True)
    dist.barrier()
comm.destroy()
dist.destroy_process_group()
