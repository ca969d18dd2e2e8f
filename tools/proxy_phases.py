"""Per-CTA phase stamps of the Proxy pipeline kernels (GINSIM_PROFILE_PHASES=1)
at the HT shape, one process per GPU; rank 0 prints, per kernel and stamp
slot, the min/median/max offset (us) from the dispatch launch's first stamp.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/proxy_phases.py
"""
import json
import os
import sys

os.environ["GINSIM_PROFILE_PHASES"] = "1"
os.environ["GINSIM_PROXY_TRACE"] = "1"
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)

    def allgather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out
    T, H, K, E = int(os.environ.get("TL_TOKENS", "4096")), 7168, 8, 256
    comm = G.Comm.create(rank, world, local, allgather, G.Config(backend="proxy", signal_cells=512))
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 1, 1, 0, 0))
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    stream = torch.cuda.Stream(device=dev)
    moe.generate(1, rank, x, idx, w, stream=stream)
    for _ in range(4):
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
    torch.cuda.synchronize()
    dist.barrier()
    comm.proxy_trace()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    G.Moe.dispatch([moe], [x], [idx], stream=stream)
    G.Moe.combine([moe], [w], [out], stream=stream)
    torch.cuda.synchronize()
    tr = comm.proxy_trace()
    st = [moe.phase_times(k).astype(np.int64) for k in range(3)]
    t0 = st[0][:, 0][st[0][:, 0] > 0].min()
    res = {"rank": rank, "world": world, "transport": moe.transport(),
           "copies": [[int(b), int(c), round(h, 1), round(s, 1), round(d, 1),
                       round(b / max(d, 1e-3) / 1e3, 1)] for b, c, h, s, d in tr]}
    for k, name in enumerate(("dispatch", "combine_send", "reduce")):
        rows = {}
        for s in range(8):
            col = st[k][:, s]
            col = col[col > 0]
            if len(col):
                rel = (col - t0) / 1e3
                rows[s] = [round(float(rel.min()), 1), round(float(np.median(rel)), 1), round(float(rel.max()), 1)]
        res[name] = rows
    outs = [None] * world
    dist.all_gather_object(outs, res)
    if rank == 0:
        for r in outs:
            print(json.dumps(r), flush=True)
    moe.destroy()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
