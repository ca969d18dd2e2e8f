"""LL shape (128 tokens/rank, hidden 7168, top-8 of 256, bf16) per engine and
layout: dispatch / combine p50 device time, max over ranks.  torchrun."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")

    def ag(blob):
        o = [None] * world
        dist.all_gather_object(o, blob)
        return o
    comm = G.Comm.create(rank, world, local, ag, G.Config(signal_cells=512))
    T, H, K, E = 128, 7168, 8, 256
    dev = torch.device("cuda", local)
    res = {}
    for engine, layout in ((2, 1), (1, 1), (2, 2), (2, 0), (1, 0)):
        moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 1, layout, 0, engine))
        x = torch.empty(T * H, dtype=torch.int16, device=dev)
        idx = torch.empty(T * K, dtype=torch.int32, device=dev)
        w = torch.empty(T * K, dtype=torch.float32, device=dev)
        out = torch.empty(T * H, dtype=torch.int16, device=dev)
        moe.generate(1, rank, x, idx, w)
        s = torch.cuda.Stream()
        for _ in range(5):
            G.Moe.dispatch([moe], [x], [idx], stream=s)
            G.Moe.combine([moe], [w], [out], stream=s)
        torch.cuda.synchronize()
        dist.barrier()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(50)]
        for e in ev:
            e[0].record(s)
            G.Moe.dispatch([moe], [x], [idx], stream=s)
            e[1].record(s)
            G.Moe.combine([moe], [w], [out], stream=s)
            e[2].record(s)
        torch.cuda.synchronize()
        comm.check_device()
        d = sorted(e[0].elapsed_time(e[1]) for e in ev)[25]
        c = sorted(e[1].elapsed_time(e[2]) for e in ev)[25]
        t = torch.tensor([d, c], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        res[f"engine{engine}_layout{layout}"] = [round(t[0].item() * 1e3, 1), round(t[1].item() * 1e3, 1)]
        moe.destroy()
    if rank == 0:
        print(json.dumps({"world": world, "ll_dispatch_combine_us": res}))
    dist.barrier()


if __name__ == "__main__":
    main()
