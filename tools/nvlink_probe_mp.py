"""NVLink write-path roofline, one process per GPU (torchrun).

Every rank copies `bytes` from its own window into the window of peer
(rank + 1) % world with each engine of ginsim_cuda_copy_bench_ex, all ranks
at once (so every GPU's NVLink carries egress and ingress together, as in the
dispatch / combine all-to-all), then rank 0 alone (one direction).  Rank 0
prints one JSON line with per-rank egress GB/s (max-over-ranks time).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvlink_probe_mp.py
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402

ENGINES = ["lsu128", "tma", "lsu256", "copy_engine", "tma_store_only"]


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def allgather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out
    comm = G.Comm.create(rank, world, local, allgather, G.Config())
    size = int(os.environ.get("PROBE_BYTES", 512 << 20))
    src, dst = comm.mem_alloc(size), comm.mem_alloc(size)
    ws, wd = comm.window_register(src, size), comm.window_register(dst, size)
    peer = (rank + 1) % world
    dev = torch.device("cuda", local)
    rows = []
    configs = []
    for eng in (0, 2):
        for ctas in (16, 32, 64, 148, 296):
            configs.append((eng, ctas, 4096))
    for eng in (1, 4):
        for ctas in (16, 32, 64, 148):
            for chunk in ((2048, 4096, 8192, 16384) if eng == 4 else (2048, 4096, 6144)):
                configs.append((eng, ctas, chunk))
    configs.append((3, 0, 4096))
    for mode in ("bidir", "unidir"):
        for eng, ctas, chunk in configs:
            for target in ("peer", "local"):
                p = peer if target == "peer" else rank
                ms = ctypes.c_float(0.0)
                dist.barrier()
                active = mode == "bidir" or rank == 0
                if active:
                    G.check(G.lib().ginsim_cuda_copy_bench_ex(comm.h, ws, wd, p, size, eng, ctas, chunk, 5,
                                                              ctypes.byref(ms), None))
                t = torch.tensor([ms.value if active else 0.0], dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                rows.append({"mode": mode, "engine": ENGINES[eng], "ctas": ctas or 0, "chunk": chunk, "target": target,
                             "ms": t.item(), "GBps": size / (t.item() * 1e-3) / 1e9})
    if rank == 0:
        best = {}
        for r in rows:
            k = (r["mode"], r["target"], r["engine"])
            if k not in best or r["GBps"] > best[k]["GBps"]:
                best[k] = r
        print(json.dumps({"gpus": world, "bytes": size, "best": list(best.values()), "rows": rows}))
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
