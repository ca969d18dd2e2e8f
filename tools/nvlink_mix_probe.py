"""NVLink push vs pull vs copy-engine vs hybrid ceilings, one process per GPU (torchrun).

Every rank moves `bytes` between its window and peer (rank + 1) % world at once
(push: write the peer's window; pull: read the peer's window into its own;
hybrid: TMA pushes part while the copy engine pushes the rest on a side
stream).  Rank 0 prints one JSON line per case with the per-rank GB/s
(max-over-ranks time).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/nvlink_mix_probe.py
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
    cases = [("tma_push", 1, 148, 4096, None), ("ce_push", 3, 0, 4096, None),
             ("tma_pull", 5, 148, 4096, None), ("tma_pull_296", 5, 296, 4096, None),
             ("tma_pull_6k", 5, 148, 6144, None), ("lsu256_pull", 7, 296, 4096, None),
             ("lsu256_pull_592", 7, 592, 4096, None)]
    if world > 2:
        cases.append(("ce_all_peers", 8, 0, 4096, None))
        cases.append(("tma_push_one_peer", 1, 148, 4096, None))
    if os.environ.get("MIX_ONLY_CE"):
        cases = [c for c in cases if c[1] in (1, 3, 8)]
    for pct in (() if os.environ.get("MIX_ONLY_CE") else (10, 20, 30, 40, 60)):
        cases.append((f"hybrid_ce{pct}", 6, 148, 4096, pct))
        cases.append((f"hybrid_ce{pct}_64cta", 6, 64, 4096, pct))
    for name, eng, ctas, chunk, pct in cases:
        if pct is not None:
            os.environ["GINSIM_HYBRID_CE_PCT"] = str(pct)
        ms = ctypes.c_float(0.0)
        dist.barrier()
        G.check(G.lib().ginsim_cuda_copy_bench_ex(comm.h, ws, wd, peer, size, eng, ctas, chunk, 5,
                                                   ctypes.byref(ms), None))
        t = torch.tensor([ms.value], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            print(json.dumps({"case": name, "world": world, "bytes": size, "ms": round(t.item(), 4),
                              "GBps_per_gpu": round(size / t.item() / 1e6, 1)}), flush=True)
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
