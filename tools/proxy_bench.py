"""Proxy backend dispatch/combine at the HT and LL shapes (bench.py's
measure_proxy), with the pipelined transport and with the one-shot LSU
staging kernels (GINSIM_PROXY_PIPE=0), one process per GPU.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/proxy_bench.py
"""
import os as _os
# every stream its own hardware queue: a proxy-agent stream aliased onto the queue of
# a kernel that waits for the agent would stall behind it (csrc/proxy.cu)
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
import paper_2511_15076_b200 as G  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(device=dev)

    def allgather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out
    variants = os.environ.get("PB_VARIANTS", "pipe,lsu").split(",")
    for T in (4096, 128):
        for var in variants:
            os.environ["GINSIM_PROXY_PIPE"] = "0" if var == "lsu" else "1"
            r = bench.measure_proxy(G, rank, world, local, dist, torch, dev, stream, allgather, T,
                                    int(os.environ.get("PB_STEPS", "10")))
            if rank == 0:
                r["variant"] = var
                print(json.dumps(r), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
