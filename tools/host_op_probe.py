"""Cost of the proxy agent's building blocks on this box: stream memops
(cuStreamBatchMemOp 64-bit writes, various batch sizes) and small / large
cudaMemcpyAsync copies into a peer's window (2 ranks, one process each).

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/host_op_probe.py
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
    size = 64 << 20
    src, dst = comm.mem_alloc(size), comm.mem_alloc(size)
    ws, wd = comm.window_register(src, size), comm.window_register(dst, size)
    peer = (rank + 1) % world
    cases = []
    for tgt in ("local", "peer"):
        for batch in (1, 32, 128):
            cases.append((tgt, 0, 512, batch, 0))
        for nbytes in (8, 256, 4096, 65536):
            cases.append((tgt, 1, 256, 1, nbytes))
    out = (ctypes.c_float * 2)()
    for tgt, kind, n_ops, batch, nbytes in cases:
        if rank == 0:
            p = peer if tgt == "peer" else rank
            G.check(G.lib().ginsim_cuda_host_op_bench(comm.h, ws, wd, p, kind, n_ops, batch, nbytes, out, None))
            print(json.dumps({"target": tgt, "op": "memop64" if kind == 0 else "memcpy", "n_ops": n_ops,
                              "batch": batch, "bytes": nbytes, "dev_us_per_op": round(out[0], 3),
                              "host_us_per_op": round(out[1], 3)}), flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
