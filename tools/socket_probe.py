"""Socket transport (Config(transport="socket"), net.cu) throughput and round
trip between two processes, against the same host-issued ops on the fabric.

  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/socket_probe.py

Bandwidth: rank 0 puts `reps` x S bytes (host-issued, one signal at the end),
flushes (local completion = the peer acked every frame) and reports S*reps /
time.  Round trip: rank 0 puts 8 B + SignalInc, rank 1 waits for it from the
host and answers the same way; p50 over 200 rounds.  One JSON line (rank 0).
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def run(transport, rank, world, local, allgather):
    cfg = G.Config(backend="proxy", transport=transport, timeout_ms=30000, signal_cells=512)
    comm = G.Comm.create(rank, world, local, allgather, cfg)
    S_MAX = 16 << 20
    sb, rb = comm.mem_alloc(S_MAX), comm.mem_alloc(S_MAX)
    ws, wr = comm.window_register(sb, S_MAX), comm.window_register(rb, S_MAX)
    g = G.Gin(comm, 0)
    out = {"transport": transport, "bw": [], "rtt_8B_us": None}
    peer = 1 - rank
    sig = 10
    for S in (4096, 65536, 1 << 20, 4 << 20, 16 << 20):
        reps = max(4, min(200, (256 << 20) // S))
        dist.barrier()
        if rank == 0:
            t0 = time.perf_counter()
            for i in range(reps):
                g.put(peer, wr, 0, ws, 0, S, signal=sig if i == reps - 1 else None)
            g.flush()
            dt = time.perf_counter() - t0
            out["bw"].append({"bytes": S, "reps": reps, "GBps": S * reps / dt / 1e9})
        else:
            comm.wait_signal(sig, 1)
        sig += 1
        dist.barrier()
    rtts = []
    dist.barrier()
    for i in range(200):
        if rank == 0:
            t0 = time.perf_counter()
            g.put_value(peer, wr, 0, i, 8, signal=100)
            comm.wait_signal(101, i + 1)
            rtts.append(time.perf_counter() - t0)
        else:
            comm.wait_signal(100, i + 1)
            g.put_value(peer, wr, 0, i, 8, signal=101)
    if rtts:
        out["rtt_8B_us"] = float(np.median(rtts) * 1e6)
    if transport == "socket":
        out["net_stats"] = comm.net_stats()
    dist.barrier()
    comm.destroy()
    return out


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")

    def allgather(blob):
        o = [None] * world
        dist.all_gather_object(o, blob)
        return o
    res = [run(t, rank, world, local, allgather) for t in ("socket", "fabric")]
    if rank == 0:
        print(json.dumps({"tool": "socket_probe", "world": world, "host_issued": True, "runs": res}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
