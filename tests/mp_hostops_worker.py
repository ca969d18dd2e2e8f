"""One rank of a multi-process run through host-issued ops only (no kernel
spins on a peer, so two processes may share one GPU without MPS): the
cross-process window path -- POSIX-FD export, pidfd_getfd import,
cuMemImportFromShareableHandle + cuMemMap -- exercised by put / put_value /
signal / counters / flush on both backends, window deregistration and id
reuse across processes, and (MP_ORDERING=1, distinct GPUs only) the
acceptance-#1 ordering stress over real NVLink.  Launched by
tests/test_gpu_multi.py; writes rank<i>.json into $MP_OUT."""
import os as _os
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def pattern(src, n):
    return ((np.arange(n, dtype=np.uint64) * 131 + src * 7 + 3) % 251).astype(np.uint8)


def main():
    import torch
    import torch.distributed as dist

    import paper_2511_15076_b200 as G
    from tests import gpu_util as U

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = 0 if os.environ.get("MP_SAME_DEVICE") == "1" else local
    torch.cuda.set_device(dev)
    U.set_device(dev)
    dist.init_process_group("gloo")

    def allgather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out

    res = {"rank": rank, "device": dev}
    socket = os.environ.get("MP_TRANSPORT") == "socket"
    # the socket transport (GIN1 frames over TCP between the agents) runs on
    # the Proxy backend only
    for backend in (("socket",) if socket else ("direct", "proxy")):
        cfg = (G.Config(backend="proxy", transport="socket", timeout_ms=20000, signal_cells=512) if backend == "socket"
               else G.Config(backend=backend, timeout_ms=20000))
        comm = G.Comm.create(rank, world, dev, allgather, cfg)
        S = 1 << 20
        # separate send and receive windows: a receive slot must never be
        # another put's source (a peer's put could land in it first)
        sbuf = comm.mem_alloc(world * S)
        swin = comm.window_register(sbuf, world * S)
        buf = comm.mem_alloc(world * S)
        win = comm.window_register(buf, world * S)
        U.h2d(sbuf, np.tile(pattern(rank, S), world))
        U.sync()
        torch.cuda.synchronize()
        dist.barrier()
        g = G.Gin(comm, rank % 4)
        # everyone puts its pattern into every peer's slot [rank], SignalAdd(1) on cell 100
        for p in range(world):
            if p != rank:
                g.put(p, win, rank * S, swin, p * S, S, signal=100, add=1, counter=1)
        # and an inline value + SignalInc on cell 101
        for p in range(world):
            if p != rank:
                g.put_value(p, win, rank * S + S - 8, 0x0102030405060708 + rank, 8, signal=101)
        g.flush()
        comm.wait_signal(100, world - 1)
        comm.wait_signal(101, world - 1)
        ok = True
        got = U.d2h(buf, world * S)
        for p in range(world):
            if p == rank:
                continue
            want = pattern(p, S).copy()
            want[S - 8:] = np.frombuffer(np.uint64(0x0102030405060708 + p).tobytes(), np.uint8)
            bad = np.nonzero(got[p * S:(p + 1) * S] != want)[0]
            if bad.size:
                ok = False
                res[f"{backend}_first_bad"] = [int(bad[0]), int(bad.size), int(got[p * S + bad[0]]), int(want[bad[0]])]
        res[f"{backend}_payload_exact"] = ok
        res[f"{backend}_counter"] = comm.read_counter(1)
        res[f"{backend}_cells"] = [comm.read_signal(100), comm.read_signal(101)]
        dist.barrier()
        # deregister + re-register: the freed id is reused on every process
        comm.window_deregister(win)
        comm.mem_free(buf)  # (the freed id is the receive window's, 1; the send window stays at 0)
        buf2 = comm.mem_alloc(4096)
        win2 = comm.window_register(buf2, 4096)
        res[f"{backend}_reused_id"] = win2 == win
        dist.barrier()
        nxt = (rank + 1) % world
        G.Gin(comm, 0).put_value(nxt, win2, 0, 0xABCD0000 + rank, 4, signal=102)
        G.Gin(comm, 0).flush()
        comm.wait_signal(102, 1)
        prev = (rank + world - 1) % world
        res[f"{backend}_after_reuse"] = int(U.d2h(buf2, 4, np.uint32)[0]) == 0xABCD0000 + prev
        dist.barrier()
        if backend == "socket":
            res["net_stats"] = comm.net_stats()
            if os.environ.get("MP_SAME_DEVICE") != "1" and world > 1:
                # device-initiated traffic over the socket transport: the ring
                # program's Gin puts + signals and its device BarrierSession go
                # through descriptors -> agent -> GIN1 frames -> the peer's agent
                S = 4096
                sb, rb = comm.mem_alloc(world * S), comm.mem_alloc(world * S)
                ws_, wr_ = comm.window_register(sb, world * S), comm.window_register(rb, world * S)
                dist.barrier()
                G.check(G.lib().ginsim_cuda_team_ring(G.comm_handles([comm]), 1, 0, ws_, wr_, S, 6, 300, None))
                comm.check_device()
                res["socket_ring_ok"] = True
                # a small MoE step (Proxy kernels submit every cross-rank byte
                # as descriptors): outputs equal the oracle's
                from oracle import oracle as O
                E, K, T, H = 16 * world, 4, 32, 256
                moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 0, 0, 0, 0))
                x = torch.empty(T * H, dtype=torch.int16, device=f"cuda:{dev}")
                idx = torch.empty(T * K, dtype=torch.int32, device=f"cuda:{dev}")
                w = torch.empty(T * K, dtype=torch.int16, device=f"cuda:{dev}")
                out = torch.empty(T * H, dtype=torch.int16, device=f"cuda:{dev}")
                moe.generate(3, rank, x, idx, w)
                torch.cuda.synchronize()
                dist.barrier()
                for _ in range(2):
                    G.Moe.dispatch([moe], [x], [idx])
                    G.Moe.combine([moe], [w], [out])
                torch.cuda.synchronize()
                comm.check_device()
                exp, _ = O.combine(3, E, K, H, rank, T)
                res["socket_moe_exact"] = bool((out.cpu().numpy().view(np.uint16).reshape(T, H) == exp).all())
                d, comb, _ = O.moe_rank_state(3, world, E, K, T, H, rank)
                res["socket_moe_windows_exact"] = bool(
                    (U.d2h(comm.window_ptr(moe.win_dispatch, rank), len(d)) == d).all() and
                    (U.d2h(comm.window_ptr(moe.win_combine, rank), len(comb)) == comb).all())
                dist.barrier()
                moe.destroy()
                res["net_stats_after"] = comm.net_stats()
        if os.environ.get("MP_ORDERING") == "1" and backend == "direct":
            channels, nbytes, rounds = 8, 64 << 10, 200
            size = 2 * channels * nbytes
            sb, db = comm.mem_alloc(size), comm.mem_alloc(size)
            ws, wd = comm.window_register(sb, size), comm.window_register(db, size)
            dist.barrier()
            for _ in range(2):
                G.check(G.lib().ginsim_cuda_ordering_stress(G.comm_handles([comm]), 1, ws, wd, nbytes, channels,
                                                           rounds, None))
            comm.check_device()
            res["ordering_cell"] = comm.read_signal(0)
            res["ordering_expected"] = 2 * rounds
        dist.barrier()
        comm.destroy()
    print("MPRESULT " + json.dumps(res), flush=True)
    out_dir = os.environ.get("MP_OUT")
    if out_dir:
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(res, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
