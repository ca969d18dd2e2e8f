"""One rank of a multi-process (torchrun) parity run: real GPUs, one process
per GPU, NVLink peer mappings imported through POSIX-FD handles.
Launched by tests/test_gpu_multi.py; prints one JSON line per rank."""
import os as _os
# every stream its own hardware queue: a proxy-agent stream aliased onto the queue of
# a kernel that waits for the agent would stall behind it (csrc/proxy.cu)
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist

    import paper_2511_15076_b200 as G
    from oracle import oracle as O

    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")

    def allgather(blob):
        out = [None] * world
        dist.all_gather_object(out, blob)
        return out

    T = int(os.environ.get("MP_TOKENS", "256"))
    mode = int(os.environ.get("MP_MODE", "0"))
    layout = int(os.environ.get("MP_LAYOUT", "1"))
    E, K, H, seed = 256, 8, 7168, 1
    backend = os.environ.get("MP_BACKEND", "direct")
    iters = int(os.environ.get("MP_ITERS", "3"))
    comm = G.Comm.create(rank, world, local, allgather, G.Config(backend=backend, signal_cells=512, timeout_ms=20000))
    cfg = G.MoeConfig(E, K, T, H, mode, layout, 0)
    moe = G.Moe(comm, cfg)
    dev = torch.device("cuda", local)
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32 if mode else torch.int16, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(seed, rank, x, idx, w)
    torch.cuda.synchronize()
    res = {"rank": rank, "ok": True}
    if os.environ.get("MP_GRAPH") == "1":
        # one eager step (plans the grids), then the step captured once in a
        # CUDA graph and replayed: the pipelined combine's programmatic
        # dependent launch becomes a graph edge; outputs are cleared first so
        # the replays must rewrite them
        G.Moe.dispatch([moe], [x], [idx])
        G.Moe.combine([moe], [w], [out])
        torch.cuda.synchronize()
        s = torch.cuda.Stream()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            G.Moe.dispatch([moe], [x], [idx], stream=s)
            G.Moe.combine([moe], [w], [out], stream=s)
        out.zero_()
        torch.cuda.synchronize()
        dist.barrier()
        for it in range(iters - 1):
            g.replay()
    else:
        for it in range(iters):  # back to back on one stream: no host sync between steps
            G.Moe.dispatch([moe], [x], [idx])
            G.Moe.combine([moe], [w], [out])
    torch.cuda.synchronize()
    comm.check_device()
    got = out.cpu().numpy().view(np.uint16).reshape(T, H)
    exp, _ = O.combine(seed, E, K, H, rank, T, mode=mode)
    res["combine_exact"] = bool((got == exp).all())
    cnt = O.counts(seed, world, E, K, T)
    sig, _ = comm.snapshot_cells(512, 256)
    e_local = E // world
    res["cells_exact"] = all(sig[e] == iters * ((world << 32) + int(cnt[rank * e_local + e].sum()))
                             for e in range(e_local)) and sig[e_local] == iters * T * K
    if mode in (0, 1) and T >= 1024:
        # every dispatch message and combine record against the oracle's
        # digests (the bench's own check; the dedup transport ends in layout
        # 1's windows)
        dmsg, cmsg = 2 * H + 16, 2 * H
        lay = 1 if layout == 2 else layout
        slots = world * T * K if lay == 1 else (E // world) * world * T
        dd = torch.empty(slots, dtype=torch.int64, device=dev)
        cd = torch.empty(T * K, dtype=torch.int64, device=dev)
        G.digest(comm.window_ptr(moe.win_dispatch, rank), dmsg, slots, dd)
        G.digest(comm.window_ptr(moe.win_combine, rank), cmsg, T * K, cd)
        torch.cuda.synchronize()
        d, v, cdig = O.window_digests(seed, world, E, K, T, H, rank, mode=mode, layout=lay)
        res["dispatch_digests_exact"] = bool((dd.cpu().numpy().view("<u8")[v] == d[v]).all())
        res["combine_digests_exact"] = bool((cd.cpu().numpy().view("<u8") == cdig).all())
    if layout != 0 and T <= 4096 and mode in (0, 1):
        # compact window (layouts 1 and 2): every message of a sample carries
        # its source's token row byte for byte and the reference meta
        from tests import gpu_util as U
        dmsg = 2 * H + 16
        e_local = E // world
        win = comm.window_ptr(moe.win_dispatch, rank)
        rng = np.random.default_rng(rank)
        ok = True
        for src in range(world):
            total = int(cnt[rank * e_local:(rank + 1) * e_local, src].sum())
            xs = O.tokens(seed, src, T, H, mode=mode)
            for q in rng.choice(total, size=min(48, total), replace=False) if total else []:
                off = (src * T * K + int(q)) * dmsg
                msg = U.d2h(win + off, dmsg) if isinstance(win, int) else None
                meta = msg[2 * H:].view("<u4")
                ok &= bool(meta[0] == src and meta[3] == meta[2] + 1)
                ok &= bool((msg[:2 * H].view("<u2") == xs[int(meta[1])]).all())
        res["compact_sample_exact"] = ok
    if layout == 0 and T <= 256:
        from tests import gpu_util as U
        d, comb, _ = O.moe_rank_state(seed, world, E, K, T, H, rank, mode=mode)
        win = U.d2h(comm.window_ptr(moe.win_dispatch, rank), len(d))
        res["dispatch_window_exact"] = bool((win == d).all())
        cwin = U.d2h(comm.window_ptr(moe.win_combine, rank), len(comb))
        res["combine_window_exact"] = bool((cwin == comb).all())
    # BarrierSession: dissemination over signal cells and, where the box has
    # NVLink SHARP, the multicast barrier -- both must complete every round
    if os.environ.get("MP_BARRIER", "0") == "1":
        ns = torch.zeros(500, dtype=torch.int64, device=dev)
        res["nvls_enabled"] = comm.nvls_enabled()
        for mode in (0, 1) if res["nvls_enabled"] else (0,):
            for _ in range(2):  # rounds continue across calls
                G.check(G.lib().ginsim_cuda_barrier_bench(G.comm_handles([comm]), 1, mode, 500, ns.data_ptr(), None))
                torch.cuda.synchronize()
                comm.check_device()
            res[f"barrier_mode{mode}_p50_ns"] = int(np.sort(ns.cpu().numpy())[250])
        # the ring (harness_ring.cpp:18-57) across processes: its world-team
        # BarrierSession runs on the NVLS multicast cells where they exist
        S = 4096
        sb, rb = comm.mem_alloc(world * S), comm.mem_alloc(world * S)
        ws_, wr_ = comm.window_register(sb, world * S), comm.window_register(rb, world * S)
        dist.barrier()
        for _ in range(2):
            # (team 0 = world; signal cell 300: cells from 0 up belong to the MoE handle above)
            G.check(G.lib().ginsim_cuda_team_ring(G.comm_handles([comm]), 1, 0, ws_, wr_, S, 20, 300, None))
            comm.check_device()
            dist.barrier()
        res["ring_ok"] = True
        if res["nvls_enabled"]:
            # multicast signal broadcast: every rank adds rank+1 to cell 7 of
            # every rank with one multimem.red
            comm.signal_broadcast(7, rank + 1)
            torch.cuda.synchronize()
            want = world * (world + 1) // 2
            import time
            t0 = time.time()
            while comm.read_broadcast(7) < want and time.time() - t0 < 10:
                time.sleep(0.001)
            res["broadcast_cell"] = comm.read_broadcast(7)
            res["broadcast_expected"] = want
    # put+signal ping-pong over NVLink between ranks 0 and 1 (K14)
    if world >= 2 and os.environ.get("MP_PINGPONG", "1") == "1":
        size = 1 << 22
        sbuf = comm.mem_alloc(size)
        rbuf = comm.mem_alloc(size)
        ws = comm.window_register(sbuf, size)
        wr = comm.window_register(rbuf, size)
        rows = []
        rtt = torch.zeros(1000, dtype=torch.int64, device=dev)
        for sz in [8, 64, 512, 4096, 32768, 262144, 1 << 20, 1 << 22]:
            iters = 1000 if sz <= 65536 else 200
            if rank in (0, 1):
                G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles([comm]), 1, 0, 1, ws, wr, sz, iters, 100, 401, 512,
                                                     rtt.data_ptr(), None))
            dist.barrier()
            if rank == 0:
                t = np.sort(rtt[:iters].cpu().numpy())
                rows.append({"size": sz, "iters": iters, "p50_ns": int(t[iters // 2]),
                             "p99_ns": int(t[min(iters - 1, iters * 99 // 100)]), "mean_ns": float(t.mean())})
        res["pingpong"] = rows
    dist.barrier()
    out_dir = os.environ.get("MP_OUT")
    if out_dir:
        with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as f:
            json.dump(res, f)
    print("MPRESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
