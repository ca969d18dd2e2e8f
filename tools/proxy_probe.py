"""Proxy-backend diagnostics: per-step time and agent statistics of MoE
dispatch/combine over the proxy backend at a given token count, one process
per GPU (torchrun) or N emulated ranks on one GPU (no torchrun).
  PROBE_TOKENS=128 python -m torch.distributed.run --nproc-per-node 2 tools/proxy_probe.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def main():
    T = int(os.environ.get("PROBE_TOKENS", "128"))
    steps = int(os.environ.get("PROBE_STEPS", "3"))
    H, K, E = 7168, 8, 256
    if "RANK" in os.environ:
        rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")

        def ag(blob):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out
        comms = [G.Comm.create(rank, world, local, ag, G.Config(backend="proxy", signal_cells=512, timeout_ms=15000))]
        moes = [G.Moe(comms[0], G.MoeConfig(E, K, T, H, 1, 1, 0, 0))]
        ranks = [rank]
    else:
        world = int(os.environ.get("PROBE_RANKS", "2"))
        rank = 0
        comms = G.Comm.create_all([0] * world, G.Config(backend="proxy", signal_cells=512, timeout_ms=15000))
        moes = G.Moe.create_all(comms, G.MoeConfig(E, K, T, H, 1, 1, 0, 0))
        ranks = list(range(world))
    dev = torch.device("cuda", torch.cuda.current_device())
    bufs = []
    for m, r in zip(moes, ranks):
        x = torch.empty(T * H, dtype=torch.int16, device=dev)
        idx = torch.empty(T * K, dtype=torch.int32, device=dev)
        w = torch.empty(T * K, dtype=torch.float32, device=dev)
        out = torch.empty(T * H, dtype=torch.int16, device=dev)
        m.generate(1, r, x, idx, w)
        bufs.append((x, idx, w, out))
    torch.cuda.synchronize()
    rows = []
    for s in range(steps):
        st0 = comms[0].proxy_stats()
        t0 = time.time()
        G.Moe.dispatch(moes, [b[0] for b in bufs], [b[1] for b in bufs])
        torch.cuda.synchronize()
        t1 = time.time()
        G.Moe.combine(moes, [b[2] for b in bufs], [b[3] for b in bufs])
        torch.cuda.synchronize()
        t2 = time.time()
        st1 = comms[0].proxy_stats()
        err = [c.device_error(clear=False) for c in comms]
        rows.append({"step": s, "dispatch_ms": (t1 - t0) * 1e3, "combine_ms": (t2 - t1) * 1e3,
                     "descriptors": st1["descriptors"] - st0["descriptors"], "copies": st1["copies"] - st0["copies"],
                     "busy_frac": (st1["busy_ns"] - st0["busy_ns"]) / max(1, st1["wall_ns"] - st0["wall_ns"]),
                     "device_error": err})
        print(json.dumps({"rank": rank, "T": T, **rows[-1]}), flush=True)
        if any(err):
            break
    if "RANK" in os.environ:
        dist.barrier()


if __name__ == "__main__":
    main()
