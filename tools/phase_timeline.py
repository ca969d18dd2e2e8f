"""Per-phase timeline of the HT dispatch/combine kernels from in-kernel
%globaltimer stamps (GINSIM_PROFILE_PHASES=1).  One JSON line per rank:
for each kernel, per phase, the median and max over CTAs of the phase's
duration, and the spread of CTA start/end times (tail effects).

  python tools/phase_timeline.py                         # N=1
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/phase_timeline.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["GINSIM_PROFILE_PHASES"] = "1"

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402

NAMES = {0: ["own_hist", "bar1+col_scan", "bar2+slots", "bar3", "puts", "release", "fanout(L2)/acquire"], 1: ["counts_scan", "transform_puts", "flag_release"],
         2: ["flag_acquire", "reduce"]}


def summarize(st):
    t0 = st[:, 0].min()
    out = {"ctas": int(st.shape[0]), "start_spread_us": float((st[:, 0].max() - t0) / 1e3)}
    nz = [i for i in range(8) if (st[:, i] > 0).all()]
    last = max(nz)
    out["kernel_us"] = float((st[:, last].max() - t0) / 1e3)
    out["end_spread_us"] = float((st[:, last].max() - st[:, last].min()) / 1e3)
    return out, nz


def main():
    T, H, K, E = int(os.environ.get("TL_TOKENS", 4096)), 7168, 8, 256
    if "RANK" in os.environ:
        rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
        torch.cuda.set_device(local)
        dist.init_process_group("gloo")

        def ag(blob):
            o = [None] * world
            dist.all_gather_object(o, blob)
            return o
        comm = G.Comm.create(rank, world, local, ag, G.Config(signal_cells=512))
    else:
        rank, world, local = 0, 1, 0
        comm = G.Comm.create_all([0], G.Config(signal_cells=512))[0]
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, int(os.environ.get("TL_MODE", 1)), int(os.environ.get("TL_LAYOUT", 1)), 0, 0))
    dev = torch.device("cuda", local)
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(1, (rank + int(os.environ.get("TL_SHIFT", 0))) % world, x, idx, w)
    for _ in range(4):
        G.Moe.dispatch([moe], [x], [idx])
        G.Moe.combine([moe], [w], [out])
    torch.cuda.synchronize()
    res = {"rank": rank, "world": world, "tokens": T}
    for kern in (0, 1, 2):
        st = moe.phase_times(kern).astype(np.int64)
        if not (st[:, 0] > 0).all():  # kernel not launched (LL: reduce fused into the send)
            continue
        summ, nz = summarize(st)
        phases = {}
        for a, b in zip(nz[:-1], nz[1:]):
            d = (st[:, b] - st[:, a]) / 1e3
            phases[NAMES[kern][a] if a < len(NAMES[kern]) else f"p{a}"] = {
                "median_us": float(np.median(d)), "max_us": float(d.max())}
        summ["phases"] = phases
        res[["dispatch", "combine_send", "combine_reduce"][kern]] = summ
    print(json.dumps(res), flush=True)
    if world > 1:
        dist.barrier()


def print_logs(paths):
    """python tools/phase_timeline.py --print gpurun_out/tl_n*.log"""
    for path in paths:
        for line in open(path):
            if not line.startswith("{"):
                continue
            d = json.loads(line)
            print(f"rank {d['rank']}/{d['world']}")
            for k in ("dispatch", "combine_send", "combine_reduce"):
                if k not in d:
                    continue
                head = {a: (round(b, 1) if isinstance(b, float) else b) for a, b in d[k].items() if a != "phases"}
                print("  ", k, head)
                for p, v in d[k]["phases"].items():
                    print("      ", p, {a: round(b, 1) for a, b in v.items()})


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--print":
        print_logs(sys.argv[2:])
    else:
        main()
