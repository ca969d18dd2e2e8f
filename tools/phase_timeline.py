"""Per-phase timeline of the HT dispatch/combine kernels from in-kernel
%globaltimer stamps (GINSIM_PROFILE_PHASES=1).  One JSON line per rank:
for each kernel, per phase, the median and max over CTAs of the phase's
duration, and the spread of CTA start/end times (tail effects).

  python tools/phase_timeline.py                         # N=1
  TL_RANKS=8 TL_MODE=0 python tools/phase_timeline.py    # the bench's N=1 config: 8 emulated ranks
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
    R = int(os.environ.get("TL_RANKS", 1))  # emulated ranks on this GPU (world == 1 only)
    mode = int(os.environ.get("TL_MODE", 1))
    cfg = G.MoeConfig(E, K, T, H, mode, int(os.environ.get("TL_LAYOUT", 1)), int(os.environ.get("TL_CTAS", 0)), 0)
    if world > 1:
        comms = [comm]
        moes = [G.Moe(comm, cfg)]
    else:
        comms = G.Comm.create_all([0] * R, G.Config(signal_cells=512))
        moes = G.Moe.create_all(comms, cfg) if R > 1 else [G.Moe(comms[0], cfg)]
    dev = torch.device("cuda", local)
    xs = [torch.empty(T * H, dtype=torch.int16, device=dev) for _ in moes]
    idxs = [torch.empty(T * K, dtype=torch.int32, device=dev) for _ in moes]
    ws = [torch.empty(T * K, dtype=torch.float32 if mode == 1 else torch.int16, device=dev) for _ in moes]
    outs = [torch.empty(T * H, dtype=torch.int16, device=dev) for _ in moes]
    for c, m, x, i, w in zip(comms, moes, xs, idxs, ws):
        m.generate(1, (c.rank + int(os.environ.get("TL_SHIFT", 0))) % max(world, R), x, i, w)
    for _ in range(4):
        G.Moe.dispatch(moes, xs, idxs)
        G.Moe.combine(moes, ws, outs)
    torch.cuda.synchronize()
    moe = moes[0]
    res = {"rank": rank, "world": world, "tokens": T}
    for kern in (0, 1, 2):
        st = moe.phase_times(kern).astype(np.int64)
        st = st[st[:, 0] > 0]  # CTAs that ran (the pipelined combine's send kernel leaves SMs to the reducer)
        if st.shape[0] == 0:  # kernel not launched (LL: reduce fused into the send)
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
