#!/usr/bin/env python3
"""bench.py — DeepEP-style MoE dispatch+combine over the B200 GIN path.

Workload (BASELINE.json configs[3], the metric's "at 8xB200" config):
high-throughput dispatch/combine, 8 ranks x 4096 tokens per rank, hidden 7168,
top-8 of 256 experts, in the reference's own u16 arithmetic (so both arms
compute the identical function, bit for bit).
  * --gpus 1: the 8 ranks are emulated on the one GPU (every rank's windows in
    its HBM, one cooperative launch per phase with blockIdx.y = rank), so the
    whole 8-rank protocol runs and the path is HBM-bound.
  * --gpus N (torchrun): one rank per GPU, N ranks x 4096 tokens; the remote
    share crosses NVLink 5 peer mappings.
A step = one dispatch (route + puts + per-expert releases) and one combine
(expert transform fused into the return puts + flag wait + top-k weighted
reduce) over one batch of synthetic tokens already in HBM.  After the timed
region the measured state is checked against the CPU oracle (outputs and
every window record); `e2e` repeats the step through the public API with
host buffers and the copies inside the timed region.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
--impl reference runs the unmodified reference (oracle/_ref) on the same
workload (a bounded token sample per step, stated in the line) on the host.
Prints one JSON line on rank 0.
"""
from __future__ import annotations

import os as _os
# every stream its own hardware queue: a proxy-agent stream aliased onto the queue of
# a kernel that waits for the agent would stall behind it (csrc/proxy.cu)
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE dispatch+combine µs & GB/s/GPU at 8×B200; put+signal latency vs msg size"
N_TOK, HIDDEN, TOPK, EXPERTS = 4096, 7168, 8, 256


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--tokens", type=int, default=N_TOK)
    p.add_argument("--mode", type=int, default=0, help="0 = u16 exact (the reference's arithmetic), 1 = bf16")
    p.add_argument("--ranks", type=int, default=0, help="ranks per process (0 = 8 emulated at --gpus 1, else 1)")
    p.add_argument("--no-verify", action="store_true", help="skip the post-run parity check against the oracle")
    p.add_argument("--layout", type=int, default=-1,
                   help="0 = reference layout, 1 = compact, 2 = compact + dedup transport; "
                        "-1 = auto (1 at --gpus 1, where 8 emulated ranks share HBM; 2 over NVLink). "
                        "Layouts 1 and 2 end in bit-identical windows and cells.")
    p.add_argument("--ctas", type=int, default=0)
    p.add_argument("--engine", type=int, default=0, help="0 = auto (TMA), 1 = LSU stores, 2 = TMA")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the LL and ping-pong sub-measurements")
    p.add_argument("--csv", default="", help="prefix: write ping-pong / bw rows in the reference's CSV schema")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk.get("hbm_gbs", 6650.0), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc = gpu, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
        self.t.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# --------------------------------------------------------------------- workload (both arms)
UNIT = "GB/s (dispatch+combine message bytes, all ranks)"


def ranks_per_process(args, world):
    """Ranks this process drives: at N=1 the BASELINE 8-rank HT config runs as 8
    emulated ranks on the one GPU (one cooperative launch, blockIdx.y = rank);
    under torchrun one rank per GPU."""
    if args.ranks:
        return args.ranks
    return 8 if world == 1 else 1


def workload(R, T, H=HIDDEN, K=TOPK, E=EXPERTS, mode=0):
    arith = {0: "u16 reference arithmetic", 1: "bf16"}.get(mode, f"mode {mode}")
    return f"DeepEP HT dispatch+combine: {R} ranks x {T} tokens/rank, hidden {H}, top-{K} of {E} experts, {arith}"


def step_bytes(R, T, H=HIDDEN, K=TOPK):
    """Algorithmic bytes of one step: every (token, k) message once each way."""
    return R * T * K * ((2 * H + 16) + 2 * H)


# --------------------------------------------------------------------- reference arm
def mem_available():
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(R, T_max, steps, warmup, budget_s):
    """The reference's own CPU implementation (oracle/_ref: ginsim compiled
    from /root/reference by oracle/build_ref.sh) through its public harness
    run_moe_ll (harness_moe.cpp:252) with R in-process ranks (2 host threads
    each), hidden 7168, top-8 of 256, seed 1.  Each step is one run_moe_ll
    call on a bounded sample of T_ref tokens per rank: the reference sizes
    its receive windows for the worst case (T*(E+K)*(dmsg+cmsg) bytes per
    rank, harness_moe.cpp:122-125), so T_ref is the largest power of two
    <= T_max that fits 60% of MemAvailable and the time budget (from an
    untimed calibration run at 128 tokens).  Throughput counts the same
    message bytes as the GPU arm."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    H, K, E = HIDDEN, TOPK, EXPERTS
    per_token = R * (E + K) * ((2 * H + 16) + 2 * H)
    mem = mem_available()

    def once(T):
        j = O.ref_run("moe-ll", "--ranks", R, "--experts", E, "--topk", K, "--tokens", T, "--hidden", H,
                      "--seed", 1, "--backend", "direct", timeout=1800)
        return j["best_s"]

    t0 = min(128, T_max)
    probe = once(t0)  # calibration (counts as the first warm-up run)
    runs_left = steps + max(0, warmup - 1)
    s_tok = probe / t0
    T = T_max
    while T > t0 and (T * per_token > 0.6 * mem or runs_left * s_tok * T > budget_s):
        T //= 2
    for _ in range(max(0, warmup - 1)):
        once(T)
    times = [once(T) for _ in range(steps)]
    mean = sum(times) / len(times)
    return {"value": step_bytes(R, T) / mean / 1e9, "s_per_step": mean, "tokens": T, "cores": min(2 * R, os.cpu_count() or 1),
            "mem_available_gb": round(mem / 2**30, 1), "calibration_s": probe,
            "sample": f"reference run_moe_ll (harness_moe.cpp:252) per step: {R} in-process ranks x 2 host threads, "
                      f"{T} tokens/rank (largest power of two <= {T_max} fitting 60% of MemAvailable "
                      f"{mem / 2**30:.0f} GiB and a {budget_s:.0f} s budget), hidden {H}, top-{K} of {E}, "
                      f"u16, verification included; mean of {len(times)} after {warmup} warm-up"}


def reference_main(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    R = world * ranks_per_process(args, world)
    budget = float(os.environ.get("GINSIM_REF_BUDGET_S", "240"))
    r = run_reference(R, args.tokens, args.steps, args.warmup, budget)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built (reference sources absent)"}))
        return
    line = {"impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["s_per_step"] * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u16", "data": "synthetic",
            "config": {"workload": workload(R, args.tokens), "ranks": R, "tokens_per_rank": args.tokens,
                       "sample_tokens_per_rank": r["tokens"], "hidden": HIDDEN, "top_k": TOPK, "experts": EXPERTS,
                       "device": "host CPU only (the reference has no GPU code)"},
            "host": {"nproc": os.cpu_count(), "cpu_model": cpu_model(), "mem_available_gb": r["mem_available_gb"]},
            "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# --------------------------------------------------------------------- secondary configs
def measure_ll(G, comm, rank, world, dist, torch, dev, stream, steps=50):
    """BASELINE configs[2]: LL dispatch/combine, 128 tokens/rank, hidden 7168,
    top-8 of 256, bf16 — per-phase device time (max over ranks), µs."""
    T, H, K, E = 128, HIDDEN, TOPK, EXPERTS
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 1, 0, 0, 0))
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(1, rank, x, idx, w, stream=stream)
    for _ in range(5):
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(stream)
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        ev[i][1].record(stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    comm.check_device()
    d = sorted(e[0].elapsed_time(e[1]) for e in ev)
    c = sorted(e[1].elapsed_time(e[2]) for e in ev)
    t = torch.tensor([d[len(d) // 2], c[len(c) // 2]], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dmsg, cmsg = 2 * H + 16, 2 * H
    disp_us, comb_us = t[0].item() * 1e3, t[1].item() * 1e3
    # the same step captured once in a CUDA graph (the kernels read their
    # iteration from device counters, so every replay is a full step): what a
    # serving loop pays per step without per-launch host overhead
    graph_us = None
    try:
        gs = torch.cuda.Stream(device=dev)
        gs.wait_stream(stream)
        gph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gph, stream=gs):
            G.Moe.dispatch([moe], [x], [idx], stream=gs)
            G.Moe.combine([moe], [w], [out], stream=gs)
        torch.cuda.synchronize()
        with torch.cuda.stream(gs):  # replay() launches on the current stream
            for _ in range(5):
                gph.replay()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        gev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        with torch.cuda.stream(gs):
            for e0, e1 in gev:
                e0.record(gs)
                gph.replay()
                e1.record(gs)
        torch.cuda.synchronize()
        comm.check_device()
        gt = sorted(e0.elapsed_time(e1) for e0, e1 in gev)
        tg = torch.tensor([gt[len(gt) // 2]], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tg, op=dist.ReduceOp.MAX)
        graph_us = tg.item() * 1e3
    except Exception as e:  # noqa: BLE001
        graph_us = f"unavailable: {str(e)[:120]}"
    return {"workload": f"DeepEP LL dispatch/combine, {T} tokens/rank, hidden {H}, top-{K} of {E}, bf16, {world} GPU(s)",
            "dispatch_us_p50": disp_us, "combine_us_p50": comb_us,
            "dispatch_GBps_per_gpu": T * K * dmsg / (disp_us * 1e-6) / 1e9,
            "combine_GBps_per_gpu": T * K * cmsg / (comb_us * 1e-6) / 1e9,
            "step_us_p50_cuda_graph": graph_us,
            "paper_h100_reference_us": {"dispatch": 40.62, "combine": 69.0}}


def measure_pingpong(G, comm, rank, world, dist, torch, dev):
    """BASELINE configs[0] on hardware: put+SignalInc ping-pong between ranks 0
    and 1 over NVLink (harness_bench.cpp:47-90), 8 B .. 4 MiB, %globaltimer
    inside one persistent kernel; zero-byte put+signal = the raw release/
    acquire round-trip floor."""
    import ctypes  # noqa: F401
    import numpy as np
    size_max = 4 << 20
    sb, rb = comm.mem_alloc(size_max), comm.mem_alloc(size_max)
    ws, wr = comm.window_register(sb, size_max), comm.window_register(rb, size_max)
    rtt = torch.zeros(1000, dtype=torch.int64, device=dev)
    rows = []
    for sz in [0, 8, 64, 512, 4096, 32768, 262144, 1 << 20, 4 << 20]:
        iters = 1000 if sz <= 65536 else 200
        if rank in (0, 1):
            G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles([comm]), 1, 0, 1, ws, wr, sz, iters, 100, 4001, 0,
                                                 rtt.data_ptr(), None))
        dist.barrier()
        if rank == 0:
            row = G.summarize(sz, rtt[:iters].cpu().numpy())  # harness_bench.cpp:20-32
            row["one_way_ns"] = row["p50_ns"] / 2
            row["GBps_per_direction"] = (2 * sz / (row["p50_ns"] * 1e-9) / 1e9) if sz else None
            rows.append(row)
    # worst-pair scan: 8-byte put+signal RTT between every pair
    pairs = []
    if world > 2:
        for a in range(world):
            for b in range(a + 1, world):
                if rank in (a, b):
                    G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles([comm]), 1, a, b, ws, wr, 8, 500, 50, 4001, 0,
                                                         rtt.data_ptr(), None))
                dist.barrier()
                t = torch.tensor([float(np.sort(rtt[:500].cpu().numpy())[250]) if rank == a else 0.0],
                                 dtype=torch.float64, device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                pairs.append({"pair": [a, b], "p50_ns": int(t.item())})
    # the raw NVLink round trip with no API: one thread per
    # rank flips a flag word in the peer's signal table (cells 4010/4011)
    floor = {}
    for mode, name in ((0, "release_acquire"), (1, "relaxed"), (2, "release_relaxed_poll_fence"),
                       (3, "release_add_relaxed_poll_fence")):
        if rank in (0, 1):
            G.check(G.lib().ginsim_cuda_rtt_floor(G.comm_handles([comm]), 1, 0, 1, mode, 1000, 100, 4010,
                                                  rtt.data_ptr(), None))
        dist.barrier()
        if rank == 0:
            t = np.sort(rtt[:1000].cpu().numpy())
            floor[name] = {"p50_ns": int(t[500]), "p99_ns": int(t[990]), "mean_ns": float(t.mean())}
    if rows:  # each size against the raw round-trip floor and, for bandwidth, against 900 GB/s
        f0 = floor.get("release_acquire", {}).get("p50_ns") or rows[0]["p50_ns"]
        for r in rows:
            r["x_rtt_floor"] = r["p50_ns"] / f0
            r["frac_of_900"] = r["GBps_per_direction"] / 900.0 if r["GBps_per_direction"] else None
    return {"rows": rows, "target_us": 5.0, "target_metric": "RTT p50 of an 8-byte put+SignalInc (the paper's metric, "
            "PAPER.md:952-958); one-way = RTT/2", "raw_floor": floor,
            "floor_ns": floor.get("release_acquire", {}).get("p50_ns"),
            "pair_scan_8B": pairs or None,
            "worst_pair_8B": max(pairs, key=lambda r: r["p50_ns"]) if pairs else None,
            "csv_schema": "size_bytes,iters,p50_ns,p99_ns,mean_ns,backend=direct,transport=nvlink"}


def measure_bw(G, comm, rank, world, dist, torch, dev, window=16):
    """bw_rank_program (harness_bench.cpp:92-129) on hardware: rank 0 puts
    `window` messages into rank 1's window, then flushes; per-iteration time
    (p50/p99/mean, the reference's summarize) and GB/s = window*size/p50."""
    sizes = [4 << 10, 32 << 10, 256 << 10, 2 << 20, 4 << 20]
    smax = sizes[-1]
    sb, rb = comm.mem_alloc(smax), comm.mem_alloc(window * smax)
    ws = comm.window_register(sb, smax)
    wr = comm.window_register(rb, window * smax)
    ns = torch.zeros(200, dtype=torch.int64, device=dev)
    rows = []
    for sz in sizes:
        iters = 200 if sz <= (256 << 10) else 50
        dist.barrier()
        if rank == 0:
            G.check(G.lib().ginsim_cuda_bw(G.comm_handles([comm]), 1, 0, 1, ws, wr, sz, window, iters, 10, 0,
                                           ns.data_ptr(), None))
            row = G.summarize(sz, ns[:iters].cpu().numpy())
            row["GBps"] = window * sz / (row["p50_ns"] * 1e-9) / 1e9
            row["frac_of_900"] = row["GBps"] / 900.0
            rows.append(row)
    dist.barrier()
    comm.check_device()
    return {"workload": f"windowed put bandwidth, {window} puts + flush per iteration, rank 0 -> 1", "rows": rows}


def measure_a2a(G, comm, rank, world, dist, torch, dev, stream):
    """BASELINE configs[1]: one-sided all-to-all via put+signal on registered
    windows (K15): every rank puts M bytes to each of the
    n-1 peers at recv[src*M] and releases one SignalInc per peer, then waits
    for n-1 arrivals.  Per-GPU egress = (n-1)*M / time (max over ranks)."""
    sizes = [1 << 10, 4 << 10, 16 << 10, 64 << 10, 256 << 10, 1 << 20, 4 << 20, 16 << 20, 64 << 20]
    cap = world * sizes[-1]
    sb, rb = comm.mem_alloc(cap), comm.mem_alloc(cap)
    ws, wr = comm.window_register(sb, cap), comm.window_register(rb, cap)
    # (every MoE handle on this comm owns e_local + 7 cells from 0 up; the
    # headline, LL and variant handles stay far below)
    sid = 4000  # below the barrier slots; the ping-pong uses 4001/4002
    h = G.comm_handles([comm])
    rows = []
    for M in sizes:
        iters = 50 if M <= (1 << 20) else 10
        base = comm.read_signal(sid)
        dist.barrier()  # every rank holds its base before any rank's first put of this size
        k = 0

        def once():
            nonlocal k
            k += 1
            G.check(G.lib().ginsim_cuda_alltoall(h, 1, ws, wr, M, sid, base + (world - 1) * k, 0,
                                                 ctypes_stream(stream)))
        for _ in range(3):
            once()
        torch.cuda.synchronize()
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(iters):
            once()
        s1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([s0.elapsed_time(s1) / iters], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = t.item() * 1e3
        gbps = (world - 1) * M / (us * 1e-6) / 1e9
        rows.append({"bytes_per_peer": M, "iters": iters, "us": us, "egress_GBps_per_gpu": gbps,
                     "frac_of_900": gbps / 900.0, "frac_of_measured_770": gbps / 770.0})
    comm.check_device()
    return {"workload": f"one-sided all-to-all put+signal, {world} GPUs, 1 KiB..64 MiB per peer", "rows": rows}


def measure_proxy(G, rank, world, local, dist, torch, dev, stream, allgather, T, steps):
    """BASELINE configs[4]: the Proxy backend (GPU -> pinned-host 64-B
    descriptor rings -> host agent thread -> cudaMemcpyAsync + stream-memop
    signals) on the same dispatch/combine workload as the
    direct path: per-phase device time (max over ranks), descriptors/s and
    the agent thread's busy fraction."""
    H, K, E = HIDDEN, TOPK, EXPERTS
    cfg = G.Config(backend="proxy", signal_cells=512)
    comm = (G.Comm.create(rank, world, local, allgather, cfg) if world > 1
            else G.Comm.create_all([local], cfg)[0])
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 1, 1, 0, 0))
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(1, rank, x, idx, w, stream=stream)
    for _ in range(2):
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    st0 = comm.proxy_stats()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(stream)
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        ev[i][1].record(stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    st1 = comm.proxy_stats()
    comm.check_device()
    d = sorted(e[0].elapsed_time(e[1]) for e in ev)
    c = sorted(e[1].elapsed_time(e[2]) for e in ev)
    tot = sum(e[0].elapsed_time(e[2]) for e in ev)
    t = torch.tensor([d[len(d) // 2], c[len(c) // 2], tot], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ndesc = st1["descriptors"] - st0["descriptors"]
    ncopy = st1["copies"] - st0["copies"]
    busy = (st1["busy_ns"] - st0["busy_ns"]) / max(1, st1["wall_ns"] - st0["wall_ns"])
    dmsg, cmsg = 2 * H + 16, 2 * H
    disp_us, comb_us = t[0].item() * 1e3, t[1].item() * 1e3
    remote = int(((idx.cpu().numpy().reshape(T, K) // (E // world)) != rank).sum())
    pipe = moe.pipelined()
    res = {"workload": f"proxy backend dispatch/combine, {T} tokens/rank, hidden {H}, top-{K} of {E}, bf16, "
                       f"{world} GPU(s), " + ("pipelined: staged chunks handed to the copy engines as they fill"
                                             if pipe else "one copy-engine put per destination after the staging kernel"),
           "transport": "pipeline" if pipe else "one-shot",
           "dispatch_us_p50": disp_us, "combine_us_p50": comb_us,
           "dispatch_GBps_per_gpu": T * K * dmsg / (disp_us * 1e-6) / 1e9,
           "combine_GBps_per_gpu": T * K * cmsg / (comb_us * 1e-6) / 1e9,
           "dispatch_remote_GBps_per_gpu": remote * dmsg / (disp_us * 1e-6) / 1e9,
           "dispatch_remote_frac_of_900": remote * dmsg / (disp_us * 1e-6) / 1e9 / 900.0,
           "descriptors_per_step": ndesc / steps, "copies_per_step": ncopy / steps,
           "descriptors_per_s": ndesc / (t[2].item() * 1e-3), "agent_thread_busy_frac": busy,
           "host_threads": 1}
    moe.destroy()
    comm.destroy()
    return res


def measure_barrier(G, comm, rank, world, dist, torch, dev, iters=2000):
    """BarrierSession latency (runtime.cpp:638-666), one thread per rank, p50
    over back-to-back barriers timed with %globaltimer: the reference's
    dissemination barrier (ceil(log2 n) rounds of signals) vs the NVLS
    multicast barrier (one multimem.red arrival)."""
    import numpy as np
    out = {"workload": f"barrier latency, {world} GPUs, {iters} back-to-back barriers", "nvls_enabled": comm.nvls_enabled()}
    ns = torch.zeros(iters, dtype=torch.int64, device=dev)
    for mode, name in ((0, "dissemination"), (1, "nvls")):
        if mode == 1 and not out["nvls_enabled"]:
            continue
        dist.barrier()
        G.check(G.lib().ginsim_cuda_barrier_bench(G.comm_handles([comm]), 1, mode, iters, ns.data_ptr(), None))
        torch.cuda.synchronize()
        comm.check_device()
        t = np.sort(ns.cpu().numpy()[100:])
        out[name] = {"p50_ns": int(t[len(t) // 2]), "p99_ns": int(t[len(t) * 99 // 100]), "mean_ns": float(t.mean())}
    return out


def measure_overlap(G, comm, rank, world, dist, torch, dev, T, ctas=74, steps=6):
    """Co-residency: the HT dispatch+combine step on `ctas` CTAs per rank (half
    the GPU; at N=2 that costs nothing, profiles/r2_ctas_sweep_n2.json) next to
    a bf16 GEMM stream on a second CUDA stream.  Reports each alone and both
    together (device time of the joint region, max over ranks)."""
    H, K, E = HIDDEN, TOPK, EXPERTS
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, 0, 1, ctas, 0))
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.int16, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(1, rank, x, idx, w)
    a = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    bm = torch.randn(8192, 8192, dtype=torch.bfloat16, device=dev)
    cm = torch.empty(8192, 8192, dtype=torch.bfloat16, device=dev)
    s_moe, s_mm = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)

    def moe_steps():
        for _ in range(steps):
            G.Moe.dispatch([moe], [x], [idx], stream=s_moe)
            G.Moe.combine([moe], [w], [out], stream=s_moe)

    def gemms(nm):
        with torch.cuda.stream(s_mm):
            for _ in range(nm):
                torch.matmul(a, bm, out=cm)

    def timed(fn_moe, fn_mm):
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s_moe)
        s_mm.wait_event(e0)
        if fn_moe:
            fn_moe()
        if fn_mm:
            fn_mm()
        s_moe.wait_stream(s_mm)
        e1.record(s_moe)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    moe_steps()
    gemms(2)
    torch.cuda.synchronize()
    t_moe = timed(moe_steps, None)
    n_mm = max(1, int(round(t_moe / max(1e-3, timed(None, lambda: gemms(1))))))
    t_mm = timed(None, lambda: gemms(n_mm))
    t_both = timed(moe_steps, lambda: gemms(n_mm))
    comm.check_device()
    moe.destroy()
    return {"workload": f"{steps} HT dispatch+combine steps on {ctas} CTAs/rank ({T} tokens/rank, u16) next to "
                        f"{n_mm} bf16 8192^3 GEMMs on a second stream, {world} GPU(s)",
            "moe_alone_ms": t_moe, "gemm_alone_ms": t_mm, "both_ms": t_both,
            "overlap_gain": (t_moe + t_mm) / t_both if t_both else None}


def measure_variant(G, comm, rank, world, dist, torch, dev, stream, T, layout, mode, label, steps=10):
    """Labelled variants beside the headline (same windows/cells contract,
    tests/test_gpu_moe.py): layout 2 = the compact receive layout with a
    per-rank dedup transport (one NVLink row per (token,
    destination rank), fanned out into the expert slots by the destination);
    mode 2 = fp8 dispatch (e4m3 codes + per-128 fp32 scales, SURVEY §8f f3,
    the paper's LL format); mode 3 = fp8 dispatch and fp8 combine messages.
    Per-phase device time, max over ranks."""
    H, K, E = HIDDEN, TOPK, EXPERTS
    moe = G.Moe(comm, G.MoeConfig(E, K, T, H, mode, layout, 0, 0))
    x = torch.empty(T * H, dtype=torch.int16, device=dev)
    idx = torch.empty(T * K, dtype=torch.int32, device=dev)
    w = torch.empty(T * K, dtype=torch.float32, device=dev)
    out = torch.empty(T * H, dtype=torch.int16, device=dev)
    moe.generate(1, rank, x, idx, w, stream=stream)
    for _ in range(3):
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for i in range(steps):
        ev[i][0].record(stream)
        G.Moe.dispatch([moe], [x], [idx], stream=stream)
        ev[i][1].record(stream)
        G.Moe.combine([moe], [w], [out], stream=stream)
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    comm.check_device()
    d = sorted(e[0].elapsed_time(e[1]) for e in ev)[steps // 2]
    c = sorted(e[1].elapsed_time(e[2]) for e in ev)[steps // 2]
    t = torch.tensor([d, c], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ih = idx.cpu().numpy().reshape(T, K) // (E // world)
    rows_remote = sum(len(set(int(v) for v in row) - {rank}) for row in ih)
    msgs_remote = int((ih != rank).sum())
    dmsg = (H + H // 32 if mode >= 2 else 2 * H) + 16
    wire = rows_remote * (2 * H + 128) if layout == 2 else msgs_remote * dmsg
    disp_us = t[0].item() * 1e3
    moe.destroy()
    return {"workload": f"labelled variant: {label}, {T} tokens/rank, hidden {H}, top-{K} of {E}, {world} GPU(s)",
            "dispatch_us_p50": disp_us, "combine_us_p50": t[1].item() * 1e3,
            "remote_wire_bytes_per_rank": wire, "wire_GBps_per_gpu": wire / (disp_us * 1e-6) / 1e9}


def launches_per_step(args, world, R, T, K, E):
    """Kernels one step launches, mirroring the library's choice
    (csrc/kernels_moe.cu plan(): the pipelined combine runs with one rank per
    GPU over NVLink, cooperative route tables (T*K >= 8192 pairs) and C =
    min(GINSIM_COMBINE_CHUNKS or 4, 8, 1024 // E) >= 2 chunks)."""
    if args.engine not in (0, 2):
        return 2
    c = int(os.environ.get("GINSIM_COMBINE_CHUNKS") or 4)
    c = min(c, 8, 1024 // E)
    coop = T * K >= int(os.environ.get("GINSIM_DISPATCH_COOP_MIN_PAIRS") or 8192)
    early = os.environ.get("GINSIM_EARLY_RED_SMS", "64") != "0"
    return 4 if (world > 1 and R == 1 and coop and c >= 2 and early) else 3


def ctypes_stream(stream):
    return None if stream is None else stream.cuda_stream


# --------------------------------------------------------------------- parity self-check
def verify_step(G, torch, comms, moes, outs, seed, R_total, T, H, K, E, mode, layout, stream):
    """Checker (after the timed region; never timed): every output token of
    every local rank against the CPU oracle's combine (oracle/ginsim_oracle.c,
    pinned to the reference), and every dispatch-window message and
    combine-window record against the oracle's expected record digests
    (device digests: ginsim_cuda_digest).  Bit-exact in u16 mode; bf16 mode
    compares with the fp32-sequential oracle bit for bit as well."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import oracle as O
    dev = outs[0].device
    dmsg, cmsg = 2 * H + 16, 2 * H
    layout = 1 if layout == 2 else layout  # the dedup transport ends in layout 1's windows
    slots = (R_total * T * K) if layout == 1 else (E // R_total) * R_total * T
    got = []
    for c, m, o in zip(comms, moes, outs):
        dd = torch.empty(slots, dtype=torch.int64, device=dev)
        cd = torch.empty(T * K, dtype=torch.int64, device=dev)
        G.digest(c.window_ptr(m.win_dispatch, c.rank), dmsg, slots, dd, stream=stream)
        G.digest(c.window_ptr(m.win_combine, c.rank), cmsg, T * K, cd, stream=stream)
        got.append((dd, cd, o))
    torch.cuda.synchronize()

    def expect(r):
        exp, _ = O.combine(seed, E, K, H, r, T, mode=mode)
        d, v, cdig = O.window_digests(seed, R_total, E, K, T, H, r, mode=mode, layout=layout)
        return exp, d, v, cdig

    with ThreadPoolExecutor(max_workers=max(1, min(len(comms), os.cpu_count() or 1))) as ex:
        exps = list(ex.map(expect, [c.rank for c in comms]))
    ok_out = ok_disp = ok_comb = True
    msgs = 0
    for (dd, cd, o), (exp, d, v, cdig) in zip(got, exps):
        out = o.view(torch.int16).cpu().numpy().view("<u2").reshape(T, H)
        ok_out &= bool((out == exp).all())
        dh = dd.cpu().numpy().view("<u8")
        ok_disp &= bool((dh[v] == d[v]).all())
        msgs += int(v.sum())
        ok_comb &= bool((cd.cpu().numpy().view("<u8") == cdig).all())
    return {"outputs": ok_out, "dispatch_windows": ok_disp, "combine_windows": ok_comb,
            "ranks_checked": [c.rank for c in comms], "tokens_checked_per_rank": T,
            "dispatch_messages_checked": msgs, "combine_records_checked": len(comms) * T * K,
            "oracle": "oracle/ginsim_oracle.c (restatement pinned to the reference); records compared by digest",
            "exact": True}


# --------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        reference_main(args)
        return
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist

    import paper_2511_15076_b200 as G

    torch.cuda.set_device(local)
    R = ranks_per_process(args, world)
    if world > 1 and R != 1:
        raise SystemExit("bench.py: one rank per GPU under torchrun (--ranks applies to --gpus 1)")
    R_total = world * R
    cfg_comm = G.Config(signal_cells=4096)
    allgather = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

        def allgather(blob: bytes):
            out = [None] * world
            dist.all_gather_object(out, blob)
            return out
        comms = [G.Comm.create(rank, world, local, allgather, cfg_comm)]
    else:
        comms = G.Comm.create_all([local] * R, cfg_comm)

    T, H, K, E = args.tokens, HIDDEN, TOPK, EXPERTS
    seed = 1
    if args.layout < 0:
        # Over NVLink the dedup transport (one row per (token, destination
        # rank), fanned out into the same compact windows by the destination)
        # moves 0.45x (N=4) .. 0.66x (N=8) of the wire bytes.  With every rank
        # in one GPU's HBM the fan-out is an extra HBM pass, so N=1 keeps the
        # direct compact layout.
        args.layout = 2 if world > 1 else 1
    cfg = G.MoeConfig(E, K, T, H, args.mode, args.layout, args.ctas, args.engine)
    moes = G.Moe.create_all(comms, cfg) if R > 1 else [G.Moe(comms[0], cfg)]
    dev = torch.device("cuda", local)
    wdt = torch.float32 if args.mode == 1 else torch.int16
    xs = [torch.empty(T * H, dtype=torch.int16, device=dev) for _ in comms]
    idxs = [torch.empty(T * K, dtype=torch.int32, device=dev) for _ in comms]
    ws = [torch.empty(T * K, dtype=wdt, device=dev) for _ in comms]
    outs = [torch.empty(T * H, dtype=torch.int16, device=dev) for _ in comms]
    stream = torch.cuda.Stream(device=dev)
    for c, m, x, i, w in zip(comms, moes, xs, idxs, ws):
        m.generate(seed, c.rank, x, i, w, stream=stream)
    torch.cuda.synchronize()

    def step(xb=xs, ib=idxs, wb=ws, ob=outs):
        G.Moe.dispatch(moes, xb, ib, stream=stream)
        G.Moe.combine(moes, wb, ob, stream=stream)

    e_local = E // R_total
    remote_msgs = remote_rows = 0
    for c, i in zip(comms, idxs):
        dst = i.cpu().numpy().reshape(T, K) // e_local
        remote_msgs += int((dst != c.rank).sum())
        remote_rows += sum(len(set(int(v) for v in row) - {c.rank}) for row in dst)
    dmsg, cmsg = 2 * H + 16, 2 * H
    bytes_step = step_bytes(R_total, T)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    for c in comms:
        c.check_device()

    # --- device-timed region: K steps, events around each launch ---------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.3)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record(stream)
    for i in range(args.steps):
        ev[i][0].record(stream)
        G.Moe.dispatch(moes, xs, idxs, stream=stream)
        ev[i][1].record(stream)
        G.Moe.combine(moes, ws, outs, stream=stream)
        ev[i][2].record(stream)
    end.record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    for c in comms:
        c.check_device()
    total_ms = start.elapsed_time(end)
    d_ms = [e[0].elapsed_time(e[1]) for e in ev]
    c_ms = [e[1].elapsed_time(e[2]) for e in ev]
    t = torch.tensor([total_ms, statistics.mean(d_ms), statistics.mean(c_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms, d_mean, c_mean = t.tolist()
    ms_per_step = total_ms / args.steps
    value = bytes_step / (ms_per_step * 1e-3) / 1e9

    # --- parity self-check of the measured state (checker, untimed) ------------
    parity = None
    if not args.no_verify and args.mode in (0, 1) and args.layout in (0, 1, 2):
        try:
            parity = verify_step(G, torch, comms, moes, outs, seed, R_total, T, H, K, E, args.mode, args.layout, stream)
        except Exception as e:  # noqa: BLE001
            parity = {"error": str(e)[:300]}
        if world > 1:
            okv = all(parity.get(k) is True for k in ("outputs", "dispatch_windows", "combine_windows"))
            f = torch.tensor([1.0 if okv else 0.0], device=dev)
            dist.all_reduce(f, op=dist.ReduceOp.MIN)
            parity["all_ranks_ok"] = bool(f.item() == 1.0)

    # --- secondary configs on a single-rank comm: LL latency, RTT, variants ----
    if R > 1:
        comm_x = G.Comm.create_all([local], cfg_comm)[0]
    else:
        comm_x = comms[0]
    ll = None if args.no_extras else measure_ll(G, comm_x, rank, world, dist, torch, dev, stream)
    pp = None if (args.no_extras or world < 2) else measure_pingpong(G, comm_x, rank, world, dist, torch, dev)
    bw = None if (args.no_extras or world < 2) else measure_bw(G, comm_x, rank, world, dist, torch, dev)
    if rank == 0 and args.csv and pp:
        # the reference's CSV schema (harness_bench.cpp:167-178)
        G.write_csv(args.csv + ".pingpong.csv", pp["rows"])
        if bw:
            G.write_csv(args.csv + ".bw.csv", bw["rows"])
    a2a = None if (args.no_extras or world < 2) else measure_a2a(G, comm_x, rank, world, dist, torch, dev, stream)
    barrier = None if (args.no_extras or world < 2) else measure_barrier(G, comm_x, rank, world, dist, torch, dev)
    variants = None
    if not args.no_extras:
        variants = {"bf16_ht": measure_variant(G, comm_x, rank, world, dist, torch, dev, stream, T, 1, 1,
                                               "bf16 payloads and arithmetic, compact layout"),
                    "fp8_ht": measure_variant(G, comm_x, rank, world, dist, torch, dev, stream, T, 1, 2,
                                              "fp8 dispatch (e4m3 + per-128 scales), compact layout"),
                    "fp8_ll": measure_variant(G, comm_x, rank, world, dist, torch, dev, stream, 128, 0, 2,
                                              "fp8 dispatch, LL shape", steps=30),
                    "fp8_both_ht": measure_variant(G, comm_x, rank, world, dist, torch, dev, stream, T, 1, 3,
                                                   "fp8 dispatch + fp8 combine messages, compact layout")}
        if world > 1:
            variants["dedup_ht"] = measure_variant(G, comm_x, rank, world, dist, torch, dev, stream, T, 2, 1,
                                                   "dedup transport (layout 2), bf16")
            if args.layout == 2:
                # the per-message transport the reference's protocol uses, for
                # the NVLink-fraction figure (every message crosses the link)
                variants["message_transport_ht"] = measure_variant(
                    G, comm_x, rank, world, dist, torch, dev, stream, T, 1, args.mode,
                    "per-message transport (layout 1), headline arithmetic")
    overlap = None
    if not args.no_extras and world > 1:
        try:
            overlap = measure_overlap(G, comm_x, rank, world, dist, torch, dev, T)
        except Exception as e:  # noqa: BLE001
            overlap = {"error": str(e)[:200]}
    proxy = None
    if not args.no_extras:
        proxy = {"ll": measure_proxy(G, rank, world, local, dist, torch, dev, stream, allgather, 128, 10),
                 "ht": measure_proxy(G, rank, world, local, dist, torch, dev, stream, allgather, T, 3)}

    # --- e2e: host buffers through the public API, copies inside the region ---
    # Every step copies every local rank's inputs (x, topk_idx, weights) from
    # pinned host memory and reads every output back.  The copies run on their
    # own streams and are double-buffered, so step i+1's H2D and step i-1's D2H
    # overlap step i's dispatch/combine (what a serving loop does); the region
    # spans the first H2D to the last D2H.
    e2e = None
    if not args.no_e2e:
        xh = [x.cpu().pin_memory() for x in xs]
        ih = [i.cpu().pin_memory() for i in idxs]
        wh = [w.cpu().pin_memory() for w in ws]
        ohs = [[torch.empty_like(o, device="cpu").pin_memory() for o in outs] for _ in range(2)]
        bufs = [(xs, idxs, ws, outs), ([x.clone() for x in xs], [i.clone() for i in idxs], [w.clone() for w in ws],
                                       [o.clone() for o in outs])]
        h2d_s, d2h_s = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        e_steps = max(4, args.steps)

        def run_e2e(nsteps, s_ev=None, e_ev=None):
            h2d_done = [torch.cuda.Event() for _ in range(nsteps)]
            comp_done = [torch.cuda.Event() for _ in range(nsteps)]
            d2h_done = [torch.cuda.Event() for _ in range(nsteps)]
            if s_ev is not None:
                s_ev.record(h2d_s)
            for i in range(nsteps):
                b = i % 2
                bx, bi, bw, bo = bufs[b]
                with torch.cuda.stream(h2d_s):
                    if i >= 2:
                        h2d_s.wait_event(comp_done[i - 2])   # buffer b free again
                    for j in range(len(comms)):
                        bx[j].copy_(xh[j], non_blocking=True)
                        bi[j].copy_(ih[j], non_blocking=True)
                        bw[j].copy_(wh[j], non_blocking=True)
                    h2d_done[i].record(h2d_s)
                stream.wait_event(h2d_done[i])
                if i >= 2:
                    stream.wait_event(d2h_done[i - 2])       # outputs of buffer b read back
                step(bx, bi, bw, bo)
                comp_done[i].record(stream)
                with torch.cuda.stream(d2h_s):
                    d2h_s.wait_event(comp_done[i])
                    for j in range(len(comms)):
                        ohs[b][j].copy_(bo[j], non_blocking=True)
                    d2h_done[i].record(d2h_s)
            if e_ev is not None:
                stream.wait_event(d2h_done[-1])
                e_ev.record(stream)
        run_e2e(3)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        run_e2e(e_steps, s2, e2)
        torch.cuda.synchronize()
        te = torch.tensor([s2.elapsed_time(e2)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e_ms = te.item() / e_steps
        last = (e_steps - 1) % 2
        ok = all(bool((ohs[last][j] == outs[j].cpu()).all()) for j in range(len(comms)))
        e2e = {"value": bytes_step / (e_ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": e_ms, "steps": e_steps,
               "h2d_bytes_per_step": int(sum(x.numel() * 2 + i.numel() * 4 + w.numel() * w.element_size()
                                             for x, i, w in zip(xh, ih, wh))) * world,
               "d2h_bytes_per_step": int(sum(o.numel() * 2 for o in ohs[0])) * world,
               "pipelined": "double-buffered H2D/D2H streams", "output_matches_device_path": ok}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_kind = load_peaks()
    # dominant kernel and its algorithmic HBM bytes per launch:
    # one launch covers the R ranks of this process.  Symmetric traffic: every
    # message a rank writes lands in some rank's HBM and, on average, as many
    # land in it.
    #   dispatch: read T rows (2H) + idx, write T*K messages (dmsg)
    #   combine (send + reduce kernels): read T*K messages, write T*K combine
    #   rows (cmsg), read them back, write T output rows (+ weights)
    wb = 4 if args.mode == 1 else 2
    disp_hbm = R * (T * H * 2 + T * K * 4 + T * K * dmsg)
    comb_hbm = R * (T * K * dmsg + 2 * T * K * cmsg + T * H * 2 + T * K * wb)
    dom = "dispatch" if d_mean >= c_mean else "combine"
    dom_ms = max(d_mean, c_mean)
    dom_bytes = disp_hbm if dom == "dispatch" else comb_hbm
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        tr = tr.get(f"R{R}") if world == 1 else None  # captured at N=1 only (profiles/ncu_traffic.json)
        if tr:
            traffic = tr.get("dispatch") if dom == "dispatch" else (tr.get("combine", 0) + tr.get("reduce", 0)) or None
    except Exception:  # noqa: BLE001
        pass
    line = {
        "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if args.mode == 1 else "u16", "data": "synthetic",
        "config": {"workload": workload(R_total, T, mode=args.mode), "ranks": R_total, "tokens_per_rank": T,
                   "hidden": H, "top_k": K, "experts": E,
                   "placement": (f"{R} ranks emulated on 1 GPU (one cooperative launch per phase)" if R > 1
                                 else f"1 rank per GPU x {world}"),
                   "layout": {0: "reference", 1: "compact", 2: "compact + dedup"}[args.layout],
                   "parallelism": f"ep{R_total}",
                   "l2": f"inputs larger than L2 ({R * T * K * dmsg / 1e6:.0f} MB of messages per phase per GPU)"},
        "us_per_step": ms_per_step * 1e3, "dispatch_us": d_mean * 1e3, "combine_us": c_mean * 1e3,
        "per_gpu_GBps": value / world,
        "parity": parity,
        "roofline": {"bound": "hbm",
                     "kernel": ({"dispatch": "moe_dispatch_dedup_kernel" if args.layout == 2 else "moe_dispatch_tma_kernel",
                                 "combine": "moe_combine_tma_kernel + moe_combine_reduce_kernel"}[dom]
                                if args.engine in (0, 2) else f"moe_{dom}_kernel"),
                     "achieved": achieved, "peak": peak,
                     "unit": "GB/s", "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "algorithmic_bytes_per_launch": dom_bytes},
        "clocks": clk,
        # dispatch + combine-send + reduce kernels per step (one launch covers every emulated rank),
        # + the early reducer of the pipelined combine over NVLink (kernels_moe.cu plan())
        "gpu_launches": launches_per_step(args, world, R, T, K, E) * args.steps,
        "e2e": e2e,
        "ll": ll,
        "pingpong": pp,
        "bw": bw,
        "alltoall": a2a,
        "barrier": barrier,
        "variants": variants,
        "proxy_vs_direct": proxy,
        "overlap_with_compute": overlap,
    }
    if world > 1:
        # Over NVLink the dominant kernel's binding resource is the fabric, not
        # HBM: its remote bytes per launch over its time, against the measured
        # 705 GB/s ceiling of SM-issued peer writes and 900 nominal
        dom_remote = remote_msgs * cmsg if dom == "combine" else (
            remote_rows * (2 * H + 128) if args.layout == 2 else remote_msgs * dmsg)
        nv = dom_remote / (dom_ms * 1e-3) / 1e9
        line["roofline"]["binding"] = "nvlink"
        line["roofline"]["nvlink"] = {"achieved": nv, "peak_sm_write_measured": 705.0, "frac": nv / 705.0,
                                      "frac_of_900": nv / 900.0, "unit": "GB/s", "remote_bytes_per_launch": dom_remote}
        rem_msg_bytes = remote_msgs * dmsg
        rem_disp = remote_rows * (2 * H + 128) if args.layout == 2 else rem_msg_bytes
        line["nvlink"] = {"transport": "dedup rows (2H + 128 B per remote (token, rank))" if args.layout == 2
                          else "one message (dmsg) per remote (token, k)",
                          "remote_bytes_per_rank_dispatch": rem_disp,
                          "remote_message_bytes_per_rank_dispatch": rem_msg_bytes,
                          "dispatch_effective_message_GBps_per_gpu": rem_msg_bytes / (d_mean * 1e-3) / 1e9,
                          "dispatch_remote_GBps_per_gpu": rem_disp / (d_mean * 1e-3) / 1e9,
                          "combine_remote_GBps_per_gpu": remote_msgs * cmsg / (c_mean * 1e-3) / 1e9,
                          "frac_of_900": rem_disp / (d_mean * 1e-3) / 1e9 / 900.0,
                          "frac_of_measured_770": rem_disp / (d_mean * 1e-3) / 1e9 / 770.0,
                          "frac_of_sm_write_ceiling_705": rem_disp / (d_mean * 1e-3) / 1e9 / 705.0,
                          "note": "N>1 the step is NVLink-bound: the HBM roofline above is not the binding one; "
                                  "combine_remote_GBps includes the reduce kernel's time"}
    if world == 1 and not args.no_cpu_baseline:
        try:
            r = run_reference(R_total, T, 2, 1, float(os.environ.get("GINSIM_CPU_BASELINE_BUDGET_S", "20")))
        except Exception as e:  # noqa: BLE001
            r = None
            line["cpu_baseline_error"] = str(e)[:200]
        if r:
            line["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "reference",
                                    "sample": r["sample"]}
    print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
