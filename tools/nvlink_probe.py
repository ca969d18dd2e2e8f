"""Measured copy rooflines for the put path: local HBM copy and NVLink peer
writes with both engines (LSU 128-bit stores vs TMA bulk), and a concurrent
all-pairs write to measure per-GPU egress when every GPU sends at once.
Single process, one comm per visible GPU.  Prints one JSON line."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2511_15076_b200 as G  # noqa: E402


def main():
    import torch
    n = torch.cuda.device_count()
    comms = G.Comm.create_all(list(range(n)), G.Config())
    size = 256 << 20
    srcs = [c.mem_alloc(size) for c in comms]
    dsts = [c.mem_alloc(size) for c in comms]
    ws = G.Comm.window_register_all(comms, srcs, [size] * n)
    wd = G.Comm.window_register_all(comms, dsts, [size] * n)
    out = {"gpus": n, "bytes": size, "rows": []}
    for engine in (0, 1):
        for ctas in (0, 32, 64):
            for peer in ([0, 1] if n > 1 else [0]):
                ms = ctypes.c_float()
                G.check(G.lib().ginsim_cuda_copy_bench(comms[0].h, ws, wd, peer, size, engine, ctas, 10,
                                                       ctypes.byref(ms), None))
                out["rows"].append({"engine": ["lsu", "tma"][engine], "ctas": ctas or 148,
                                    "target": "local" if peer == 0 else "peer", "ms": ms.value,
                                    "GBps": size / (ms.value * 1e-3) / 1e9})
    # HBM direction probes: write-only (fill) and read-only (sum) streams, 4 GiB
    buf = torch.empty(1 << 31, dtype=torch.int16, device="cuda:0")
    for name, fn, nbytes in [("write_only_fill", lambda: buf.fill_(3), buf.numel() * 2),
                             ("read_only_sum", lambda: buf.sum(dtype=torch.int32), buf.numel() * 2),
                             ("copy_rw", lambda: buf[: buf.numel() // 2].copy_(buf[buf.numel() // 2:]), buf.numel() * 2)]:
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(10):
            fn()
        e.record()
        torch.cuda.synchronize()
        ms = s.elapsed_time(e) / 10
        out["rows"].append({"engine": "torch", "target": name, "ms": ms, "GBps": nbytes / (ms * 1e-3) / 1e9})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
