"""H2D / D2H copy rates from pinned host memory, alone and concurrently (the
e2e leg's transfers): one 59 MB buffer each way, CUDA events."""
import json
import torch

dev = torch.device("cuda", 0)
n = 4096 * 7168  # int16 elements = 58.7 MB
h_in = torch.empty(n, dtype=torch.int16).pin_memory()
h_out = torch.empty(n, dtype=torch.int16).pin_memory()
d_in = torch.empty(n, dtype=torch.int16, device=dev)
d_out = torch.empty(n, dtype=torch.int16, device=dev)
s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
res = {}
for name in ("h2d", "d2h", "both"):
    for _ in range(3):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(s1)
        s2.wait_event(t0)
        if name in ("h2d", "both"):
            with torch.cuda.stream(s1):
                d_in.copy_(h_in, non_blocking=True)
        if name in ("d2h", "both"):
            with torch.cuda.stream(s2):
                h_out.copy_(d_out, non_blocking=True)
        e2 = torch.cuda.Event()
        e2.record(s2)
        s1.wait_event(e2)
        t1.record(s1)
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
    res[name] = {"ms": round(ms, 3), "GBps_each_way": round(n * 2 / ms / 1e6, 1)}
print(json.dumps(res))
