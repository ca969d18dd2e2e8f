"""PCIe floor of the e2e step: 8 ranks x 58.7 MB pinned H2D and D2H copies, one direction or both
concurrently, over 1/2/4/8 streams per direction.  One JSON line (GB/s per direction)."""
import torch, time, json
dev = torch.device("cuda", 0)
n, sz = 8, 4096 * 7168
hx = [torch.empty(sz, dtype=torch.int16).pin_memory() for _ in range(n)]
ho = [torch.empty(sz, dtype=torch.int16).pin_memory() for _ in range(n)]
dx = [torch.empty(sz, dtype=torch.int16, device=dev) for _ in range(n)]
do = [torch.empty(sz, dtype=torch.int16, device=dev) for _ in range(n)]
res = []
for ns in (1, 2, 4, 8):
    hs = [torch.cuda.Stream() for _ in range(ns)]
    ds = [torch.cuda.Stream() for _ in range(ns)]
    def rnd():
        for j in range(n):
            with torch.cuda.stream(hs[j % ns]):
                dx[j].copy_(hx[j], non_blocking=True)
            with torch.cuda.stream(ds[j % ns]):
                ho[j].copy_(do[j], non_blocking=True)
    for mode in ("both", "h2d", "d2h"):
        def go():
            for j in range(n):
                if mode in ("both", "h2d"):
                    with torch.cuda.stream(hs[j % ns]):
                        dx[j].copy_(hx[j], non_blocking=True)
                if mode in ("both", "d2h"):
                    with torch.cuda.stream(ds[j % ns]):
                        ho[j].copy_(do[j], non_blocking=True)
        go(); torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(5): go()
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) / 5 * 1e3
        per_dir = n * sz * 2 / (ms * 1e-3) / 1e9
        res.append({"streams_per_dir": ns, "mode": mode, "ms_per_round": round(ms, 2), "GBps_per_direction": round(per_dir, 1)})
print(json.dumps(res))
