"""HBM direction ceilings on one B200: TMA copy / TMA store-only (write-only stream) / LSU copies
(ginsim_cuda_copy_bench_ex) and torch fill / sum / copy, 2-4 GiB.  One JSON line (traffic GB/s)."""
import json, ctypes, sys, os
sys.path.insert(0, '.')
import torch
import paper_2511_15076_b200 as G
comms = G.Comm.create_all([0], G.Config())
size = 2 << 30
src = comms[0].mem_alloc(size); dst = comms[0].mem_alloc(size)
ws = G.Comm.window_register_all(comms, [src], [size]); wd = G.Comm.window_register_all(comms, [dst], [size])
rows = []
for engine, name in ((1, "tma_copy"), (4, "tma_store_only"), (0, "lsu_copy"), (2, "lsu256_copy")):
    for chunk in ((4096, 6144) if engine in (1, 4) else (4096,)):
        ms = ctypes.c_float()
        G.check(G.lib().ginsim_cuda_copy_bench_ex(comms[0].h, ws, wd, 0, size, engine, 0, chunk, 10, ctypes.byref(ms), None))
        traffic = size * (1 if engine == 4 else 2)
        rows.append({"engine": name, "chunk": chunk, "ms": round(ms.value, 3), "GBps_traffic": round(traffic / (ms.value * 1e-3) / 1e9, 1)})
buf = torch.empty(1 << 31, dtype=torch.int16, device="cuda:0")
for name, fn, nbytes in [("torch_fill_write_only", lambda: buf.fill_(3), buf.numel() * 2),
                         ("torch_sum_read_only", lambda: buf.sum(dtype=torch.int32), buf.numel() * 2),
                         ("torch_copy_rw", lambda: buf[: buf.numel() // 2].copy_(buf[buf.numel() // 2:]), buf.numel() * 2)]:
    fn(); torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): fn()
    e.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    rows.append({"engine": name, "ms": round(ms, 3), "GBps_traffic": round(nbytes / (ms * 1e-3) / 1e9, 1)})
print(json.dumps(rows))
