"""Do the proxy agent's copies need SMs?  Holds every SM of cuda:0 with a
spinning kernel, then issues each kind of copy the agent uses on another
stream and reports whether it completes while the GPU is full.
Prints one JSON line.  Diagnostic only (tests/test_gpu_p2p.py asserts it)."""
import ctypes
import glob
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def cudart():
    import nvidia.cuda_runtime as m
    path = glob.glob(os.path.join(os.path.dirname(m.__file__), "lib", "libcudart.so*"))[0]
    L = ctypes.CDLL(path)
    L.cudaMemcpyAsync.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    L.cudaMemcpyAsync.restype = ctypes.c_int
    L.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                    ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
    L.cudaMemcpy2DAsync.restype = ctypes.c_int
    L.cudaMemcpyPeerAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t,
                                      ctypes.c_void_p]
    L.cudaMemcpyPeerAsync.restype = ctypes.c_int
    return L


def run_case(name, issue, dev=0, hold_s=1.5):
    rel = torch.zeros(1, dtype=torch.int32).pin_memory()
    occ = torch.cuda.Stream(device=dev)
    side = torch.cuda.Stream(device=dev)
    G.check(G.lib().ginsim_cuda_occupy(dev, 2, ctypes.c_void_p(rel.data_ptr()), 10000, ctypes.c_void_p(occ.cuda_stream)))
    time.sleep(0.2)  # let the occupier fill the SMs
    issue(side)
    ev = torch.cuda.Event()
    ev.record(side)
    t0 = time.time()
    done = False
    while time.time() - t0 < hold_s:
        if ev.query():
            done = True
            break
        time.sleep(0.005)
    rel[0] = 1
    torch.cuda.synchronize(dev)
    return {"case": name, "completed_while_sms_held": done, "ms": (time.time() - t0) * 1e3 if done else None}


def main():
    rt = cudart()
    n = torch.cuda.device_count()
    torch.cuda.set_device(0)
    rows = []
    nb = 14336 * 64
    a = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(nb, dtype=torch.uint8, device="cuda:0")
    rows.append(run_case("d2d_cudamalloc_same_device", lambda s: rt.cudaMemcpyAsync(
        b.data_ptr(), a.data_ptr(), nb, 4, s.cuda_stream)))
    comms = G.Comm.create_all(list(range(min(n, 2))), G.Config())
    va = comms[0].mem_alloc(nb)
    vb = comms[0].mem_alloc(nb)
    rows.append(run_case("d2d_vmm_same_device", lambda s: rt.cudaMemcpyAsync(vb, va, nb, 4, s.cuda_stream)))
    rows.append(run_case("d2d_vmm_same_device_2d_h1", lambda s: rt.cudaMemcpy2DAsync(vb, nb, va, nb, nb, 1, 3,
                                                                                    s.cuda_stream)))
    rows.append(run_case("d2d_vmm_same_device_2d_h2", lambda s: rt.cudaMemcpy2DAsync(vb, nb // 2, va, nb // 2, nb // 2, 2,
                                                                                    3, s.cuda_stream)))
    rows.append(run_case("d2d_vmm_same_device_peerasync", lambda s: rt.cudaMemcpyPeerAsync(vb, 0, va, 0, nb,
                                                                                         s.cuda_stream)))
    hp = torch.zeros(8, dtype=torch.int64).pin_memory()
    rows.append(run_case("h2d_pinned_to_vmm_8B", lambda s: rt.cudaMemcpyAsync(vb, hp.data_ptr(), 8, 1, s.cuda_stream)))
    if n >= 2:
        size = nb
        srcs = [c.mem_alloc(size) for c in comms]
        dsts = [c.mem_alloc(size) for c in comms]
        G.Comm.window_register_all(comms, srcs, [size] * 2)
        wd = G.Comm.window_register_all(comms, dsts, [size] * 2)
        peer_dst = comms[0].window_ptr(wd, 1)
        rows.append(run_case("d2d_vmm_to_peer_mapping", lambda s: rt.cudaMemcpyAsync(peer_dst, srcs[0], size, 4, s.cuda_stream)))
        # a device-0 -> device-0 copy issued on a stream of device 1 (its copy engine, over NVLink)
        def other_dev(s):
            with torch.cuda.device(1):
                s1 = torch.cuda.Stream(device=1)
                rt.cudaMemcpyAsync(vb, va, nb, 4, s1.cuda_stream)
                e = torch.cuda.Event()
                e.record(s1)
            s.wait_event(e)
        rows.append(run_case("d2d_dev0_buffers_issued_on_dev1", other_dev))
        rows.append(run_case("h2d_pinned_to_peer_mapping_8B", lambda s: rt.cudaMemcpyAsync(peer_dst, hp.data_ptr(), 8, 1,
                                                                                        s.cuda_stream)))
    print(json.dumps({"gpus": n, "rows": rows}))


if __name__ == "__main__":
    main()
