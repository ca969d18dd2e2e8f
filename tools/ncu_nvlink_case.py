"""Profiling harness for NVLink evidence under ncu (single process, 2 GPUs).

ncu serialises kernels, so kernels that acquire a peer's release cannot be
replayed across GPUs.  This script drives the kernels that only PUSH: the
copy probe to the peer, and each rank's MoE dispatch (with
GINSIM_PROFILE_NO_WAIT=1, which skips the final acquire) and combine-send,
one after another, so every launch runs alone and its nvltx/nvlrx + DRAM
counters are attributable.  Not a benchmark: numbers printed here are not
bench values.

  GINSIM_NVLS=0 GINSIM_PROFILE_NO_WAIT=1 ncu --section Nvlink --section SpeedOfLight \
      --metrics nvltx__bytes.sum,nvlrx__bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      python tools/ncu_nvlink_case.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402


def main():
    assert os.environ.get("GINSIM_PROFILE_NO_WAIT") == "1", "set GINSIM_PROFILE_NO_WAIT=1"
    n = int(os.environ.get("NVL_N", "2"))  # GPUs driven by this one process
    comms = G.Comm.create_all(list(range(n)), G.Config(signal_cells=512))
    size = 256 << 20
    srcs = [c.mem_alloc(size) for c in comms]
    dsts = [c.mem_alloc(size) for c in comms]
    ws = G.Comm.window_register_all(comms, srcs, [size] * n)
    wd = G.Comm.window_register_all(comms, dsts, [size] * n)
    ms = ctypes.c_float()
    for eng, chunk in ((1, 4096), (0, 4096)):   # TMA, LSU 128-bit: rank 0 -> rank 1
        G.check(G.lib().ginsim_cuda_copy_bench_ex(comms[0].h, ws, wd, 1, size, eng, 148, chunk, 1,
                                                  ctypes.byref(ms), None))
    T, H, K, E = 4096, 7168, 8, 256
    moes = G.Moe.create_all(comms, G.MoeConfig(E, K, T, H, 1, 1, 0, 0))
    bufs = []
    for r in range(n):
        dev = torch.device("cuda", r)
        x = torch.empty(T * H, dtype=torch.int16, device=dev)
        idx = torch.empty(T * K, dtype=torch.int32, device=dev)
        w = torch.empty(T * K, dtype=torch.float32, device=dev)
        out = torch.empty(T * H, dtype=torch.int16, device=dev)
        with torch.cuda.device(r):
            moes[r].generate(1, r, x, idx, w)
        bufs.append((x, idx, w, out))
    for r in range(n):
        torch.cuda.synchronize(r)
    # dispatch of each rank alone (no acquire), then each rank's combine-send
    for r in range(n):
        with torch.cuda.device(r):
            G.Moe.dispatch([moes[r]], [bufs[r][0]], [bufs[r][1]])
            torch.cuda.synchronize(r)
    for r in range(n):
        with torch.cuda.device(r):
            G.Moe.combine([moes[r]], [bufs[r][2]], [bufs[r][3]])   # send kernel only (reduce skipped)
            torch.cuda.synchronize(r)
    # the dedup transport (layout 2): each rank's row puts alone
    moes2 = G.Moe.create_all(comms, G.MoeConfig(E, K, T, H, 1, 2, 0, 0))
    for r in range(n):
        with torch.cuda.device(r):
            G.Moe.dispatch([moes2[r]], [bufs[r][0]], [bufs[r][1]])
            torch.cuda.synchronize(r)
    print("profiling harness done")


if __name__ == "__main__":
    main()
