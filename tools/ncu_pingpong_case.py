"""Profiling harness for the put+signal ping-pong kernel under ncu: two ranks
emulated on cuda:0 in ONE cooperative launch (ncu serialises launches, so a
cross-GPU pair cannot be replayed), 8-byte messages, 2000 round trips timed
in-kernel with %globaltimer.  Prints the in-kernel RTT p50 (not a bench value)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2511_15076_b200 as G  # noqa: E402
from tests import gpu_util as U  # noqa: E402


def main():
    U.set_device(0)
    cs = G.Comm.create_all([0, 0], G.Config())
    size = 4096
    bufs = [c.mem_alloc(size) for c in cs]
    ws = G.Comm.window_register_all(cs, bufs, [size] * 2)
    rbufs = [c.mem_alloc(size) for c in cs]
    wr = G.Comm.window_register_all(cs, rbufs, [size] * 2)
    iters = 2000
    rtt = U.malloc(8 * iters)
    for nbytes in (8, 4096):
        G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles(cs), 2, 0, 1, ws, wr, nbytes, iters, 100, 0, 256, rtt, None))
        U.sync()
        t = np.sort(U.d2h(rtt, 8 * iters, np.uint64))
        print(f"emulated ping-pong {nbytes} B: RTT p50 {int(t[iters // 2])} ns")
    U.free(rtt)


if __name__ == "__main__":
    main()
