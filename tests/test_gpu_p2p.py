"""Device API semantics on the GPU (-m gpu): host-issued ops, cells, windows,
ring / ping-pong / all-to-all / moe-ht programs, both backends.  Ranks are
emulated on cuda:0 unless a test says otherwise."""
import ctypes
import json
import os

import numpy as np
import pytest

import paper_2511_15076_b200 as G
from oracle import oracle as O
from tests import gpu_util as U

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

pytestmark = pytest.mark.gpu
BACKENDS = ["direct", "proxy"]


def world(n, backend="direct", **kw):
    U.set_device(0)
    kw.setdefault("timeout_ms", 20000)
    return G.Comm.create_all([0] * n, G.Config(backend=backend, **kw))


def register(comms, nbytes_per_rank):
    """Collective window of nbytes (int or per-rank list) on every comm."""
    sizes = nbytes_per_rank if isinstance(nbytes_per_rank, list) else [nbytes_per_rank] * len(comms)
    ptrs = [c.mem_alloc(max(1, s)) for c, s in zip(comms, sizes)]
    wid = G.Comm.window_register_all(comms, [p if s else None for p, s in zip(ptrs, sizes)], sizes)
    return wid, ptrs


def close(comms):
    for c in comms:
        c.destroy()


@pytest.mark.parametrize("backend", BACKENDS)
def test_put_value_little_endian_and_bounds(backend):
    """putValue(0xDEADBEEF) lands as EF BE AD DE; 8 bytes at size-8 OK, at
    size-7 OutOfBounds (test_plugin.cpp:191-203, test_runtime.cpp:175-199)."""
    cs = world(2, backend)
    try:
        w, ptrs = register(cs, 64)
        g = G.Gin(cs[0], 0)
        g.put_value(1, w, 4, 0xDEADBEEF, 4, signal=3)
        cs[1].wait_signal(3, 1)
        assert list(U.d2h(ptrs[1], 64)[4:8]) == [0xEF, 0xBE, 0xAD, 0xDE]
        g.put_value(1, w, 56, 0x0102030405060708, 8, signal=3)
        cs[1].wait_signal(3, 2)
        assert list(U.d2h(ptrs[1], 64)[56:64]) == [8, 7, 6, 5, 4, 3, 2, 1]
        with pytest.raises(G.OutOfBounds):
            g.put_value(1, w, 57, 1, 8)
        with pytest.raises(G.InvalidDescriptor):
            g.put_value(1, w, 0, 1, 9)
        g.flush()
    finally:
        close(cs)


@pytest.mark.parametrize("backend", BACKENDS)
def test_put_with_signal_and_counter(backend):
    """Put + SignalInc / SignalAdd + CounterInc; flush; counters exact."""
    cs = world(3, backend)
    try:
        w, ptrs = register(cs, 4096)
        src = (np.arange(4096) * 7 % 251).astype(np.uint8)
        U.h2d(ptrs[0], src)
        g = G.Gin(cs[0], 1)
        g.put(2, w, 100, w, 0, 1000, signal=5, counter=2)
        g.put(1, w, 0, w, 1000, 3000, signal=5, add=41, counter=2)
        g.signal(2, 6, add=7, counter=3)
        g.flush()
        cs[2].wait_signal(5, 1)
        cs[1].wait_signal(5, 41)
        cs[2].wait_signal(6, 7)
        assert (U.d2h(ptrs[2], 4096)[100:1100] == src[:1000]).all()
        assert (U.d2h(ptrs[1], 4096)[:3000] == src[1000:4000]).all()
        cs[0].wait_counter(2, 2)
        cs[0].wait_counter(3, 1)
        assert cs[0].read_counter(2) == 2 and cs[0].read_counter(3) == 1
        cs[0].reset_counter(2)
        assert cs[0].read_counter(2) == 0
        cs[2].reset_signal(5)
        assert cs[2].read_signal(5) == 0
        g.put(2, w, 0, w, 0, 8, signal=5)
        cs[2].wait_signal(5, 1)
        assert cs[2].read_signal(5) == 1
    finally:
        close(cs)


def test_zero_byte_put_is_pure_release():
    """fabric.cpp:54-59: a zero-byte put touches no window but its signal applies."""
    cs = world(2)
    try:
        w, ptrs = register(cs, 64)
        U.memset(ptrs[1], 0x5A, 64)
        G.Gin(cs[0]).put(1, w, 64, w, 0, 0, signal=0)
        cs[1].wait_signal(0, 1)
        assert (U.d2h(ptrs[1], 64) == 0x5A).all()
    finally:
        close(cs)


def test_validation_errors():
    """Typed errors at the host boundary (runtime.cpp:474-544)."""
    cs = world(2)
    try:
        w, _ = register(cs, [4096, 1024])  # asymmetric capacities
        assert cs[0].window_size(w, 0) == 4096 and cs[0].window_size(w, 1) == 1024
        g = G.Gin(cs[0])
        with pytest.raises(G.OutOfBounds):
            g.put(1, w, 0, w, 0, 2048)  # destination checked against the PEER's capacity
        g.put(1, w, 0, w, 0, 1024)
        with pytest.raises(G.InvalidPeer):
            g.put(2, w, 0, w, 0, 8)
        with pytest.raises(G.UnknownWindow):
            g.put(1, 7, 0, w, 0, 8)
        with pytest.raises(G.InvalidSignal):
            g.signal(1, 999)
        with pytest.raises(G.InvalidContext):
            G.Gin(cs[0], 9).put(1, w, 0, w, 0, 8)
        with pytest.raises(G.InvalidCounter):
            cs[0].read_counter(4096)
        with pytest.raises(G.RankOutOfRange):
            cs[0].window_size(w, 5)
        g.flush()
    finally:
        close(cs)


def test_zero_size_windows_and_config_mismatch():
    cs = world(2)
    try:
        w, _ = register(cs, [0, 128])
        assert cs[1].window_size(w, 0) == 0
        with pytest.raises(G.OutOfBounds):
            G.Gin(cs[1]).put(0, w, 0, w, 0, 1)
    finally:
        close(cs)
    # ranks disagreeing on the config -> ConfigMismatch (runtime.cpp:86-105)
    grp = ctypes.c_void_p()
    G.check(G.lib().ginsim_cuda_inproc_group_create(2, ctypes.byref(grp)))
    import threading
    res = [None, None]

    def make(r):
        boot = G.Bootstrap()
        G.check(G.lib().ginsim_cuda_inproc_bootstrap(grp, r, ctypes.byref(boot)))
        cfg = G.Config(signal_cells=256 if r == 0 else 512)
        out = ctypes.c_void_p()
        res[r] = G.lib().ginsim_cuda_comm_create(r, 2, 0, ctypes.byref(cfg), ctypes.byref(boot), ctypes.byref(out))
    ts = [threading.Thread(target=make, args=(r,)) for r in range(2)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert res == [G.ConfigMismatch.code] * 2


@pytest.mark.parametrize("n,S,rounds,backend", [(2, 256, 3, "direct"), (4, 512, 25, "direct"),
                                                 (8, 4096, 10, "direct"), (2, 256, 3, "proxy"),
                                                 (4, 512, 25, "proxy")])
def test_ring_matches_reference_final_state(n, S, rounds, backend):
    """Device ring program (harness_ring.cpp:18-57 on the GPU) ends in the same
    windows and cells as the reference's run_ring (tests/golden/ring.json)."""
    gold = [c for c in json.load(open(os.path.join(os.path.dirname(__file__), "golden", "ring.json")))
            if (c["ranks"], c["bytes"], c["rounds"]) == (n, S, rounds)][0]
    cs = world(n, backend)
    try:
        ws, sp = register(cs, n * S)
        wr, rp = register(cs, n * S)
        G.check(G.lib().ginsim_cuda_ring(G.comm_handles(cs), n, ws, wr, S, rounds, None))
        for r in range(n):
            assert O.checksum(U.d2h(sp[r], n * S)) == gold["state"][r]["send"]
            assert O.checksum(U.d2h(rp[r], n * S)) == gold["state"][r]["recv"]
            sig, _ = cs[r].snapshot_cells()
            assert [[i, v] for i, v in enumerate(sig) if v] == gold["state"][r]["signals_nonzero"]
    finally:
        close(cs)


@pytest.mark.parametrize("channels,slots,messages,backend", [(24, 4, 64, "direct"), (6, 4, 16, "direct"),
                                                             (2, 1, 8, "direct"), (6, 4, 16, "proxy"),
                                                             (2, 1, 8, "proxy")])
def test_moe_ht_flow_control(channels, slots, messages, backend):
    """moe-ht circular buffers (harness_moe.cpp:283-382): every message delivered
    in order with correct stamps, final receive planes equal the oracle.  The
    proxy variant drives every put/signal through the GPU-producer descriptor
    ring and the host agent."""
    n, n_ctx, seed = 2, 4, 9
    n_pool = (channels + n_ctx - 1) // n_ctx
    pools = [world(n, backend) for _ in range(n_pool)]  # pool p: comms of every rank
    try:
        recv_ptrs = []
        for p in range(n_pool):
            wr, rp = register(pools[p], n_ctx * slots * 256)
            ws, _ = register(pools[p], n_ctx * slots * 256)
            assert (wr, ws) == (0, 1)
            recv_ptrs.append(rp)
        flat = [pools[p][r] for r in range(n) for p in range(n_pool)]
        G.check(G.lib().ginsim_cuda_moe_ht_ring(G.comm_handles(flat), n, n_pool, channels, slots, messages, seed, None))
        for p in range(n_pool):
            want = O.ht_plane(seed, channels, n_ctx, slots, messages, p)
            for r in range(n):
                assert (U.d2h(recv_ptrs[p][r], len(want)) == want).all()
                sig, ctr = pools[p][r].snapshot_cells()
                for ctx in range(n_ctx):
                    if p * n_ctx + ctx < channels:
                        assert sig[2 * ctx] == messages and sig[2 * ctx + 1] == messages
                        assert ctr[ctx] == messages
    finally:
        for p in pools:
            close(p)


def test_pingpong_payload_and_counts():
    """K14: device ping-pong; payload bytes (i*31+r) arrive intact, cells count
    iterations, RTT samples are positive."""
    cs = world(2)
    try:
        size = 4096
        ws, sp = register(cs, 1 << 20)
        wr, rp = register(cs, 1 << 20)
        for r in range(2):
            U.h2d(sp[r], O.pingpong_payload(r, size))
        rtt = U.malloc(8 * 50)
        G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles(cs), 2, 0, 1, ws, wr, size, 50, 5, 0, 256, rtt, None))
        t = U.d2h(rtt, 8 * 50, np.uint64)
        assert (t > 0).all()
        assert (U.d2h(rp[1], size) == O.pingpong_payload(0, size)).all()
        assert (U.d2h(rp[0], size) == O.pingpong_payload(1, size)).all()
        assert cs[0].read_signal(0) == 55 and cs[1].read_signal(0) == 55
        # a second call continues from the cell values (no reset needed)
        G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles(cs), 2, 0, 1, ws, wr, 1 << 20, 10, 1, 0, 512, rtt, None))
        assert cs[0].read_signal(0) == 66
        assert cs[0].read_signal(1) == 2 and cs[1].read_signal(1) == 2  # one launch handshake per call
        U.free(rtt)
    finally:
        close(cs)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_alltoall_pattern(n):
    """K15: every rank's recv[src*M..] holds src's send[dst*M..] after the
    signal count reaches (n-1) per iteration."""
    cs = world(n)
    try:
        M = 64 << 10
        ws, sp = register(cs, n * M)
        wr, rp = register(cs, n * M)
        for r in range(n):
            U.h2d(sp[r], ((np.arange(n * M) * 13 + r * 101) & 0xFF).astype(np.uint8))
        for it in (1, 2):
            G.check(G.lib().ginsim_cuda_alltoall(G.comm_handles(cs), n, ws, wr, M, 1, (n - 1) * it, 0, None))
            U.sync()
        for dst in range(n):
            got = U.d2h(rp[dst], n * M)
            for src in range(n):
                if src == dst:
                    continue
                want = ((np.arange(n * M) * 13 + src * 101) & 0xFF).astype(np.uint8)[dst * M:(dst + 1) * M]
                assert (got[src * M:(src + 1) * M] == want).all()
            assert cs[dst].read_signal(1) == 2 * (n - 1)
            cs[dst].check_device()
    finally:
        close(cs)


@pytest.mark.parametrize("n", [2, 4])
def test_alltoall_varying_sizes(n):
    """Back-to-back all-to-alls whose CTA split differs (it follows the message
    size) keep the per-peer release exact: bytes land, cells count n-1 per call."""
    cs = world(n)
    try:
        sizes = [1 << 10, 256 << 10, 4 << 10, 1 << 20]
        cap = n * max(sizes)
        ws, sp = register(cs, cap)
        wr, rp = register(cs, cap)
        for r in range(n):
            U.h2d(sp[r], ((np.arange(cap) * 7 + r * 29) & 0xFF).astype(np.uint8))
        for it, M in enumerate(sizes, start=1):
            G.check(G.lib().ginsim_cuda_alltoall(G.comm_handles(cs), n, ws, wr, M, 3, (n - 1) * it, 0, None))
            U.sync()
            for c in cs:
                c.check_device()
            for dst in range(n):
                got = U.d2h(rp[dst], n * M)
                for src in range(n):
                    if src != dst:
                        want = ((np.arange(cap) * 7 + src * 29) & 0xFF).astype(np.uint8)[dst * M:(dst + 1) * M]
                        assert (got[src * M:(src + 1) * M] == want).all()
                assert cs[dst].read_signal(3) == (n - 1) * it
    finally:
        close(cs)


def test_proxy_stats_and_reset_while_outstanding():
    cs = world(2, "proxy")
    try:
        w, ptrs = register(cs, 1 << 20)
        g = G.Gin(cs[0], 0)
        for i in range(200):
            g.put(1, w, (i % 16) * 4096, w, 0, 4096, counter=1)
        g.flush()
        assert cs[0].read_counter(1) == 200
        st = cs[0].proxy_stats()
        assert st["descriptors"] >= 200 and st["copies"] >= 200
    finally:
        close(cs)


def test_agent_copies_progress_while_every_sm_is_held():
    """The proxy agent's data movers must not need SMs: with a kernel holding
    every SM, an H2D inline-put copy (pinned -> VMM window) and a copy into a
    peer's VMM mapping complete on the copy engines.  (A same-device D2D copy
    does NOT -- the runtime runs it as a kernel -- which is why loopback puts
    are moved by the issuing SMs in proxy mode, gin_device.cuh Gin::put.)"""
    import subprocess
    import sys
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "copy_engine_probe.py")], capture_output=True,
                       text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    rows = {x["case"]: x for x in json.loads(r.stdout.strip().splitlines()[-1])["rows"]}
    assert rows["h2d_pinned_to_vmm_8B"]["completed_while_sms_held"]
    if "d2d_vmm_to_peer_mapping" in rows:
        assert rows["d2d_vmm_to_peer_mapping"]["completed_while_sms_held"]
        assert rows["h2d_pinned_to_peer_mapping_8B"]["completed_while_sms_held"]


@pytest.mark.parametrize("n", [2, 4, 8])
def test_dissemination_barrier_emulated_and_nvls_gating(n):
    """BarrierSession (runtime.cpp:651-666) on n emulated ranks: 300 rounds of
    ceil(log2 n) signal exchanges complete on every rank (twice: rounds
    continue across calls); the NVLS barrier stays off when ranks share a
    device (multicast needs distinct devices) and asking for it is refused."""
    cs = world(n)
    try:
        assert not any(c.nvls_enabled() for c in cs)
        ns = U.malloc(8 * 300)
        for _ in range(2):
            G.check(G.lib().ginsim_cuda_barrier_bench(G.comm_handles(cs), n, 0, 300, ns, None))
            U.sync()
        t = U.d2h(ns, 8 * 300, np.uint64)
        assert (t > 0).all()
        for c in cs:
            c.check_device()
        with pytest.raises(G.UsageError):
            G.check(G.lib().ginsim_cuda_barrier_bench(G.comm_handles(cs), n, 1, 10, ns, None))
        U.free(ns)
    finally:
        close(cs)


@pytest.mark.parametrize("n,channels,rounds,nbytes,backend", [(2, 8, 200, 64 << 10, "direct"),
                                                               (4, 6, 100, 16 << 10, "direct"),
                                                               (8, 4, 60, 4 << 10, "direct"),
                                                               (2, 4, 60, 16 << 10, "proxy")])
def test_signal_orders_earlier_puts_under_concurrency(n, channels, rounds, nbytes, backend):
    """Acceptance #1 (acceptance.cpp:63-118; fabric.cpp:63-79) on the device API:
    many concurrent (ctx, src->dst) channels; whenever a receiver observes
    signal >= round+1, every byte of that round's put is already visible.
    Two launches back to back (the cells continue)."""
    cs = world(n, backend)
    try:
        size = 2 * channels * nbytes
        ws, _ = register(cs, size)
        wd, _ = register(cs, size)
        for _ in range(2):
            G.check(G.lib().ginsim_cuda_ordering_stress(G.comm_handles(cs), n, ws, wd, nbytes, channels, rounds, None))
        for c in cs:
            c.check_device()
            assert c.read_signal(0) == 2 * rounds
    finally:
        close(cs)

