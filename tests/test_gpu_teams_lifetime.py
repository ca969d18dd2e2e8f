"""Teams, device-side op validation, counters in flight, window and MoE-handle
lifetime, and multi-context signal ordering on the Proxy backend (-m gpu).

Reference semantics: register_team / team (runtime.cpp:329-343), team_translate
(types.cpp:14-20), submit_op validation (runtime.cpp:474-507), ResetWhileOutstanding
(runtime.cpp:431-438), proxy peer resolution (proxy_backend.cpp:72)."""
import ctypes
import time

import numpy as np
import pytest

import paper_2511_15076_b200 as G
from oracle import oracle as O
from tests import gpu_util as U
from tests.conftest import gpu_count

pytestmark = pytest.mark.gpu
BACKENDS = ["direct", "proxy"]


def world(n, backend="direct", devices=None, **kw):
    U.set_device(0)
    kw.setdefault("timeout_ms", 20000)
    return G.Comm.create_all(devices or [0] * n, G.Config(backend=backend, **kw))


def register(comms, nbytes):
    ptrs = [c.mem_alloc(nbytes) for c in comms]
    wid = G.Comm.window_register_all(comms, ptrs, [nbytes] * len(comms))
    return wid, ptrs


def close(comms):
    for c in comms:
        c.destroy()


def team_ring(comms, team_id, ws, wr, S, rounds, sig=0):
    G.check(G.lib().ginsim_cuda_team_ring(G.comm_handles(comms), len(comms), team_id, ws, wr, S, rounds, sig, None))


@pytest.mark.parametrize("backend", BACKENDS)
def test_sub_team_ring_and_barrier(backend):
    """A ring + BarrierSession over the sub-team [3, 1, 2] of 4 ranks: team-relative
    peers translate to world ranks on both backends (the Proxy agent resolves the
    descriptor's (team id, team rank) through the registered team).  Each member's
    receive slot holds its team predecessor's pattern, the non-member's windows and
    cells stay untouched, and the world ring still works afterwards."""
    n, S, rounds = 4, 4096, 5
    cs = world(n, backend)
    try:
        members = [3, 1, 2]
        for c in cs:
            c.register_team(7, members)
            assert c.team(7) == members
            assert c.team(0) == list(range(n))
        ws, _ = register(cs, n * S)
        wr, rptrs = register(cs, n * S)
        team_ring(cs, 7, ws, wr, S, rounds, sig=5)
        for c in cs:
            c.check_device()
        for i, r in enumerate(members):
            pred = members[(i - 1) % len(members)]
            got = U.d2h(rptrs[r] + pred * S, S)
            want = np.array([(pred * 131 + (rounds - 1) * 31 + j * 7 + 1) & 0xFF for j in range(S)], np.uint8)
            assert (got == want).all(), (r, pred)
            assert cs[r].read_signal(5) == 0  # reset every round
        assert not U.d2h(rptrs[0], n * S).any()  # rank 0 is outside the team
        # barrier cells of slot 1 on members hold the rounds; rank 0's are zero
        base = cs[0].config.signal_cells - 64 + 8
        assert cs[0].read_signal(base) == 0 and cs[3].read_signal(base) == rounds
        G.check(G.lib().ginsim_cuda_ring(G.comm_handles(cs), n, ws, wr, S, 3, None))
        for c in cs:
            c.check_device()
    finally:
        close(cs)


@pytest.mark.parametrize("backend", BACKENDS)
def test_device_validation_raises_typed_errors(backend):
    """The device API validates like submit_op: a signal id past the table raises
    InvalidSignal, an unregistered team RankOutOfRange -- through the device
    error word, as typed exceptions, without hanging the kernel."""
    n, S = 2, 256
    cs = world(n, backend, signal_cells=256)
    try:
        ws, _ = register(cs, n * S)
        wr, _ = register(cs, n * S)
        with pytest.raises(G.InvalidSignal):
            team_ring(cs, 0, ws, wr, S, 1, sig=256 + 3)
        for c in cs:
            c.device_error(clear=True)
        with pytest.raises(G.RankOutOfRange):
            team_ring(cs, 42, ws, wr, S, 1)
        for c in cs:
            c.device_error(clear=True)
        team_ring(cs, 0, ws, wr, S, 2)  # a valid ring still runs afterwards
    finally:
        close(cs)


def test_register_team_errors():
    cs = world(2)
    try:
        c = cs[0]
        with pytest.raises(G.UsageError):
            c.register_team(3, [])
        with pytest.raises(G.InvalidPeer):
            c.register_team(3, [0, 5])
        c.register_team(3, [1, 0])
        with pytest.raises(G.UsageError):
            c.register_team(3, [0])
        with pytest.raises(G.UsageError):
            c.register_team(0, [0])  # the world team is always id 0
        with pytest.raises(G.UsageError):
            c.team(9)
        assert c.team(3) == [1, 0]
    finally:
        close(cs)


def test_reset_counter_refused_while_direct_op_in_flight():
    """Direct backend (runtime.cpp:431-438): a host-issued put carrying a local
    counter is outstanding until its stream ran it; reset_counter refuses with
    ResetWhileOutstanding meanwhile and succeeds once it completed."""
    import torch
    cs = world(2)
    try:
        w, _ = register(cs, 1 << 16)
        rel_host, rel_dev = U.host_mapped_words()
        s = torch.cuda.Stream(device=0)
        torch.cuda.synchronize()
        # hold the stream: a kernel that spins until the host releases it
        G.check(G.lib().ginsim_cuda_occupy(0, 1, ctypes.c_void_p(rel_dev), 20000, ctypes.c_void_p(s.cuda_stream)))
        held = torch.cuda.Event()
        held.record(s)
        G.Gin(cs[0], 0, stream=s.cuda_stream).put(1, w, 0, w, 4096, 4096, counter=2)
        time.sleep(0.05)
        assert not held.query(), ("the occupier must still hold the stream", ctypes.c_uint32.from_address(rel_host).value,
                                  hex(rel_host), hex(rel_dev), s.query())
        with pytest.raises(G.ResetWhileOutstanding):
            cs[0].reset_counter(2)
        cs[0].reset_counter(3)  # other counters are free
        ctypes.c_uint32.from_address(rel_host).value = 1
        torch.cuda.synchronize()
        assert cs[0].read_counter(2) == 1
        cs[0].reset_counter(2)
        assert cs[0].read_counter(2) == 0
    finally:
        close(cs)


@pytest.mark.parametrize("backend", BACKENDS)
def test_window_deregister_frees_and_reuses_ids(backend):
    cs = world(2, backend)
    try:
        a, pa = register(cs, 4096)
        b, pb = register(cs, 4096)
        c_, pc = register(cs, 4096)
        assert (a, b, c_) == (0, 1, 2)
        for c in cs:
            c.window_deregister(b)
        with pytest.raises(G.UnknownWindow):
            G.Gin(cs[0], 0).put(1, b, 0, a, 0, 8)
        with pytest.raises(G.UnknownWindow):
            cs[0].window_deregister(b)
        for c, p in zip(cs, pb):
            c.mem_free(p)
        d, pd = register(cs, 8192)
        assert d == b  # lowest free id first
        g = G.Gin(cs[0], 0)
        g.put_value(1, d, 8184, 0x1122334455667788, 8, signal=4)
        cs[1].wait_signal(4, 1)
        assert U.d2h(pd[1] + 8184, 8, np.uint64)[0] == 0x1122334455667788
        g.flush()
    finally:
        close(cs)


def test_moe_handle_create_destroy_cycles_flat_memory():
    """100 create / step / destroy cycles of an HT-shaped handle (4096 tokens,
    hidden 7168, ~1 GB of windows per rank) on 2 emulated ranks: device memory
    returns to its starting level, window ids and signal-cell ranges are
    reused (512 cells hold at most 29 ranges of this handle), and the steps
    that run stay bit-exact against the oracle."""
    import torch
    n, E, K, T, H, seed = 2, 16, 8, 4096, 7168, 3
    cs = world(n, signal_cells=512)
    try:
        cfg = G.MoeConfig(E, K, T, H, 0, 1, 0, 0)
        bufs = [(U.malloc(T * H * 2), U.malloc(T * K * 4), U.malloc(T * K * 2), U.malloc(T * H * 2)) for _ in range(n)]
        torch.cuda.synchronize()
        free0 = None
        firsts = set()
        for cyc in range(100):
            moes = G.Moe.create_all(cs, cfg)
            if cyc % 20 == 0:
                for r, m in enumerate(moes):
                    m.generate(seed, r, bufs[r][0], bufs[r][1], bufs[r][2])
                G.Moe.dispatch(moes, [b[0] for b in bufs], [b[1] for b in bufs])
                G.Moe.combine(moes, [b[2] for b in bufs], [b[3] for b in bufs])
                U.sync()
                for r, c in enumerate(cs):
                    c.check_device()
                    exp, _ = O.combine(seed, E, K, H, r, T)
                    got = U.d2h(bufs[r][3], T * H * 2, np.uint16).reshape(T, H)
                    assert (got == exp).all(), (cyc, r)
                    # the (possibly reused) range holds exactly this one step
                    first, span = moes[r].cells()
                    sig, _ = c.snapshot_cells()
                    cnt = O.counts(seed, n, E, K, T)
                    e_local = E // n
                    for e_loc in range(e_local):
                        assert sig[first + e_loc] == (n << 32) + int(cnt[r * e_local + e_loc].sum()), (cyc, r)
                    assert sig[first + e_local] == T * K
            assert moes[0].win_dispatch == 0
            firsts.add(moes[0].cells()[0])
            for m in moes:
                m.destroy()
            torch.cuda.synchronize()
            free_now = torch.cuda.mem_get_info(0)[0]
            if cyc == 1:
                free0 = free_now
            elif cyc > 1:
                assert abs(free_now - free0) < (64 << 20), (cyc, free0, free_now)
        assert len(firsts) == 1  # the freed range is handed out again every cycle
        for b in bufs:
            for p in b:
                U.free(p)
    finally:
        close(cs)


def test_proxy_contexts_signalling_one_cell_stay_monotone():
    """Proxy backend on 2 GPUs (one agent with several copy streams): a large
    put + SignalAdd(1) on context 0 and a small put + SignalAdd(1) on context 1
    toward the same peer cell.  The cell ends at exactly 2 (never moved
    backwards by an older absolute write) and both payloads are complete."""
    if gpu_count() < 2:
        pytest.skip("needs >= 2 GPUs (ranks sharing a device use one agent stream)")
    cs = world(2, "proxy", devices=[0, 1])
    try:
        big = 256 << 20
        w, ptrs = register(cs, big + 4096)
        U.set_device(0)
        pat = (np.arange(big + 4096, dtype=np.uint64) * 2654435761 % 251).astype(np.uint8)
        U.h2d(ptrs[0], pat)
        for it in range(1, 6):
            G.Gin(cs[0], 0).put(1, w, 0, w, 0, big, signal=9, add=1)
            G.Gin(cs[0], 1).put(1, w, big, w, big, 4096, signal=9, add=1)
            G.Gin(cs[0], 0).flush()
            G.Gin(cs[0], 1).flush()
            cs[1].wait_signal(9, 2 * it)
            U.set_device(1)
            U.sync()
            assert cs[1].read_signal(9) == 2 * it
            got = U.d2h(ptrs[1], big + 4096)
            assert (got == pat).all()
            U.set_device(0)
    finally:
        close(cs)


@pytest.mark.parametrize("backend", BACKENDS)
def test_timeouts_become_typed_errors_and_the_comm_stays_usable(backend):
    """Failure detection (runtime.cpp:296-311, Config.timeout_ms): a host wait
    that is never satisfied raises Timeout after the comm's timeout; a device
    program waiting for a peer that never launches (ping-pong with only rank
    0 running) ends its spin at the timeout and raises Timeout through the
    device error word; afterwards the comm still carries ops."""
    cs = world(2, backend, timeout_ms=300)
    try:
        w, ptrs = register(cs, 4096)
        t0 = time.time()
        with pytest.raises(G.Timeout):
            cs[1].wait_signal(7, 1)
        assert 0.25 < time.time() - t0 < 5.0
        rtt = U.malloc(8 * 16)
        t0 = time.time()
        with pytest.raises(G.Timeout):
            G.check(G.lib().ginsim_cuda_pingpong(G.comm_handles(cs[:1]), 1, 0, 1, w, w, 8, 16, 0, 40, 0, rtt, None))
        assert time.time() - t0 < 10.0
        U.free(rtt)
        for c in cs:
            c.device_error(clear=True)
        g = G.Gin(cs[0], 0)
        g.put_value(1, w, 0, 0x5A5A, 2, signal=9)
        cs[1].wait_signal(9, 1)
        assert int(U.d2h(ptrs[1], 2, np.uint16)[0]) == 0x5A5A
        g.flush()
    finally:
        close(cs)
