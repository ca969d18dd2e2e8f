"""Full-shape parity at the BASELINE HT config (the -m gpu tier).

8 ranks emulated on one B200, 4096 tokens per rank, hidden 7168, top-8 of 256
experts: EVERY output token of every rank against the CPU oracle's combine,
and EVERY dispatch-window message and combine-window record against the
oracle's expected record digests (the windows hold 3.76 GB per rank, so the
device digests them with ginsim_cuda_digest and the oracle digests what it
expects: oracle/ginsim_oracle.c gso_moe_window_digests).  u16 mode is the
reference's arithmetic (harness_moe.cpp:17-98) and must be bit-exact; bf16
mode must equal the fp32-sequential oracle bit for bit."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import paper_2511_15076_b200 as G
from oracle import oracle as O
from tests import gpu_util as U

pytestmark = pytest.mark.gpu


def _digests(ptr, rec, count):
    out = U.malloc(count * 8)
    try:
        G.digest(ptr, rec, count, out)
        U.sync()
        return U.d2h(out, count * 8, np.uint64)
    finally:
        U.free(out)


def test_device_digest_matches_oracle_definition():
    """ginsim_cuda_digest == oracle gso_digest on random records of every
    alignment class (16-byte, 8-byte, odd sizes)."""
    U.set_device(0)
    rng = np.random.default_rng(5)
    for rec, count in [(14352, 37), (14336, 9), (24, 100), (40, 3), (7, 50), (1, 3), (4097, 5)]:
        data = rng.integers(0, 256, rec * count, dtype=np.uint8)
        p = U.malloc(rec * count)
        try:
            U.h2d(p, data)
            got = _digests(p, rec, count)
            want = [O.digest(data[i * rec:(i + 1) * rec]) for i in range(count)]
            assert [int(v) for v in got] == want, rec
        finally:
            U.free(p)


def _check_all(run, seed, mode, layout):
    n, E, K, T, H = run.n, run.E, run.K, run.T, run.H
    dmsg, cmsg = 2 * H + 16, 2 * H
    slots = n * T * K if layout == 1 else (E // n) * n * T

    def expect(r):
        exp, _ = O.combine(seed, E, K, H, r, T, mode=mode)
        return (exp,) + O.window_digests(seed, n, E, K, T, H, r, mode=mode, layout=layout)

    with ThreadPoolExecutor(max_workers=8) as ex:
        exps = list(ex.map(expect, range(n)))
    cnt = O.counts(seed, n, E, K, T)
    e_local = E // n
    for r in range(n):
        exp, d, v, cdig = exps[r]
        c, m = run.comms[r], run.moes[r]
        assert (run.output(r) == exp).all(), ("output", r)
        dd = _digests(c.window_ptr(m.win_dispatch, r), dmsg, slots)
        bad = np.nonzero(dd[v] != d[v])[0]
        assert bad.size == 0, ("dispatch records", r, bad[:8])
        assert int(v.sum()) == int(cnt[r * e_local:(r + 1) * e_local].sum())
        cd = _digests(c.window_ptr(m.win_combine, r), cmsg, T * K)
        assert (cd == cdig).all(), ("combine records", r)
        sig, _ = c.snapshot_cells()
        for e_loc in range(e_local):
            assert sig[e_loc] == (n << 32) + int(cnt[r * e_local + e_loc].sum())
        assert sig[e_local] == T * K


@pytest.mark.parametrize("mode", [0, 1])
def test_ht_8rank_4096_every_token_and_record(mode):
    """BASELINE HT shape, compact layout (the bench's headline handle): all
    4096 tokens x 8 ranks and every window record, in u16 and bf16."""
    from tests.test_gpu_moe import MoeRun
    n, E, K, T, H, seed = 8, 256, 8, 4096, 7168, 1
    run = MoeRun(n, E, K, T, H, mode=mode, layout=1)
    try:
        run.generate(seed)
        run.step()
        _check_all(run, seed, mode, 1)
    finally:
        run.close()


def test_ht_8rank_reference_layout_digests():
    """The reference's worst-case layout (harness_moe.cpp:135-137) at 8 ranks,
    T=1024 (the layout is e_local*n*T messages per rank): every record."""
    from tests.test_gpu_moe import MoeRun
    n, E, K, T, H, seed = 8, 256, 8, 1024, 7168, 2
    run = MoeRun(n, E, K, T, H, mode=0, layout=0)
    try:
        run.generate(seed)
        run.step()
        _check_all(run, seed, 0, 0)
    finally:
        run.close()
