"""Generate tests/golden/ fixtures from the UNMODIFIED reference (oracle/_ref).

Run here (where /root/reference exists):  python oracle/make_golden.py
Fixtures are small JSON files: checksums of the reference's final windows and
its signal cells for a sweep of moe-ll configs (run_moe_ll, harness_moe.cpp:252),
the routing table recovered from the reference's own dispatch window for the
BASELINE LL config, ring final states (run_ring), and 64-byte descriptor
encodings from the reference codec (encode_descriptor, descriptor.cpp:148).
"""
from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle import oracle as O  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")


checksum = O.checksum


MOE_CONFIGS = [
    # (ranks, experts, topk, tokens, hidden, seed, backend)
    (2, 4, 1, 1, 32, 3, "direct"),        # test_harness.cpp:109-120
    (2, 8, 2, 3, 64, 21, "direct"),       # test_harness.cpp:141-151
    (2, 8, 2, 3, 64, 21, "proxy"),
    (4, 16, 2, 4, 7168, 11, "proxy"),     # test_harness.cpp:122-133
    (2, 4, 2, 2, 64, 5, "proxy"),
    (8, 64, 2, 8, 7168, 0, "direct"),     # acceptance.cpp:321-338 (seeds 0..19)
    (8, 64, 2, 8, 7168, 7, "direct"),
    (8, 64, 2, 8, 7168, 19, "proxy"),
    (4, 32, 4, 16, 256, 2, "direct"),
    (8, 256, 8, 16, 7168, 1, "direct"),
    (8, 256, 8, 128, 7168, 1, "direct"),  # BASELINE LL config
    # edge shapes (appended: the GPU golden test covers the first 11)
    (4, 8, 2, 4, 96, 0, "direct"),        # acceptance.cpp:305-318 (#6 backend equivalence)
    (4, 8, 2, 4, 96, 13, "proxy"),
    (2, 4, 4, 3, 32, 9, "direct"),        # top_k == experts: every expert routed
    (4, 4, 2, 5, 64, 4, "direct"),        # one expert per rank
    (2, 2, 1, 6, 16, 8, "proxy"),         # the smallest pool
    (2, 4, 2, 3, 5, 6, "direct"),         # odd hidden (26-byte dispatch messages)
    (8, 16, 3, 1, 8, 12, "direct"),       # one token per rank on 8 ranks
]


def moe_fixture():
    out = []
    for (n, E, K, T, H, seed, backend) in MOE_CONFIGS:
        d = tempfile.mkdtemp(prefix="gold")
        try:
            O.ref_run("moe-ll", "--ranks", n, "--experts", E, "--topk", K, "--tokens", T, "--hidden", H,
                      "--seed", seed, "--backend", backend, "--dump", d)
            ranks = []
            routes = None
            for r in range(n):
                disp = np.fromfile(f"{d}/rank{r}_dispatch.bin", np.uint8)
                comb = np.fromfile(f"{d}/rank{r}_combine.bin", np.uint8)
                sig = np.fromfile(f"{d}/rank{r}_signals.bin", np.uint64)
                ctr = np.fromfile(f"{d}/rank{r}_counters.bin", np.uint64)
                nz = [[int(i), int(sig[i])] for i in np.nonzero(sig)[0]]
                ranks.append({"dispatch": checksum(disp), "combine": checksum(comb), "signals_nonzero": nz,
                              "counters_nonzero": int(np.count_nonzero(ctr))})
                if (n, E, K, T, H, seed) == (8, 256, 8, 128, 7168, 1):
                    # routing recovered from the reference's own dispatch window meta
                    if routes is None:
                        routes = np.full((n, T, K), -1, np.int32)
                    e_local, dmsg = E // n, 2 * H + 16
                    msgs = disp.reshape(e_local, n, T, dmsg)
                    meta = msgs[..., 2 * H:].copy().view("<u4").reshape(e_local, n, T, 4)
                    for e_loc in range(e_local):
                        for src in range(n):
                            for slot in range(T):
                                s, t, k, tag = meta[e_loc, src, slot]
                                if tag == 0:
                                    break
                                routes[src, t, k] = r * e_local + e_loc
            entry = {"ranks": n, "experts": E, "topk": K, "tokens": T, "hidden": H, "seed": seed,
                     "backend": backend, "state": ranks}
            if routes is not None:
                assert (routes >= 0).all()
                entry["routes"] = routes.tolist()
            out.append(entry)
            print("moe-ll", n, E, K, T, H, seed, backend, "ok", flush=True)
        finally:
            shutil.rmtree(d)
    return out


def ring_fixture():
    out = []
    # the first three are the GPU test's shapes; then acceptance #5's 100 rounds
    # (acceptance.cpp:273-300) on 8 ranks over both backends, an odd rank count
    # with a ragged size, and a one-byte payload
    for (n, S, rounds, backend) in [(2, 256, 3, "direct"), (4, 512, 25, "proxy"), (8, 4096, 10, "direct"),
                                    (8, 1024, 100, "proxy"), (8, 1024, 100, "direct"), (3, 333, 7, "direct"),
                                    (2, 1, 4, "proxy")]:
        d = tempfile.mkdtemp(prefix="gold")
        try:
            O.ref_run("ring", "--ranks", n, "--bytes", S, "--rounds", rounds, "--backend", backend, "--dump", d)
            ranks = []
            for r in range(n):
                ranks.append({"send": checksum(np.fromfile(f"{d}/ring_rank{r}_send.bin", np.uint8)),
                              "recv": checksum(np.fromfile(f"{d}/ring_rank{r}_recv.bin", np.uint8)),
                              "signals_nonzero": [[int(i), int(v)] for i, v in
                                                  enumerate(np.fromfile(f"{d}/ring_rank{r}_signals.bin", np.uint64))
                                                  if v]})
            out.append({"ranks": n, "bytes": S, "rounds": rounds, "backend": backend, "state": ranks})
        finally:
            shutil.rmtree(d)
    return out


def descriptor_fixture():
    d = tempfile.mkdtemp(prefix="gold")
    try:
        p1 = os.path.join(d, "a.bin")
        O.ref_run("descriptors", "--seed", 0xD15C0, "--count", 10000, "--out", p1)
        a = np.fromfile(p1, np.uint8).reshape(-1, 64)
        p2 = os.path.join(d, "b.bin")
        O.ref_run("descriptors", "--seed", 0xACCE55C0DE, "--count", 100000, "--out", p2)
        b = np.fromfile(p2, np.uint8).reshape(-1, 64)
        return {"seed_a": 0xD15C0, "count_a": 10000, "checksum_a": checksum(a),
                "first_a_hex": [bytes(x).hex() for x in a[:512]],
                "seed_b": 0xACCE55C0DE, "count_b": 100000, "checksum_b": checksum(b),
                "sample_b_hex": [bytes(x).hex() for x in b[::997][:100]]}
    finally:
        shutil.rmtree(d)


def wire_fixture():
    """GIN1 frames the reference encodes (wire.cpp via ref_driver `wire`):
    256 seeded frames of every type, with their fields and the exact bytes."""
    return O.ref_run("wire", "--seed", 0x6171, "--count", 256)


def main():
    if not O.ref_available():
        raise SystemExit("oracle/_ref missing: run oracle/build_ref.sh first")
    os.makedirs(GOLDEN, exist_ok=True)
    if sys.argv[1:] == ["ring"]:  # only the ring fixture
        with open(os.path.join(GOLDEN, "ring.json"), "w") as f:
            json.dump(ring_fixture(), f)
        print("ring fixture written to", GOLDEN)
        return
    if sys.argv[1:] == ["moe"]:  # only the moe-ll fixture
        with open(os.path.join(GOLDEN, "moe_ll.json"), "w") as f:
            json.dump(moe_fixture(), f)
        print("moe-ll fixture written to", GOLDEN)
        return
    with open(os.path.join(GOLDEN, "wire.json"), "w") as f:
        json.dump(wire_fixture(), f)
    if sys.argv[1:] == ["wire"]:  # only the wire fixture
        print("wire fixture written to", GOLDEN)
        return
    with open(os.path.join(GOLDEN, "descriptors.json"), "w") as f:
        json.dump(descriptor_fixture(), f)
    with open(os.path.join(GOLDEN, "ring.json"), "w") as f:
        json.dump(ring_fixture(), f)
    with open(os.path.join(GOLDEN, "moe_ll.json"), "w") as f:
        json.dump(moe_fixture(), f)
    print("golden fixtures written to", GOLDEN)


if __name__ == "__main__":
    main()
