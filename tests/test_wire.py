"""GIN1 wire codec (the socket transport's framing,
proj/core/include/ginsim/wire.hpp:12-67) through the C ABI, on the CPU.

* tests/golden/wire.json: 256 frames the UNMODIFIED reference encoded
  (oracle/ref_driver.cpp `wire`, oracle/make_golden.py); our encoder must
  produce the same bytes and our parser must decode them to the same fields.
* The reference's own cases (proj/tests/test_wire.cpp:17-115): golden header
  bytes, a byte-dribbled stream of all four types, zero-length puts, garbage
  rejected (magic, type, padding), inc signals carry operand 1 on the wire.
"""
import json
import os

import pytest

import paper_2511_15076_b200 as G

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "wire.json")
W = G.WireFrame


def _frames():
    with open(GOLDEN) as f:
        return json.load(f)["frames"]


def _encode(fr):
    body = bytes.fromhex(fr["body"])
    return G.wire_encode(fr["type"], src=fr["src"], ctx=fr["ctx"], seq=fr["seq"], window_or_signal=fr["id"],
                         dst_offset=fr["offset"], signal_add=fr["add"], operand=fr["operand"], body=body)


def test_encoder_matches_the_reference_bytes():
    frames = _frames()
    assert len(frames) == 256 and {f["type"] for f in frames} == {1, 2, 3, 4}
    for fr in frames:
        assert _encode(fr).hex() == fr["hex"], fr


def test_parser_decodes_the_reference_stream_fed_in_odd_pieces():
    frames = _frames()
    stream = b"".join(bytes.fromhex(f["hex"]) for f in frames)
    p = G.WireParser()
    got = []
    step = 1
    i = 0
    while i < len(stream):  # pieces of 1, 2, 3, ... 17 bytes: every split point is crossed
        p.feed(stream[i:i + step])
        i += step
        step = step % 17 + 1
        while (r := p.next()) is not None:
            got.append(r)
    assert len(got) == len(frames) and p.buffered() == 0
    for (f, body), fr in zip(got, frames):
        assert f.type == fr["type"] and f.src_rank == fr["src"]
        # (a control frame carries ctx 0 and seq 0, wire.cpp encode_control_frame)
        assert f.seq_or_watermark == (0 if fr["type"] == W.CONTROL else fr["seq"])
        if fr["type"] == W.PUT:
            assert (f.window_or_signal, f.dst_offset, body.hex(), f.ctx) == (fr["id"], fr["offset"], fr["body"], fr["ctx"])
        elif fr["type"] == W.SIGNAL:
            assert (f.window_or_signal, f.signal_add, f.ctx) == (fr["id"], fr["add"], fr["ctx"])
            assert f.operand == (fr["operand"] if fr["add"] else 1)
        elif fr["type"] == W.CONTROL:
            assert body.hex() == fr["body"] and f.ctx == 0
        else:
            assert f.ctx == fr["ctx"] and body == b""


def test_put_frame_header_golden_bytes():
    """test_wire.cpp:17-33."""
    f = G.wire_encode(W.PUT, src=2, ctx=1, seq=5, window_or_signal=7, dst_offset=64, body=b"\xaa\xbb\xcc")
    assert f[0:4] == bytes([0x31, 0x49, 0x4E, 0x47])  # magic 0x474E4931 little-endian
    assert f[4] == 1 and f[5] == 2 and f[9] == 1 and f[11] == 0 and f[12] == 0 and f[13] == 5
    assert len(f) == 21 + 20 + 3


def test_frames_survive_a_byte_dribbled_stream():
    """test_wire.cpp:35-76."""
    payload = bytes(range(1, 10))
    stream = (G.wire_encode(W.PUT, src=3, ctx=2, seq=11, window_or_signal=4, dst_offset=1024, body=payload) +
              G.wire_encode(W.SIGNAL, src=3, ctx=2, seq=11, window_or_signal=6, signal_add=1, operand=42) +
              G.wire_encode(W.ACK, src=1, ctx=2, seq=11) +
              G.wire_encode(W.CONTROL, src=0, body=b"hi"))
    p = G.WireParser()
    frames = []
    for b in stream:
        p.feed(bytes([b]))
        while (r := p.next()) is not None:
            frames.append(r)
    assert len(frames) == 4
    (f0, b0), (f1, _), (f2, _), (f3, b3) = frames
    assert (f0.type, f0.src_rank, f0.ctx, f0.seq_or_watermark, f0.window_or_signal, f0.dst_offset, b0) == \
        (W.PUT, 3, 2, 11, 4, 1024, payload)
    assert (f1.type, f1.window_or_signal, f1.signal_add, f1.operand) == (W.SIGNAL, 6, 1, 42)
    assert (f2.type, f2.src_rank, f2.seq_or_watermark) == (W.ACK, 1, 11)
    assert (f3.type, b3) == (W.CONTROL, b"hi")
    assert p.buffered() == 0


def test_zero_length_put_parses():
    p = G.WireParser()
    p.feed(G.wire_encode(W.PUT, seq=1))
    f, body = p.next()
    assert f.type == W.PUT and body == b""


@pytest.mark.parametrize("index,value", [(0, 0xFF), (4, 9), (11, 1)])
def test_garbage_on_the_stream_is_rejected(index, value):
    """test_wire.cpp:78-105: bad magic, unknown type, nonzero padding."""
    f = bytearray(G.wire_encode(W.ACK, seq=1))
    f[index] = value
    p = G.WireParser()
    p.feed(bytes(f))
    with pytest.raises(G.MalformedFrame):
        p.next()


def test_unknown_signal_op_is_rejected():
    f = bytearray(G.wire_encode(W.SIGNAL, window_or_signal=3, signal_add=1, operand=5))
    f[21 + 4] = 2
    p = G.WireParser()
    p.feed(bytes(f))
    with pytest.raises(G.MalformedFrame):
        p.next()


def test_inc_signals_always_carry_operand_one():
    """test_wire.cpp:107-115."""
    f = G.wire_encode(W.SIGNAL, seq=3, window_or_signal=9, signal_add=0, operand=77)
    p = G.WireParser()
    p.feed(f)
    fr, _ = p.next()
    assert fr.signal_add == 0 and fr.operand == 1


def test_partial_frames_wait_and_small_body_buffers_are_refused():
    f = G.wire_encode(W.PUT, seq=9, window_or_signal=1, body=bytes(100))
    p = G.WireParser()
    p.feed(f[:30])
    assert p.next() is None and p.buffered() == 30
    p.feed(f[30:])
    with pytest.raises(G.UsageError):  # nothing consumed: retry with room for the body
        p.next(body_cap=10)
    fr, body = p.next(body_cap=200)
    assert fr.body_bytes == 100 and body == bytes(100) and p.buffered() == 0


def test_encode_rejects_a_short_output_buffer_and_bad_ops():
    with pytest.raises(G.UsageError):
        G.wire_encode(9)
    with pytest.raises(G.UsageError):
        G.wire_encode(W.SIGNAL, signal_add=2)


# ---------------------------------------------------------------- socket rendezvous (host only)
def _rendezvous(world, port, payloads, results, rank):
    import ctypes
    boot = G.Bootstrap()
    try:
        G.check(G.lib().ginsim_cuda_socket_bootstrap_create(b"127.0.0.1", port, world, rank, 20000, ctypes.byref(boot)))
        for blob in payloads[rank]:  # successive allgathers reuse the connections
            n = len(blob)
            send = (ctypes.c_uint8 * n).from_buffer_copy(blob)
            recv = (ctypes.c_uint8 * (n * world))()
            rc = boot.allgather(boot.ctx, ctypes.cast(send, ctypes.c_void_p), ctypes.cast(recv, ctypes.c_void_p), n)
            results[rank].append((rc, bytes(recv)))
    except Exception as e:  # noqa: BLE001
        results[rank].append(("error", repr(e)))
    finally:
        G.lib().ginsim_cuda_socket_bootstrap_destroy(ctypes.byref(boot))


def test_socket_rendezvous_allgathers_rank_major():
    """comm_init_socket's rendezvous (socket_transport.cpp:178-231) on its own:
    rank 0 listens on a port from reserve_loopback_port, the others connect
    and say hello; every allgather returns the ranks' blobs rank-major, on
    every rank, call after call (the comm's window registrations reuse it)."""
    import threading
    world = 3
    port = G.reserve_loopback_port()
    payloads = [[bytes([r] * 8), bytes(range(r, r + 40)), (r * 1000).to_bytes(4, "little")] for r in range(world)]
    results = [[] for _ in range(world)]
    ts = [threading.Thread(target=_rendezvous, args=(world, port, payloads, results, r)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    for r in range(world):
        assert len(results[r]) == 3, results[r]
        for i, (rc, got) in enumerate(results[r]):
            assert rc == 0 and got == b"".join(payloads[q][i] for q in range(world)), (r, i)


def test_socket_rendezvous_rejects_bad_arguments():
    import ctypes
    boot = G.Bootstrap()
    with pytest.raises(G.UsageError):
        G.check(G.lib().ginsim_cuda_socket_bootstrap_create(b"not-an-ip", 1, 2, 0, 100, ctypes.byref(boot)))
    with pytest.raises(G.UsageError):
        G.check(G.lib().ginsim_cuda_socket_bootstrap_create(b"127.0.0.1", 1, 2, 2, 100, ctypes.byref(boot)))
    # a rank that finds nobody at the rendezvous fails with a bootstrap timeout
    with pytest.raises(G.BootstrapTimeout):
        G.check(G.lib().ginsim_cuda_socket_bootstrap_create(b"127.0.0.1", G.reserve_loopback_port(), 2, 1, 300,
                                                            ctypes.byref(boot)))
