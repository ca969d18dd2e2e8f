"""CPU ORACLE loader (test infrastructure only).

ctypes/numpy front-end of oracle/ginsim_oracle.c (the plain-C restatement of the
reference's hot-path arithmetic) and of oracle/_ref/ginsim_ref_driver (the
unmodified reference compiled from /root/reference).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module; the product (paper_2511_15076_b200/) never does.
"""
from __future__ import annotations

import ctypes
import json
import os
import subprocess
from ctypes import POINTER, c_double, c_int, c_uint8, c_uint16, c_uint32, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# GINSIM_ORACLE_SO: an alternative build of the same C file (the sanitizer
# test runs the golden checks against an -fsanitize=address,undefined build)
ORACLE_SO = os.environ.get("GINSIM_ORACLE_SO") or os.path.join(HERE, "_build", "libginsim_oracle.so")
REF_DRIVER = os.path.join(HERE, "_ref", "ginsim_ref_driver")

_L = None


def build():
    subprocess.run(["bash", os.path.join(HERE, "build_ref.sh")], check=True, stdout=subprocess.DEVNULL)


def lib():
    global _L
    if _L is None:
        if not os.path.exists(ORACLE_SO):
            build()
        L = ctypes.CDLL(ORACLE_SO)
        L.gso_mix64.restype = c_uint64
        L.gso_mix64.argtypes = [c_uint64]
        L.gso_route_table.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, POINTER(c_uint32)]
        L.gso_tokens_u16.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, POINTER(c_uint16)]
        L.gso_tokens_bf16.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, POINTER(c_uint16)]
        L.gso_weights.argtypes = [c_uint32, c_uint32, c_uint32, c_int, c_void_p]
        L.gso_oracle_combine_all.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, POINTER(c_uint16)]
        L.gso_bf16_combine_all.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                           POINTER(c_uint16), POINTER(c_double)]
        L.gso_moe_ll_rank_state.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                            POINTER(c_uint8), POINTER(c_uint8), POINTER(c_uint64), c_uint32]
        L.gso_moe_ll_rank_state.restype = c_int
        L.gso_moe_bf16_rank_state.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                              POINTER(c_uint8), POINTER(c_uint8)]
        L.gso_moe_bf16_rank_state.restype = c_int
        L.gso_moe_counts.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, POINTER(c_uint32)]
        L.gso_descriptor_encode.argtypes = [c_void_p, POINTER(c_uint8)]
        L.gso_descriptor_encode.restype = c_int
        L.gso_descriptor_decode.argtypes = [POINTER(c_uint8), c_void_p]
        L.gso_descriptor_decode.restype = c_int
        L.gso_moe_ht_plane.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, POINTER(c_uint8)]
        L.gso_bf16_round.argtypes = [ctypes.c_float]
        L.gso_bf16_round.restype = c_uint16
        L.gso_fp8_e4m3.argtypes = [ctypes.c_float]
        L.gso_fp8_e4m3.restype = c_uint8
        L.gso_fp8_to_float.argtypes = [c_uint8]
        L.gso_fp8_to_float.restype = ctypes.c_float
        L.gso_fp8_quant_row.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, POINTER(c_uint8),
                                        POINTER(ctypes.c_float)]
        L.gso_fp8_combine_all.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                          POINTER(c_uint16)]
        L.gso_moe_fp8_rank_state.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                             POINTER(c_uint8), POINTER(c_uint8)]
        L.gso_moe_fp8_rank_state.restype = c_int
        L.gso_fp8c_combine_all.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                           POINTER(c_uint16)]
        L.gso_fp8c_combine_window.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                              POINTER(c_uint8)]
        _L = L
    return _L


def _p(a, t):
    return a.ctypes.data_as(POINTER(t))


# ---------------------------------------------------------------- moe data
def route_table(seed, experts, top_k, src, tokens):
    out = np.zeros((tokens, top_k), np.uint32)
    lib().gso_route_table(seed, experts, top_k, src, tokens, _p(out, c_uint32))
    return out


def tokens(seed, src, T, H, mode=0):
    out = np.zeros((T, H), np.uint16)
    (lib().gso_tokens_u16 if mode == 0 else lib().gso_tokens_bf16)(seed, src, T, H, _p(out, c_uint16))
    return out


def weights(src, T, K, mode=0):
    out = np.zeros((T, K), np.uint16 if mode == 0 else np.float32)
    lib().gso_weights(src, T, K, mode, out.ctypes.data)
    return out


def dispatch_message_bytes(hidden, mode=0):
    """u16/bf16: 2H payload + 16-byte meta (harness.hpp:112); fp8 (mode 2):
    H e4m3 bytes + H/128 fp32 scales + meta."""
    return (hidden + hidden // 32 if mode in (2, 3) else 2 * hidden) + 16


def combine_message_bytes(hidden, mode=0):
    """bf16/u16: 2H (harness.hpp:113); fp8 combine (mode 3): H + H/32."""
    return hidden + hidden // 32 if mode == 3 else 2 * hidden


def fp8_quant_row(seed, src, token, hidden):
    q = np.zeros(hidden, np.uint8)
    sc = np.zeros(hidden // 128, np.float32)
    lib().gso_fp8_quant_row(seed, src, token, hidden, _p(q, c_uint8), _p(sc, ctypes.c_float))
    return q, sc


def combine(seed, experts, top_k, hidden, src, T, mode=0):
    """Expected combine output [T][H] (u16 exact or bf16 bits) and, for bf16,
    the fp64 reference sum (fp8 mode: bf16 bits of the dequantized path)."""
    out = np.zeros((T, hidden), np.uint16)
    if mode == 3:
        lib().gso_fp8c_combine_all(seed, experts, top_k, hidden, src, T, _p(out, c_uint16))
        return out, None
    if mode == 2:
        lib().gso_fp8_combine_all(seed, experts, top_k, hidden, src, T, _p(out, c_uint16))
        return out, None
    if mode == 0:
        lib().gso_oracle_combine_all(seed, experts, top_k, hidden, src, T, _p(out, c_uint16))
        return out, None
    f64 = np.zeros((T, hidden), np.float64)
    lib().gso_bf16_combine_all(seed, experts, top_k, hidden, src, T, _p(out, c_uint16), _p(f64, c_double))
    return out, f64


def moe_rank_state(seed, n, experts, top_k, T, hidden, r, mode=0, n_cells=256):
    """(dispatch_recv bytes, combine_recv bytes, signal cells) of rank r after
    one moe-ll round, reference (worst-case) layout."""
    e_local = experts // n
    dmsg, cmsg = dispatch_message_bytes(hidden, mode), combine_message_bytes(hidden, mode)
    d = np.zeros(e_local * n * T * dmsg, np.uint8)
    c = np.zeros(T * top_k * cmsg, np.uint8)
    cells = np.zeros(n_cells, np.uint64)
    if mode in (2, 3):
        c2 = np.zeros(T * top_k * 2 * hidden, np.uint8)
        rc = lib().gso_moe_fp8_rank_state(seed, n, experts, top_k, T, hidden, r, _p(d, c_uint8), _p(c2, c_uint8))
        if mode == 2:
            c = c2
        else:
            lib().gso_fp8c_combine_window(seed, experts, top_k, hidden, r, T, _p(c, c_uint8))
        cnt = counts(seed, n, experts, top_k, T)
        for e_loc in range(e_local):
            cells[e_loc] = (n << 32) + int(cnt[r * e_local + e_loc].sum())
        cells[e_local] = T * top_k
    elif mode == 0:
        rc = lib().gso_moe_ll_rank_state(seed, n, experts, top_k, T, hidden, r, _p(d, c_uint8), _p(c, c_uint8),
                                         _p(cells, c_uint64), n_cells)
    else:
        rc = lib().gso_moe_bf16_rank_state(seed, n, experts, top_k, T, hidden, r, _p(d, c_uint8), _p(c, c_uint8))
        cnt = counts(seed, n, experts, top_k, T)
        for e_loc in range(e_local):
            e = r * e_local + e_loc
            cells[e_loc] = (n << 32) + int(cnt[e].sum())
        cells[e_local] = T * top_k
    assert rc == 0
    return d, c, cells


def counts(seed, n, experts, top_k, T):
    """cnt[e, src]: messages source src sends to expert e."""
    out = np.zeros((experts, n), np.uint32)
    lib().gso_moe_counts(seed, n, experts, top_k, T, _p(out, c_uint32))
    return out


def compact_to_reference(buf, cnt, r, n, e_local, T, K, dmsg):
    """Map a compact-layout dispatch buffer (src*T*K + prefix + slot) of rank r
    to the reference layout ((e_loc*n+src)*T+slot)."""
    out = np.zeros(e_local * n * T * dmsg, np.uint8)
    for src in range(n):
        acc = 0
        for e_loc in range(e_local):
            c = int(cnt[r * e_local + e_loc, src])
            if c:
                a = (src * T * K + acc) * dmsg
                b = ((e_loc * n + src) * T) * dmsg
                out[b:b + c * dmsg] = buf[a:a + c * dmsg]
            acc += c
    return out


def ht_plane(seed, channels, n_ctx, slots, messages, plane):
    out = np.zeros(n_ctx * slots * 256, np.uint8)
    lib().gso_moe_ht_plane(seed, channels, n_ctx, slots, messages, plane, _p(out, c_uint8))
    return out


def pingpong_payload(rank, size):
    return ((np.arange(size, dtype=np.uint64) * 31 + rank) & 0xFF).astype(np.uint8)


def ring_payload(sender, rnd, size):
    return ((sender * 131 + rnd * 31 + np.arange(size, dtype=np.uint64) * 7 + 1) & 0xFF).astype(np.uint8)


def checksum(buf) -> str:
    """Position-weighted 64-bit checksum of a byte buffer: sum_i w_i*(2i+1) mod 2^64
    over little-endian u64 words (zero-padded), plus the byte length."""
    b = np.ascontiguousarray(buf).reshape(-1).view(np.uint8)
    pad = (-len(b)) % 8
    if pad:
        b = np.concatenate([b, np.zeros(pad, np.uint8)])
    w = b.view("<u8")
    idx = np.arange(len(w), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
    with np.errstate(over="ignore"):
        return f"{int(np.sum(w * idx, dtype=np.uint64)):016x}:{len(b) - pad}"


# ---------------------------------------------------------------- descriptors
class _Desc(ctypes.Structure):
    _fields_ = [("opcode", c_uint8), ("flags", c_uint8), ("team", ctypes.c_uint16), ("peer", c_uint32),
                ("dst_window", c_uint32), ("src_window", c_uint32), ("dst_offset", c_uint64),
                ("src_offset_or_value", c_uint64), ("bytes", c_uint64), ("signal_id", c_uint32),
                ("counter_id", c_uint32), ("signal_operand", c_uint64)]


def descriptor_decode(buf: bytes):
    """(rc, fields tuple) — rc 0 when valid."""
    d = _Desc()
    arr = (c_uint8 * 64).from_buffer_copy(buf)
    rc = lib().gso_descriptor_decode(arr, ctypes.byref(d))
    return rc, tuple(getattr(d, f[0]) for f in _Desc._fields_)


def descriptor_encode(fields):
    d = _Desc(*fields)
    out = (c_uint8 * 64)()
    rc = lib().gso_descriptor_encode(ctypes.byref(d), out)
    return rc, bytes(out)


# ---------------------------------------------------------------- the reference itself
def ref_available():
    return os.path.exists(REF_DRIVER)


def ref_run(*args, timeout=900):
    """Run the unmodified reference (oracle/_ref) and return its JSON line."""
    r = subprocess.run([REF_DRIVER, *map(str, args)], capture_output=True, text=True, timeout=timeout)
    if r.returncode != 0:
        raise RuntimeError(f"reference driver failed: {r.stdout} {r.stderr}")
    return json.loads(r.stdout.strip().splitlines()[-1])


# ---------------------------------------------------------------- digests
def digest(buf):
    """gso_digest of a byte buffer (the device utility ginsim_cuda_digest's definition)."""
    a = np.ascontiguousarray(np.frombuffer(bytes(buf), np.uint8) if not isinstance(buf, np.ndarray) else buf.view(np.uint8))
    L = lib()
    L.gso_digest.restype = c_uint64
    L.gso_digest.argtypes = [POINTER(c_uint8), c_uint64]
    return int(L.gso_digest(_p(a, c_uint8), a.nbytes))


def window_digests(seed, n, E, K, T, H, r, mode=0, layout=1):
    """Expected per-record digests of rank r after one step: (dispatch slot
    digests, valid mask, combine record digests[T*K]).  Slots: layout 0
    e_local*n*T (harness_moe.cpp:135-137), layout 1 n*T*K (compact)."""
    L = lib()
    L.gso_moe_window_digests.restype = c_int
    L.gso_moe_window_digests.argtypes = [c_uint64, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32,
                                         c_uint32, c_uint32, POINTER(c_uint64), POINTER(c_uint8), POINTER(c_uint64)]
    slots = (E // n) * n * T if layout == 0 else n * T * K
    d = np.zeros(slots, np.uint64)
    v = np.zeros(slots, np.uint8)
    c = np.zeros(T * K, np.uint64)
    rc = L.gso_moe_window_digests(seed, n, E, K, T, H, mode, layout, r, _p(d, c_uint64), _p(v, c_uint8), _p(c, c_uint64))
    if rc != 0:
        raise ValueError(f"gso_moe_window_digests rc={rc}")
    return d, v.astype(bool), c
