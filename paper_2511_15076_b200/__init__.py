"""paper_2511_15076_b200 — B200-native GIN hot path (device-initiated put/signal
over NVLink 5, Proxy backend, DeepEP-style MoE dispatch/combine).

Python host-side mirror of the reference's C++ API (/root/reference/proj/core/
include/ginsim/runtime.hpp, types.hpp, errors.hpp), bound through ctypes to the
C-ABI library ``_lib/libginsim_b200.so`` (include/ginsim_cuda.h).  There is no
fallback: importing works without a GPU, but every compute call goes through
the CUDA library and raises if it is missing.
"""
from __future__ import annotations

import ctypes
import os
import threading
from ctypes import (POINTER, byref, c_char_p, c_int, c_int32, c_size_t, c_uint8, c_uint16, c_uint32,
                    c_uint64, c_void_p)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GINSIM_LIB") or os.path.join(_HERE, "_lib", "libginsim_b200.so")

# --------------------------------------------------------------------- errors
# One class per ginsim exception (errors.hpp:24-52), codes as in ginsim_cuda.h.


class Error(RuntimeError):
    code = 25


def _mk(name, code):
    return type(name, (Error,), {"code": code})


InvalidDescriptor = _mk("InvalidDescriptor", 1)
MalformedDescriptor = _mk("MalformedDescriptor", 2)
OutOfBounds = _mk("OutOfBounds", 3)
UnknownWindow = _mk("UnknownWindow", 4)
RankOutOfRange = _mk("RankOutOfRange", 5)
DuplicateEndpoint = _mk("DuplicateEndpoint", 6)
UnknownChannel = _mk("UnknownChannel", 7)
MalformedFrame = _mk("MalformedFrame", 8)
UnknownHandle = _mk("UnknownHandle", 9)
BackendMismatch = _mk("BackendMismatch", 10)
InvalidContext = _mk("InvalidContext", 11)
ConfigMismatch = _mk("ConfigMismatch", 12)
BootstrapTimeout = _mk("BootstrapTimeout", 13)
RegistrationMismatch = _mk("RegistrationMismatch", 14)
InvalidPeer = _mk("InvalidPeer", 15)
InvalidSignal = _mk("InvalidSignal", 16)
InvalidCounter = _mk("InvalidCounter", 17)
ResetWhileOutstanding = _mk("ResetWhileOutstanding", 18)
Timeout = _mk("Timeout", 19)
VerificationFailure = _mk("VerificationFailure", 20)
FlowControlViolation = _mk("FlowControlViolation", 21)
ChildFailure = _mk("ChildFailure", 22)
UsageError = _mk("UsageError", 23)
CudaError = _mk("CudaError", 24)
_BY_CODE = {c.code: c for c in [InvalidDescriptor, MalformedDescriptor, OutOfBounds, UnknownWindow,
                                 RankOutOfRange, DuplicateEndpoint, UnknownChannel, MalformedFrame,
                                 UnknownHandle, BackendMismatch, InvalidContext, ConfigMismatch,
                                 BootstrapTimeout, RegistrationMismatch, InvalidPeer, InvalidSignal,
                                 InvalidCounter, ResetWhileOutstanding, Timeout, VerificationFailure,
                                 FlowControlViolation, ChildFailure, UsageError, CudaError, Error]}

# --------------------------------------------------------------------- C structs


class Config(ctypes.Structure):
    """runtime.hpp:29-44 (Config); defaults from ginsim_cuda_config_default."""
    _fields_ = [("n_contexts", c_uint32), ("backend", c_uint32), ("signal_cells", c_uint32),
                ("counter_cells", c_uint32), ("queue_depth", c_uint32), ("transport", c_uint32),
                ("timeout_ms", c_uint64)]

    DIRECT = 0
    PROXY = 1
    FABRIC = 0   # transport: NVLink peer mappings / copy engines
    SOCKET = 1   # transport: GIN1 frames over TCP between the ranks' agents (Proxy backend)

    def __init__(self, **kw):
        super().__init__()
        lib().ginsim_cuda_config_default(byref(self)) if _lib_loaded() else self._py_defaults()
        for k, v in kw.items():
            if k == "backend" and isinstance(v, str):
                v = {"direct": 0, "proxy": 1}[v]
            if k == "transport" and isinstance(v, str):
                v = {"fabric": 0, "nvlink": 0, "socket": 1}[v]
            setattr(self, k, v)

    def _py_defaults(self):
        self.n_contexts, self.backend, self.signal_cells, self.counter_cells = 4, 0, 256, 256
        self.queue_depth, self.timeout_ms = 1024, 30000


class Bootstrap(ctypes.Structure):
    _fields_ = [("ctx", c_void_p),
                ("allgather", ctypes.CFUNCTYPE(c_int, c_void_p, c_void_p, c_void_p, c_size_t))]


class Action(ctypes.Structure):
    """CompletionAction (types.hpp:45-72): optional remote signal + local counter."""
    _fields_ = [("signal_id", c_int32), ("signal_add", c_uint32), ("operand", c_uint64),
                ("counter_id", c_int32), ("reserved", c_uint32)]

    @staticmethod
    def make(signal=None, add=None, counter=None):
        a = Action()
        a.signal_id = -1 if signal is None else signal
        a.signal_add = 0 if add is None else 1
        a.operand = 1 if add is None else add
        a.counter_id = -1 if counter is None else counter
        return a


class Descriptor(ctypes.Structure):
    """64-byte proxy descriptor fields (descriptor.hpp:13-27)."""
    _fields_ = [("opcode", c_uint8), ("flags", c_uint8), ("team", c_uint16), ("peer", c_uint32),
                ("dst_window", c_uint32), ("src_window", c_uint32), ("dst_offset", c_uint64),
                ("src_offset_or_value", c_uint64), ("bytes", c_uint64), ("signal_id", c_uint32),
                ("counter_id", c_uint32), ("signal_operand", c_uint64)]

    def astuple(self):
        return tuple(getattr(self, f[0]) for f in self._fields_)


class WireFrame(ctypes.Structure):
    """One GIN1 frame's fields (wire.hpp:12-45); the body travels separately."""
    _fields_ = [("type", c_uint32), ("src_rank", c_uint32), ("ctx", c_uint16), ("pad", c_uint16),
                ("window_or_signal", c_uint32), ("seq_or_watermark", c_uint64), ("dst_offset", c_uint64),
                ("signal_add", c_uint32), ("reserved", c_uint32), ("operand", c_uint64), ("body_bytes", c_uint64)]
    PUT, SIGNAL, ACK, CONTROL = 1, 2, 3, 4


class MoeConfig(ctypes.Structure):
    _fields_ = [("experts", c_uint32), ("top_k", c_uint32), ("tokens", c_uint32), ("hidden", c_uint32),
                ("mode", c_uint32), ("layout", c_uint32), ("ctas", c_uint32), ("engine", c_uint32)]

    def __init__(self, experts=256, top_k=8, tokens=128, hidden=7168, mode=0, layout=0, ctas=0, engine=0):
        super().__init__(experts, top_k, tokens, hidden, mode, layout, ctas, engine)

    @property
    def dispatch_message_bytes(self):  # harness.hpp:112
        return self.hidden * 2 + 16

    @property
    def combine_message_bytes(self):  # harness.hpp:113
        return self.hidden * 2


# --------------------------------------------------------------------- library
_LIB = None
_LOCK = threading.Lock()


def _lib_loaded():
    return _LIB is not None


def lib():
    """The CUDA library.  Raises (never falls back) when it is not built."""
    global _LIB
    if _LIB is not None:
        return _LIB
    with _LOCK:
        if _LIB is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (make -C paper_2511_15076_b200)")
            L = ctypes.CDLL(LIB_PATH)
            _declare(L)
            _LIB = L
    return _LIB


def _declare(L):
    P = c_void_p
    sigs = {
        "ginsim_cuda_last_error": ([], c_char_p),
        "ginsim_cuda_abi_version": ([], c_int),
        "ginsim_cuda_config_default": ([POINTER(Config)], None),
        "ginsim_cuda_config_from_env": ([POINTER(Config)], c_int),
        "ginsim_cuda_inproc_group_create": ([c_uint32, POINTER(P)], c_int),
        "ginsim_cuda_inproc_group_destroy": ([P], c_int),
        "ginsim_cuda_inproc_bootstrap": ([P, c_uint32, POINTER(Bootstrap)], c_int),
        "ginsim_cuda_comm_create": ([c_uint32, c_uint32, c_int, POINTER(Config), POINTER(Bootstrap), POINTER(P)], c_int),
        "ginsim_cuda_comm_create_all": ([c_uint32, POINTER(c_int), POINTER(Config), POINTER(P)], c_int),
        "ginsim_cuda_comm_destroy": ([P], c_int),
        "ginsim_cuda_comm_info": ([P, POINTER(c_uint32), POINTER(c_uint32), POINTER(c_int), POINTER(c_uint32)], c_int),
        "ginsim_cuda_devcomm_view": ([P, POINTER(P)], c_int),
        "ginsim_cuda_comm_config": ([P, POINTER(Config)], c_int),
        "ginsim_cuda_mem_alloc": ([P, c_uint64, POINTER(P)], c_int),
        "ginsim_cuda_mem_free": ([P, P], c_int),
        "ginsim_cuda_window_register": ([P, P, c_uint64, POINTER(c_uint32)], c_int),
        "ginsim_cuda_window_register_all": ([POINTER(P), c_uint32, POINTER(P), POINTER(c_uint64), POINTER(c_uint32)], c_int),
        "ginsim_cuda_moe_create_all": ([POINTER(P), c_uint32, POINTER(MoeConfig), POINTER(P)], c_int),
        "ginsim_cuda_window_size": ([P, c_uint32, c_uint32, POINTER(c_uint64)], c_int),
        "ginsim_cuda_window_ptr": ([P, c_uint32, c_uint32, POINTER(P)], c_int),
        "ginsim_cuda_put": ([P, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint64, c_uint64, POINTER(Action), P], c_int),
        "ginsim_cuda_put_value": ([P, c_uint32, c_uint32, c_uint32, c_uint64, c_uint64, c_uint32, POINTER(Action), P], c_int),
        "ginsim_cuda_signal": ([P, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, POINTER(Action), P], c_int),
        "ginsim_cuda_flush": ([P, c_uint32, P], c_int),
        "ginsim_cuda_read_signal": ([P, c_uint32, POINTER(c_uint64)], c_int),
        "ginsim_cuda_wait_signal": ([P, c_uint32, c_uint64], c_int),
        "ginsim_cuda_reset_signal": ([P, c_uint32], c_int),
        "ginsim_cuda_read_counter": ([P, c_uint32, POINTER(c_uint64)], c_int),
        "ginsim_cuda_wait_counter": ([P, c_uint32, c_uint64], c_int),
        "ginsim_cuda_reset_counter": ([P, c_uint32], c_int),
        "ginsim_cuda_snapshot_cells": ([P, POINTER(c_uint64), POINTER(c_uint64)], c_int),
        "ginsim_cuda_device_error": ([P, POINTER(c_uint32), c_int], c_int),
        "ginsim_cuda_proxy_stats": ([P, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)], c_int),
        "ginsim_cuda_proxy_trace": ([P, POINTER(ctypes.c_double), c_uint32, POINTER(c_uint32)], c_int),
        "ginsim_cuda_descriptor_encode": ([POINTER(Descriptor), POINTER(c_uint8)], c_int),
        "ginsim_cuda_descriptor_decode": ([POINTER(c_uint8), POINTER(Descriptor)], c_int),
        "ginsim_cuda_pingpong": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32,
                                  c_uint32, c_uint32, c_uint32, P, P], c_int),
        "ginsim_cuda_alltoall": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint64, c_uint32, P], c_int),
        "ginsim_cuda_copy_bench": ([P, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint32, c_uint32,
                                    POINTER(ctypes.c_float), P], c_int),
        "ginsim_cuda_copy_bench_ex": ([P, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint32, c_uint32,
                                       c_uint32, POINTER(ctypes.c_float), P], c_int),
        "ginsim_cuda_nvls_enabled": ([P, POINTER(c_int)], c_int),
        "ginsim_cuda_barrier_bench": ([POINTER(P), c_uint32, c_uint32, c_uint32, P, P], c_int),
        "ginsim_cuda_occupy": ([c_int, c_uint32, P, c_uint64, P], c_int),
        "ginsim_cuda_host_op_bench": ([P, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64,
                                       POINTER(ctypes.c_float), P], c_int),
        "ginsim_cuda_ordering_stress": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint32, P], c_int),
        "ginsim_cuda_ring":([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, P], c_int),
        "ginsim_cuda_moe_ht_ring": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, P], c_int),
        "ginsim_cuda_moe_create": ([P, POINTER(MoeConfig), POINTER(P)], c_int),
        "ginsim_cuda_moe_destroy": ([P], c_int),
        "ginsim_cuda_moe_windows": ([P, POINTER(c_uint32), POINTER(c_uint32), POINTER(c_uint32)], c_int),
        "ginsim_cuda_moe_generate": ([P, c_uint64, c_uint32, P, P, P, P], c_int),
        "ginsim_cuda_moe_dispatch": ([POINTER(P), c_uint32, POINTER(P), POINTER(P), P], c_int),
        "ginsim_cuda_moe_combine": ([POINTER(P), c_uint32, POINTER(P), POINTER(P), P], c_int),
        "ginsim_cuda_moe_phase_times": ([P, c_uint32, POINTER(c_uint64), POINTER(c_uint32)], c_int),
        "ginsim_cuda_moe_last_launch": ([P, POINTER(c_uint32), POINTER(c_uint32)], c_int),
        "ginsim_cuda_moe_transport": ([P, POINTER(c_uint32)], c_int),
        "ginsim_cuda_moe_cells": ([P, POINTER(c_uint32), POINTER(c_uint32)], c_int),
        "ginsim_cuda_digest": ([P, c_uint64, c_uint64, P, P], c_int),
        "ginsim_cuda_window_deregister": ([P, c_uint32], c_int),
        "ginsim_cuda_plugin_create": ([P, c_uint32, POINTER(P)], c_int),
        "ginsim_cuda_plugin_destroy": ([P], c_int),
        "ginsim_cuda_rtt_floor": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, P,
                                   P], c_int),
        "ginsim_cuda_bw": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint32,
                            c_uint32, c_uint32, P, P], c_int),
        "ginsim_cuda_signal_broadcast": ([P, c_uint32, c_uint64, P], c_int),
        "ginsim_cuda_read_broadcast": ([P, c_uint32, POINTER(c_uint64)], c_int),
        "ginsim_cuda_team_ring": ([POINTER(P), c_uint32, c_uint32, c_uint32, c_uint32, c_uint64, c_uint32, c_uint32, P],
                                  c_int),
        "ginsim_cuda_register_team": ([P, c_uint32, POINTER(c_uint32), c_uint32], c_int),
        "ginsim_cuda_team": ([P, c_uint32, POINTER(c_uint32), POINTER(c_uint32)], c_int),
        "ginsim_cuda_wire_encode": ([POINTER(WireFrame), P, P, ctypes.c_size_t, POINTER(ctypes.c_size_t)], c_int),
        "ginsim_cuda_wire_parser_create": ([POINTER(P)], c_int),
        "ginsim_cuda_wire_parser_feed": ([P, P, ctypes.c_size_t], c_int),
        "ginsim_cuda_wire_parser_next": ([P, POINTER(WireFrame), P, ctypes.c_size_t, POINTER(c_int)], c_int),
        "ginsim_cuda_wire_parser_buffered": ([P], ctypes.c_size_t),
        "ginsim_cuda_wire_parser_destroy": ([P], c_int),
        "ginsim_cuda_socket_bootstrap_create": ([c_char_p, ctypes.c_uint16, c_uint32, c_uint32, c_uint64,
                                                 POINTER(Bootstrap)], c_int),
        "ginsim_cuda_socket_bootstrap_destroy": ([POINTER(Bootstrap)], c_int),
        "ginsim_cuda_reserve_loopback_port": ([POINTER(ctypes.c_uint16)], c_int),
        "ginsim_cuda_net_stats": ([P, POINTER(c_uint64), POINTER(c_uint64), POINTER(c_uint64)], c_int),
    }
    for name, (args, res) in sigs.items():
        fn = getattr(L, name, None)
        if fn is None and os.environ.get("GINSIM_LIB"):  # an older build loaded for an A/B comparison
            continue
        if fn is None:
            raise ImportError(f"{LIB_PATH} does not export {name}")
        fn.argtypes = args
        fn.restype = res


def exported_symbols():
    """Every entry point include/ginsim_cuda.h declares (for the ABI test)."""
    import re
    hdr = os.path.join(os.path.dirname(_HERE), "include", "ginsim_cuda.h")
    txt = open(hdr).read()
    return sorted(set(re.findall(r"\b(ginsim_cuda_[a-z0-9_]+)\s*\(", txt)))


def check(rc):
    if rc != 0:
        msg = lib().ginsim_cuda_last_error().decode()
        raise _BY_CODE.get(rc, Error)(msg)


def _ptr(x):
    """Device pointer of a torch tensor / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


def _stream(s):
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# --------------------------------------------------------------------- comms


class Comm:
    """One rank's communicator (DevComm, runtime.hpp:123-246) on one GPU."""

    def __init__(self, handle):
        self.h = c_void_p(handle) if isinstance(handle, int) else handle
        r, w, d, b = c_uint32(), c_uint32(), c_int(), c_uint32()
        check(lib().ginsim_cuda_comm_info(self.h, byref(r), byref(w), byref(d), byref(b)))
        self.rank, self.world_size, self.device, self.backend = r.value, w.value, d.value, b.value
        self.config = Config()
        check(lib().ginsim_cuda_comm_config(self.h, byref(self.config)))
        self.n_windows = 0

    # -- construction
    @staticmethod
    def create_all(devices, config=None):
        """All ranks of an in-process group (InProcGroup + comm_init per rank;
        devices may repeat: emulated ranks on one GPU)."""
        n = len(devices)
        devs = (c_int * n)(*devices)
        out = (c_void_p * n)()
        cfg = config or Config()
        check(lib().ginsim_cuda_comm_create_all(n, devs, byref(cfg), out))
        return [Comm(out[i]) for i in range(n)]

    @staticmethod
    def create(rank, world, device, allgather, config=None):
        """comm_init over an external bootstrap: allgather(bytes)->list[bytes]
        (e.g. torch.distributed all_gather_object; bootstrap only)."""
        cfg = config or Config()

        @ctypes.CFUNCTYPE(c_int, c_void_p, c_void_p, c_void_p, c_size_t)
        def _ag(ctx, send, recv, nbytes):
            try:
                mine = ctypes.string_at(send, nbytes)
                parts = allgather(mine)
                blob = b"".join(parts)
                ctypes.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 - reported as BootstrapTimeout
                return 1

        boot = Bootstrap(None, _ag)
        out = c_void_p()
        check(lib().ginsim_cuda_comm_create(rank, world, device, byref(cfg), byref(boot), byref(out)))
        c = Comm(out)
        c._boot_keepalive = (_ag, boot)  # window_register reuses the bootstrap
        return c

    @staticmethod
    def create_socket(host, port, world, rank, device, config=None):
        """comm_init_socket (socket_transport.hpp:117-126): rank 0 hosts the
        rendezvous at host:port (IPv4); the comm runs the Proxy backend with
        the socket transport (GIN1 frames between the ranks' agents)."""
        cfg = config or Config()
        cfg.backend, cfg.transport = Config.PROXY, Config.SOCKET
        boot = Bootstrap()
        check(lib().ginsim_cuda_socket_bootstrap_create(host.encode(), port, world, rank, cfg.timeout_ms, byref(boot)))
        out = c_void_p()
        try:
            check(lib().ginsim_cuda_comm_create(rank, world, device, byref(cfg), byref(boot), byref(out)))
        except Exception:
            lib().ginsim_cuda_socket_bootstrap_destroy(byref(boot))
            raise
        c = Comm(out)
        c._socket_boot = boot  # window_register reuses the bootstrap; freed after the comm
        return c

    def destroy(self):
        if self.h:
            check(lib().ginsim_cuda_comm_destroy(self.h))
            self.h = None
        boot = getattr(self, "_socket_boot", None)
        if boot is not None:
            lib().ginsim_cuda_socket_bootstrap_destroy(byref(boot))
            self._socket_boot = None

    # -- memory and windows
    def mem_alloc(self, nbytes):
        p = c_void_p()
        check(lib().ginsim_cuda_mem_alloc(self.h, nbytes, byref(p)))
        return p.value or 0

    def mem_free(self, ptr):
        check(lib().ginsim_cuda_mem_free(self.h, ptr))

    def window_register(self, ptr, nbytes):
        wid = c_uint32()
        check(lib().ginsim_cuda_window_register(self.h, ptr, nbytes, byref(wid)))
        self.n_windows = max(self.n_windows, wid.value + 1)
        return wid.value

    @staticmethod
    def window_register_all(comms, ptrs, sizes):
        """Collective registration of every rank of an in-process group."""
        n = len(comms)
        wid = c_uint32()
        check(lib().ginsim_cuda_window_register_all(comm_handles(comms), n, (c_void_p * n)(*ptrs),
                                                    (c_uint64 * n)(*sizes), byref(wid)))
        for c in comms:
            c.n_windows = max(c.n_windows, wid.value + 1)
        return wid.value

    def window_deregister(self, win):
        """Release window `win` on this rank (local; ids are reused lowest-first)."""
        check(lib().ginsim_cuda_window_deregister(self.h, win))

    # -- teams (runtime.hpp:145-148)
    def register_team(self, team_id, members):
        m = (c_uint32 * len(members))(*members)
        check(lib().ginsim_cuda_register_team(self.h, team_id, m, len(members)))

    def team(self, team_id):
        m = (c_uint32 * 8)()
        n = c_uint32()
        check(lib().ginsim_cuda_team(self.h, team_id, m, byref(n)))
        return list(m[:n.value])

    def window_size(self, win, rank):
        v = c_uint64()
        check(lib().ginsim_cuda_window_size(self.h, win, rank, byref(v)))
        return v.value

    def window_ptr(self, win, rank):
        p = c_void_p()
        check(lib().ginsim_cuda_window_ptr(self.h, win, rank, byref(p)))
        return p.value or 0

    def view(self):
        p = c_void_p()
        check(lib().ginsim_cuda_devcomm_view(self.h, byref(p)))
        return p.value

    # -- cells (runtime.cpp:404-443)
    def read_signal(self, sid):
        v = c_uint64()
        check(lib().ginsim_cuda_read_signal(self.h, sid, byref(v)))
        return v.value

    def wait_signal(self, sid, expected):
        check(lib().ginsim_cuda_wait_signal(self.h, sid, expected))

    def reset_signal(self, sid):
        check(lib().ginsim_cuda_reset_signal(self.h, sid))

    def read_counter(self, cid):
        v = c_uint64()
        check(lib().ginsim_cuda_read_counter(self.h, cid, byref(v)))
        return v.value

    def wait_counter(self, cid, expected):
        check(lib().ginsim_cuda_wait_counter(self.h, cid, expected))

    def reset_counter(self, cid):
        check(lib().ginsim_cuda_reset_counter(self.h, cid))

    def snapshot_cells(self, signal_cells=None, counter_cells=None):
        """DevComm::snapshot_cells (runtime.hpp:178): every signal and counter cell."""
        s = (c_uint64 * self.config.signal_cells)()
        c = (c_uint64 * self.config.counter_cells)()
        check(lib().ginsim_cuda_snapshot_cells(self.h, s, c))
        return list(s), list(c)

    def device_error(self, clear=True):
        v = c_uint32()
        check(lib().ginsim_cuda_device_error(self.h, byref(v), 1 if clear else 0))
        return v.value

    def check_device(self):
        code = self.device_error(clear=True)
        if code:
            raise _BY_CODE.get(code, Error)(f"device-side error {code} on rank {self.rank}")

    def nvls_enabled(self):
        v = c_int()
        check(lib().ginsim_cuda_nvls_enabled(self.h, byref(v)))
        return bool(v.value)

    def signal_broadcast(self, cell, amount=1, stream=None):
        """+amount on broadcast cell `cell` of every rank (one NVLS multimem.red)."""
        check(lib().ginsim_cuda_signal_broadcast(self.h, cell, amount, _stream(stream)))

    def read_broadcast(self, cell):
        v = c_uint64()
        check(lib().ginsim_cuda_read_broadcast(self.h, cell, byref(v)))
        return v.value

    def proxy_trace(self, max_records=4096):
        """[(bytes, ctx, host_issue_us, dev_start_us, dev_us)] of the agent's copies
        since the last call (GINSIM_PROXY_TRACE=1 at creation)."""
        buf = (ctypes.c_double * (5 * max_records))()
        n = c_uint32()
        check(lib().ginsim_cuda_proxy_trace(self.h, buf, max_records, byref(n)))
        return [tuple(buf[5 * i:5 * i + 5]) for i in range(n.value)]

    def proxy_stats(self):
        a, b, c, d = c_uint64(), c_uint64(), c_uint64(), c_uint64()
        check(lib().ginsim_cuda_proxy_stats(self.h, byref(a), byref(b), byref(c), byref(d)))
        return {"descriptors": a.value, "copies": b.value, "busy_ns": c.value, "wall_ns": d.value}

    def net_stats(self):
        """Socket transport counters of this rank (Config(transport="socket"))."""
        a, b, c = c_uint64(), c_uint64(), c_uint64()
        check(lib().ginsim_cuda_net_stats(self.h, byref(a), byref(b), byref(c)))
        return {"tx_frames": a.value, "rx_puts": b.value, "rx_bytes": c.value}


class Gin:
    """Host-issued per-context handle (runtime.hpp:260-306), executed on the GPU."""

    def __init__(self, comm: Comm, ctx: int = 0, stream=None):
        self.comm, self.ctx, self.stream = comm, ctx, stream

    def put(self, peer, dst_win, dst_off, src_win, src_off, nbytes, signal=None, add=None, counter=None):
        a = Action.make(signal, add, counter)
        check(lib().ginsim_cuda_put(self.comm.h, self.ctx, peer, dst_win, dst_off, src_win, src_off, nbytes,
                                    byref(a), _stream(self.stream)))

    def put_value(self, peer, dst_win, dst_off, value, width, signal=None, add=None, counter=None):
        a = Action.make(signal, add, counter)
        check(lib().ginsim_cuda_put_value(self.comm.h, self.ctx, peer, dst_win, dst_off, value, width,
                                          byref(a), _stream(self.stream)))

    def signal(self, peer, sid, add=None, counter=None):
        a = Action.make(None, None, counter)
        check(lib().ginsim_cuda_signal(self.comm.h, self.ctx, peer, sid, 0 if add is None else 1,
                                       1 if add is None else add, byref(a), _stream(self.stream)))

    def flush(self):
        check(lib().ginsim_cuda_flush(self.comm.h, self.ctx, _stream(self.stream)))

    def read_signal(self, sid):
        return self.comm.read_signal(sid)

    def wait_signal(self, sid, expected):
        self.comm.wait_signal(sid, expected)

    def reset_signal(self, sid):
        self.comm.reset_signal(sid)

    def read_counter(self, cid):
        return self.comm.read_counter(cid)

    def wait_counter(self, cid, expected):
        self.comm.wait_counter(cid, expected)

    def reset_counter(self, cid):
        self.comm.reset_counter(cid)


def pool_select(channel_id: int, n_contexts: int = 4):
    """runtime.hpp:51-58: flat channel id -> (comm index, context index)."""
    return channel_id // n_contexts, channel_id % n_contexts


def digest(records, record_bytes, count, out, stream=None):
    """Per-record digests of `count` records at device pointer `records` into
    the device buffer `out` (count u64): the checker compares them with the
    CPU oracle's (ginsim_cuda_digest, include/ginsim_cuda.h)."""
    check(lib().ginsim_cuda_digest(_ptr(records), record_bytes, count, _ptr(out), _stream(stream)))


def summarize(size, samples_ns):
    """BenchRow of harness_bench.cpp:20-32: p50 = s[n/2], p99 = s[min(n-1, 99n/100)], mean."""
    s = sorted(int(x) for x in samples_ns)
    n = len(s)
    row = {"size_bytes": int(size), "iters": n, "p50_ns": 0, "p99_ns": 0, "mean_ns": 0.0}
    if n:
        row.update(p50_ns=s[n // 2], p99_ns=s[min(n - 1, (n * 99) // 100)], mean_ns=sum(s) / n)
    return row


def write_csv(path, rows, backend="direct", transport="nvlink", seed=0):
    """write_csv (harness_bench.cpp:167-178): the reference's benchmark CSV schema."""
    with open(path, "w") as f:
        f.write("size_bytes,iters,p50_ns,p99_ns,mean_ns,backend,transport,seed\n")
        for r in rows:
            f.write(f"{r['size_bytes']},{r['iters']},{r['p50_ns']},{r['p99_ns']},{r['mean_ns']},{backend},{transport},{seed}\n")


def wire_encode(type, src=0, ctx=0, seq=0, window_or_signal=0, dst_offset=0, signal_add=0, operand=1,
                body=b"") -> bytes:
    """encode_{put,signal,ack,control}_frame (wire.hpp:47-53) through the C ABI."""
    f = WireFrame()
    f.type, f.src_rank, f.ctx, f.seq_or_watermark = type, src, ctx, seq
    f.window_or_signal, f.dst_offset, f.signal_add, f.operand = window_or_signal, dst_offset, signal_add, operand
    f.body_bytes = len(body)
    n = ctypes.c_size_t()
    cap = 64 + len(body)
    out = (c_uint8 * cap)()
    src_buf = (c_uint8 * max(1, len(body))).from_buffer_copy(body or b"\0")
    check(lib().ginsim_cuda_wire_encode(byref(f), src_buf, out, cap, byref(n)))
    return bytes(out[:n.value])


class WireParser:
    """FrameParser (wire.hpp:57-66): feed() bytes as they arrive, next() returns
    (WireFrame, body bytes) or None; MalformedFrame on garbage."""

    def __init__(self):
        self.h = c_void_p()
        check(lib().ginsim_cuda_wire_parser_create(byref(self.h)))

    def feed(self, data: bytes):
        buf = (c_uint8 * max(1, len(data))).from_buffer_copy(data or b"\0")
        check(lib().ginsim_cuda_wire_parser_feed(self.h, buf, len(data)))

    def next(self, body_cap=1 << 20):
        f = WireFrame()
        body = (c_uint8 * max(1, body_cap))()
        ready = c_int()
        check(lib().ginsim_cuda_wire_parser_next(self.h, byref(f), body, body_cap, byref(ready)))
        return (f, bytes(body[:f.body_bytes])) if ready.value else None

    def buffered(self):
        return lib().ginsim_cuda_wire_parser_buffered(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib_loaded():
            lib().ginsim_cuda_wire_parser_destroy(self.h)
            self.h = None


def reserve_loopback_port() -> int:
    p = ctypes.c_uint16()
    check(lib().ginsim_cuda_reserve_loopback_port(byref(p)))
    return p.value


def descriptor_encode(d: Descriptor) -> bytes:
    out = (c_uint8 * 64)()
    check(lib().ginsim_cuda_descriptor_encode(byref(d), out))
    return bytes(out)


def descriptor_decode(buf: bytes) -> Descriptor:
    if len(buf) != 64:
        raise MalformedDescriptor(f"descriptor must be exactly 64 bytes, got {len(buf)}")
    arr = (c_uint8 * 64).from_buffer_copy(buf)
    d = Descriptor()
    check(lib().ginsim_cuda_descriptor_decode(arr, byref(d)))
    return d


def _arr(ptrs):
    return (c_void_p * len(ptrs))(*ptrs)


class Moe:
    """DeepEP-style dispatch/combine engine of one rank (harness_moe.cpp:105-250)."""

    def __init__(self, comm: Comm, cfg: MoeConfig, handle=None):
        self.comm, self.cfg = comm, cfg
        if handle is None:
            handle = c_void_p()
            check(lib().ginsim_cuda_moe_create(comm.h, byref(cfg), byref(handle)))
        self.h = handle if isinstance(handle, c_void_p) else c_void_p(handle)
        h = self.h
        d, c, cb = c_uint32(), c_uint32(), c_uint32()
        check(lib().ginsim_cuda_moe_windows(h, byref(d), byref(c), byref(cb)))
        self.win_dispatch, self.win_counts, self.win_combine = d.value, c.value, cb.value

    @staticmethod
    def create_all(comms, cfg: MoeConfig):
        """moe_create for every rank of an in-process group (collective)."""
        n = len(comms)
        out = (c_void_p * n)()
        check(lib().ginsim_cuda_moe_create_all(comm_handles(comms), n, byref(cfg), out))
        return [Moe(c, cfg, out[i]) for i, c in enumerate(comms)]

    def generate(self, seed, src, x=None, idx=None, weights=None, stream=None):
        check(lib().ginsim_cuda_moe_generate(self.h, seed, src, _ptr(x), _ptr(idx), _ptr(weights), _stream(stream)))

    @staticmethod
    def dispatch(moes, xs, idxs, stream=None):
        n = len(moes)
        check(lib().ginsim_cuda_moe_dispatch(_arr([m.h.value for m in moes]), n, _arr([_ptr(x) for x in xs]),
                                             _arr([_ptr(i) for i in idxs]), _stream(stream)))

    @staticmethod
    def combine(moes, ws, outs, stream=None):
        n = len(moes)
        check(lib().ginsim_cuda_moe_combine(_arr([m.h.value for m in moes]), n, _arr([_ptr(w) for w in ws]),
                                            _arr([_ptr(o) for o in outs]), _stream(stream)))

    def cells(self):
        """(first, span) of the signal cells this handle owns."""
        a, b = c_uint32(), c_uint32()
        check(lib().ginsim_cuda_moe_cells(self.h, byref(a), byref(b)))
        return a.value, b.value

    def last_launch(self):
        a, b = c_uint32(), c_uint32()
        check(lib().ginsim_cuda_moe_last_launch(self.h, byref(a), byref(b)))
        return a.value, b.value

    def transport(self):
        """0 direct, 1 proxy one-shot staging, 2 proxy pipeline."""
        k = c_uint32()
        check(lib().ginsim_cuda_moe_transport(self.h, byref(k)))
        return k.value

    def pipelined(self):
        return self.transport() == 2

    def phase_times(self, kernel):
        """[ctas][8] %globaltimer stamps of the last launch of `kernel` (0 dispatch,
        1 combine send, 2 reduce); needs GINSIM_PROFILE_PHASES=1 at creation."""
        import numpy as np
        buf = (c_uint64 * (1024 * 8))()
        g = c_uint32()
        check(lib().ginsim_cuda_moe_phase_times(self.h, kernel, buf, byref(g)))
        return np.frombuffer(buf, dtype=np.uint64).reshape(1024, 8)[:g.value].copy()

    def destroy(self):
        if self.h:
            check(lib().ginsim_cuda_moe_destroy(self.h))
            self.h = None


def comm_handles(comms):
    return _arr([c.h.value if isinstance(c.h, c_void_p) else c.h for c in comms])
