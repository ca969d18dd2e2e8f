/*
 * ginsim_cuda.h — the C-ABI drop-in boundary of the B200-native GIN hot path.
 *
 * Plain C: integer status codes, plain pointers and sizes, no C++ or torch
 * types.  Every entry point names the reference interface it replaces
 * (/root/reference-relative file:line).  The reference is C++; a maintainer
 * binds this header from ginsim's own classes as INTEGRATION.md shows (the
 * C++ host layer in include/ginsim/*.hpp is exactly that binding).
 *
 * Error convention: every function returns a ginsim_status; on failure the
 * thread-local ginsim_cuda_last_error() holds the message.  The codes mirror
 * the reference's typed exceptions (proj/core/include/ginsim/errors.hpp:24-52)
 * one to one so the C++ layer can rethrow the same type.
 *
 * Threading: a comm may be used from any host thread (runtime.hpp:128-134);
 * collective calls (comm_create, window_register) must be entered by every
 * rank of the comm, in the same order (runtime.cpp:128-175).
 */
#ifndef GINSIM_CUDA_H
#define GINSIM_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GINSIM_CUDA_ABI_VERSION 1

typedef enum ginsim_status {
  GINSIM_OK = 0,
  GINSIM_E_INVALID_DESCRIPTOR = 1,   /* errors.hpp:25 InvalidDescriptor */
  GINSIM_E_MALFORMED_DESCRIPTOR = 2, /* errors.hpp:26 */
  GINSIM_E_OUT_OF_BOUNDS = 3,        /* errors.hpp:27 */
  GINSIM_E_UNKNOWN_WINDOW = 4,       /* errors.hpp:28 */
  GINSIM_E_RANK_OUT_OF_RANGE = 5,    /* errors.hpp:29 */
  GINSIM_E_DUPLICATE_ENDPOINT = 6,   /* errors.hpp:32 */
  GINSIM_E_UNKNOWN_CHANNEL = 7,      /* errors.hpp:33 */
  GINSIM_E_MALFORMED_FRAME = 8,      /* errors.hpp:34 */
  GINSIM_E_UNKNOWN_HANDLE = 9,       /* errors.hpp:37 */
  GINSIM_E_BACKEND_MISMATCH = 10,    /* errors.hpp:38 */
  GINSIM_E_INVALID_CONTEXT = 11,     /* errors.hpp:39 */
  GINSIM_E_CONFIG_MISMATCH = 12,     /* errors.hpp:42 */
  GINSIM_E_BOOTSTRAP_TIMEOUT = 13,   /* errors.hpp:43 */
  GINSIM_E_REGISTRATION_MISMATCH = 14, /* errors.hpp:44 */
  GINSIM_E_INVALID_PEER = 15,        /* errors.hpp:45 */
  GINSIM_E_INVALID_SIGNAL = 16,      /* errors.hpp:46 */
  GINSIM_E_INVALID_COUNTER = 17,     /* errors.hpp:47 */
  GINSIM_E_RESET_WHILE_OUTSTANDING = 18, /* errors.hpp:48 */
  GINSIM_E_TIMEOUT = 19,             /* errors.hpp:49 */
  GINSIM_E_VERIFICATION_FAILURE = 20, /* errors.hpp:52 */
  GINSIM_E_FLOW_CONTROL_VIOLATION = 21, /* errors.hpp:53 */
  GINSIM_E_CHILD_FAILURE = 22,       /* errors.hpp:54 */
  GINSIM_E_USAGE = 23,               /* errors.hpp:55 UsageError */
  GINSIM_E_CUDA = 24,                /* a CUDA runtime/driver call failed */
  GINSIM_E_GENERIC = 25              /* plain ginsim::Error */
} ginsim_status;

/* Thread-local message of the last failure on this thread (never NULL). */
const char* ginsim_cuda_last_error(void);
int ginsim_cuda_abi_version(void);

/* ---------------------------------------------------------------- config
 * proj/core/include/ginsim/runtime.hpp:29-44 (Config).  Latency-model fields
 * of the simulator have no meaning on hardware and are absent. */
typedef struct ginsim_cuda_config {
  uint32_t n_contexts;    /* default 4 */
  uint32_t backend;       /* 0 = direct (NVLink stores), 1 = proxy (GPU->CPU ring) */
  uint32_t signal_cells;  /* default 256; top 64 reserved for barriers */
  uint32_t counter_cells; /* default 256 */
  uint32_t queue_depth;   /* proxy ring capacity per context, power of two; default 1024 */
  uint32_t transport;     /* proxy backend: 0 = the fabric (NVLink peer mappings, copy engines),
                             1 = socket: GIN1 frames over TCP between the ranks' host agents
                             (the reference's SocketTransport, socket_transport.cpp:498-590) */
  uint64_t timeout_ms;    /* default 30000 */
} ginsim_cuda_config;

/* Config{} defaults (runtime.hpp:29-44). */
void ginsim_cuda_config_default(ginsim_cuda_config* cfg);
/* config_from_env (runtime.cpp:42-60): GINSIM_BACKEND / GINSIM_QUEUE_DEPTH /
 * GINSIM_TIMEOUT_MS.  USAGE on an unparsable value. */
int ginsim_cuda_config_from_env(ginsim_cuda_config* cfg);

/* ---------------------------------------------------------------- bootstrap
 * Out-of-band exchange used only during comm/window setup (NCCL or an
 * in-process group; never on the data path).  allgather: every rank passes
 * `bytes` bytes; recv receives world*bytes, rank-major.  Returns 0 on success. */
typedef struct ginsim_cuda_bootstrap {
  void* ctx;
  int (*allgather)(void* ctx, const void* send, void* recv, size_t bytes);
} ginsim_cuda_bootstrap;

/* comm_init_socket's rendezvous (socket_transport.hpp:117-126,
 * socket_transport.cpp:178-231): rank 0 listens on host:port (IPv4), every
 * other rank connects to it; the returned bootstrap's allgather gathers to
 * rank 0 and broadcasts back.  Keep it alive as long as the comm (window
 * registration is collective over it); destroy it after the comm. */
int ginsim_cuda_socket_bootstrap_create(const char* host, uint16_t port, uint32_t world, uint32_t rank,
                                        uint64_t timeout_ms, ginsim_cuda_bootstrap* out);
int ginsim_cuda_socket_bootstrap_destroy(ginsim_cuda_bootstrap* boot);
/* reserve_loopback_port (socket_transport.hpp:128-129): a currently free
 * loopback TCP port for a launcher. */
int ginsim_cuda_reserve_loopback_port(uint16_t* port);

typedef struct ginsim_cuda_group_s* ginsim_cuda_group_t;
typedef struct ginsim_cuda_comm_s* ginsim_cuda_comm_t;

/* InProcGroup::create (runtime.hpp:73).  Ranks are host threads of this
 * process (one per GPU, or several emulated ranks sharing one GPU). */
int ginsim_cuda_inproc_group_create(uint32_t world_size, ginsim_cuda_group_t* out);
int ginsim_cuda_inproc_group_destroy(ginsim_cuda_group_t group);
/* A bootstrap vtable for `rank` of an in-process group. */
int ginsim_cuda_inproc_bootstrap(ginsim_cuda_group_t group, uint32_t rank, ginsim_cuda_bootstrap* out);

/* comm_init (runtime.hpp:251-252, runtime.cpp:582-599).  Collective.
 * Allocates this rank's signal/counter tables on `device`, exchanges and maps
 * every peer's signal table, starts the proxy agent when backend == proxy.
 * CONFIG_MISMATCH when ranks disagree on cfg (runtime.cpp:86-105). */
int ginsim_cuda_comm_create(uint32_t rank, uint32_t world_size, int device,
                            const ginsim_cuda_config* cfg, const ginsim_cuda_bootstrap* boot,
                            ginsim_cuda_comm_t* out);
/* Convenience for tests and single-process launchers (harness_launch.cpp:16-63):
 * creates all `world_size` comms of a fresh in-process group, one host thread
 * per rank.  devices[r] may repeat (emulated ranks on one GPU). */
int ginsim_cuda_comm_create_all(uint32_t world_size, const int* devices,
                                const ginsim_cuda_config* cfg, ginsim_cuda_comm_t* out);
int ginsim_cuda_comm_destroy(ginsim_cuda_comm_t comm);
int ginsim_cuda_comm_info(ginsim_cuda_comm_t comm, uint32_t* rank, uint32_t* world, int* device,
                          uint32_t* backend);
/* DevComm::config (runtime.hpp:131): the config the comm was created with. */
int ginsim_cuda_comm_config(ginsim_cuda_comm_t comm, ginsim_cuda_config* out);
/* Device pointer to the GinDevCommView kernels take (the ncclDevComm analogue). */
int ginsim_cuda_devcomm_view(ginsim_cuda_comm_t comm, const void** device_view);

/* ---------------------------------------------------------------- memory
 * gin_mem_alloc: cuMemCreate + cuMemMap on the comm's device
 * with a POSIX-FD shareable handle so peers can map it.  Zero-filled. */
int ginsim_cuda_mem_alloc(ginsim_cuda_comm_t comm, uint64_t bytes, void** ptr);
int ginsim_cuda_mem_free(ginsim_cuda_comm_t comm, void* ptr);

/* DevComm::window_register (runtime.hpp:141, runtime.cpp:347-371).  Collective:
 * every rank contributes `bytes` at `local` (from ginsim_cuda_mem_alloc; or
 * any device pointer when every rank lives in this process; or HOST memory --
 * e.g. a std::vector, as the reference's host programs register -- which is
 * pinned and mapped with cudaHostRegister so device ops reach it over PCIe
 * while the host reads and writes it directly, in-process ranks only); sizes
 * may differ, 0 is allowed.  Dense ids in call order on every rank;
 * REGISTRATION_MISMATCH when ranks disagree on the id. */
int ginsim_cuda_window_register(ginsim_cuda_comm_t comm, void* local, uint64_t bytes, uint32_t* window_id);
/* Collective registration for every rank of an in-process group from one
 * caller thread (one helper thread per rank, like the reference's launcher,
 * harness_launch.cpp:16-63).  ptrs[r]/bytes[r] as for window_register. */
int ginsim_cuda_window_register_all(const ginsim_cuda_comm_t* comms, uint32_t n, void* const* ptrs,
                                    const uint64_t* bytes, uint32_t* window_id);
/* Releases window `window_id` on this rank (no reference counterpart: the
 * reference never deregisters; SURVEY.md §8(b) lists it for GPU memory
 * lifetime).  Local, not collective: waits for this rank's device work, then
 * unmaps the peer regions imported for the window and frees the id, which the
 * next window_register reuses (lowest free id first), so ranks that register
 * and deregister in the same order keep agreeing on ids.  Every rank must
 * deregister before any rank registers a window into the freed id.  The local
 * bytes stay owned by the caller (free them with ginsim_cuda_mem_free after
 * every rank has deregistered).  UNKNOWN_WINDOW if not registered. */
int ginsim_cuda_window_deregister(ginsim_cuda_comm_t comm, uint32_t window_id);
/* Window::size_of (types.hpp:105) and the peer mapping of rank's region. */
int ginsim_cuda_window_size(ginsim_cuda_comm_t comm, uint32_t window_id, uint32_t rank, uint64_t* bytes);
int ginsim_cuda_window_ptr(ginsim_cuda_comm_t comm, uint32_t window_id, uint32_t rank, void** ptr);

/* ---------------------------------------------------------------- teams
 * DevComm::register_team / team (runtime.hpp:145-148, runtime.cpp:329-343).
 * Local.  The world team (id 0, identity) is always present.  members[i] is
 * the world rank of team rank i.  USAGE on an empty team, a duplicate id or a
 * full table (16 teams); INVALID_PEER for a member outside the world.  The
 * device API's gin::Gin::team(id) returns the registered team; on the Proxy
 * backend descriptors carry (team id, team-relative peer) and the host agent
 * resolves the world rank (proxy_backend.cpp:72). */
int ginsim_cuda_register_team(ginsim_cuda_comm_t comm, uint32_t team_id, const uint32_t* members, uint32_t n);
/* members[] receives up to 8 world ranks; USAGE if the id is not registered. */
int ginsim_cuda_team(ginsim_cuda_comm_t comm, uint32_t team_id, uint32_t* members, uint32_t* n);

/* ---------------------------------------------------------------- host ops
 * Host-issued one-sided ops (Gin, runtime.hpp:260-306), executed on the GPU
 * in stream order: the direct backend runs them as a one-warp device op, the
 * proxy backend hands them to the host agent.  `stream` is a cudaStream_t of
 * the comm's device (NULL = legacy default stream). */
typedef struct ginsim_cuda_action {
  int32_t signal_id;   /* -1 none */
  uint32_t signal_add; /* 0 = SignalInc, 1 = SignalAdd(operand) */
  uint64_t operand;
  int32_t counter_id;  /* -1 none */
  uint32_t reserved;
} ginsim_cuda_action;

int ginsim_cuda_put(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t dst_window,
                    uint64_t dst_offset, uint32_t src_window, uint64_t src_offset, uint64_t bytes,
                    const ginsim_cuda_action* action, void* stream);
int ginsim_cuda_put_value(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t dst_window,
                          uint64_t dst_offset, uint64_t le_value, uint32_t width,
                          const ginsim_cuda_action* action, void* stream);
int ginsim_cuda_signal(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t signal_id,
                       uint32_t signal_add, uint64_t operand, const ginsim_cuda_action* extra,
                       void* stream);
/* DevComm::flush (runtime.cpp:460-470): local completion of ctx's ops. */
int ginsim_cuda_flush(ginsim_cuda_comm_t comm, uint32_t ctx, void* stream);
/* Cells (runtime.cpp:404-443).  read/snapshot synchronise the device. */
int ginsim_cuda_read_signal(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value);
int ginsim_cuda_wait_signal(ginsim_cuda_comm_t comm, uint32_t id, uint64_t expected);
int ginsim_cuda_reset_signal(ginsim_cuda_comm_t comm, uint32_t id);
int ginsim_cuda_read_counter(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value);
int ginsim_cuda_wait_counter(ginsim_cuda_comm_t comm, uint32_t id, uint64_t expected);
int ginsim_cuda_reset_counter(ginsim_cuda_comm_t comm, uint32_t id);
/* DevComm::snapshot_cells (runtime.hpp:178): signal_cells + counter_cells u64. */
int ginsim_cuda_snapshot_cells(ginsim_cuda_comm_t comm, uint64_t* signals, uint64_t* counters);
/* Device error word (device-side Timeout / OutOfBounds ...), 0 if clean;
 * clear != 0 resets it. */
int ginsim_cuda_device_error(ginsim_cuda_comm_t comm, uint32_t* code, int clear);
/* Socket transport (Config.transport = 1) statistics of this rank: frames
 * sent, puts and payload bytes received and performed.  USAGE on a comm that
 * uses the fabric. */
int ginsim_cuda_net_stats(ginsim_cuda_comm_t comm, uint64_t* tx_frames, uint64_t* rx_puts, uint64_t* rx_bytes);

/* Proxy agent statistics: descriptors consumed, memcpy calls issued. */
/* Diagnostics (GINSIM_PROXY_TRACE=1 at comm creation): per agent copy
 * {bytes, ctx, host issue us, device start us, device duration us} since the
 * first traced copy, 5 doubles per record; clears the trace. */
int ginsim_cuda_proxy_trace(ginsim_cuda_comm_t comm, double* out, uint32_t max_records, uint32_t* n_out);

int ginsim_cuda_proxy_stats(ginsim_cuda_comm_t comm, uint64_t* descriptors, uint64_t* copies,
                            uint64_t* busy_ns, uint64_t* wall_ns);

/* ---------------------------------------------------------------- plugin boundary
 * FabricPlugin (proj/core/include/ginsim/plugin.hpp:64-144, plugin.cpp:18-172)
 * and DirectContext (direct_backend.hpp:17-63, direct_backend.cpp:7-57), so a
 * host runtime written against the reference's plugin interface drives the
 * GPU backends.  The semantics must match the comm's backend (0 direct,
 * 1 proxy); a call of the other semantics raises BACKEND_MISMATCH.
 * Memory-region handles are the window ids (reg_mr is idempotent). */
typedef struct ginsim_cuda_plugin_s* ginsim_cuda_plugin_t;
typedef struct ginsim_cuda_direct_ctx_s* ginsim_cuda_direct_ctx_t;

/* PutSource (plugin.hpp:39-46): a registered window range, or <= 8 inline
 * little-endian bytes carried in the descriptor. */
typedef struct ginsim_cuda_put_source {
  uint32_t is_inline;
  uint32_t mr;          /* source window (when !is_inline) */
  uint64_t offset;      /* in the source window */
  uint64_t inline_value;
} ginsim_cuda_put_source;

/* ResolvedOp (direct_backend.hpp:17-27): team translation already applied. */
typedef struct ginsim_cuda_resolved_op {
  uint32_t opcode;      /* 1 PUT, 2 PUT_INLINE, 3 SIGNAL_ONLY */
  uint32_t peer;        /* world rank */
  uint32_t dst_window;
  uint32_t src_window;  /* 0xFFFFFFFF inline */
  uint64_t dst_offset;
  uint64_t src_offset_or_value;
  uint64_t bytes;
  ginsim_cuda_action action;
} ginsim_cuda_resolved_op;

int ginsim_cuda_plugin_create(ginsim_cuda_comm_t comm, uint32_t semantics, ginsim_cuda_plugin_t* out);
int ginsim_cuda_plugin_destroy(ginsim_cuda_plugin_t plugin);
/* reg_mr (plugin.hpp:78): idempotent; UNKNOWN_WINDOW if the window is not registered. */
int ginsim_cuda_plugin_reg_mr(ginsim_cuda_plugin_t plugin, uint32_t window_id, uint32_t* mr);
int ginsim_cuda_plugin_is_registered(ginsim_cuda_plugin_t plugin, uint32_t window_id, int* registered);
/* iput / iput_signal (plugin.hpp:86-90), proxy semantics: the op goes to the
 * comm's host agent (copy engine + stream-memop signal/counter after the
 * copy); *request is unique until retired.  iput with a remote signal in
 * `action` is GENERIC ("use iput_signal"); UNKNOWN_WINDOW for an unregistered
 * mr; OUT_OF_BOUNDS / INVALID_PEER / INVALID_CONTEXT as submit_op. */
int ginsim_cuda_plugin_iput(ginsim_cuda_plugin_t plugin, const ginsim_cuda_put_source* src, uint32_t dst_mr,
                            uint64_t dst_offset, uint64_t bytes, uint32_t peer, uint32_t ctx,
                            const ginsim_cuda_action* action, uint64_t* request);
int ginsim_cuda_plugin_iput_signal(ginsim_cuda_plugin_t plugin, const ginsim_cuda_put_source* src, uint32_t dst_mr,
                                   uint64_t dst_offset, uint64_t bytes, uint32_t peer, uint32_t ctx,
                                   uint32_t signal_id, uint32_t signal_add, uint64_t operand,
                                   const ginsim_cuda_action* action, uint64_t* request);
/* test (plugin.hpp:93): *done = 1 once the request's put has completed
 * (idempotent); UNKNOWN_HANDLE for an unknown or retired id. */
int ginsim_cuda_plugin_test(ginsim_cuda_plugin_t plugin, uint64_t request, int* done);
/* retire (plugin.hpp:97): releases a completed request and returns its
 * completion action; UNKNOWN_HANDLE if unknown/retired, GENERIC before completion. */
int ginsim_cuda_plugin_retire(ginsim_cuda_plugin_t plugin, uint64_t request, ginsim_cuda_action* action);
int ginsim_cuda_plugin_outstanding(ginsim_cuda_plugin_t plugin, uint64_t* requests);
/* Posting trace through the boundary, for tests (PluginCall, plugin.hpp:48-55,
 * plugin.cpp:174-188): op 'p' = put, 's' = put with a remote signal; issuer =
 * a hash of the posting thread's id.  Enabling clears the log; *n = calls
 * recorded (the first max_calls are copied). */
typedef struct ginsim_cuda_plugin_call {
  char op;
  uint8_t pad[3];
  uint32_t ctx;
  uint32_t peer;
  uint32_t pad2;
  uint64_t bytes;
  uint64_t issuer;
} ginsim_cuda_plugin_call;
int ginsim_cuda_plugin_set_call_log(ginsim_cuda_plugin_t plugin, int enabled);
int ginsim_cuda_plugin_call_log(ginsim_cuda_plugin_t plugin, ginsim_cuda_plugin_call* out, uint32_t max_calls,
                                uint32_t* n);
/* create_context (plugin.hpp:105), direct semantics: the posting object of
 * context ctx (one CUDA stream); INVALID_CONTEXT when ctx >= n_contexts. */
int ginsim_cuda_plugin_create_context(ginsim_cuda_plugin_t plugin, uint32_t ctx, ginsim_cuda_direct_ctx_t* out);
/* DirectContext::post / poll / outstanding (direct_backend.cpp:11-57): post
 * launches the op on the context's stream (NVLink stores, red.release.sys
 * signal, counter bump on the device); poll retires the ops the stream has
 * executed (*retired = how many); outstanding = posted minus retired. */
int ginsim_cuda_direct_post(ginsim_cuda_direct_ctx_t ctx, const ginsim_cuda_resolved_op* op);
int ginsim_cuda_direct_poll(ginsim_cuda_direct_ctx_t ctx, uint64_t* retired);
int ginsim_cuda_direct_outstanding(ginsim_cuda_direct_ctx_t ctx, uint64_t* outstanding);

/* ---------------------------------------------------------------- GIN1 wire codec
 * The socket transport's framing (proj/core/include/ginsim/wire.hpp:12-67,
 * proj/core/src/wire.cpp), little-endian, one frame per message:
 *   header 21 B: magic u32 0x474E4931 "GIN1" | type u8 | src u32 | ctx u16 |
 *                pad u16 = 0 | seq_or_watermark u64
 *   PUT     (1): dst_window u32 | dst_offset u64 | len u64 | payload
 *   SIGNAL  (2): signal_id u32 | op u8 (0 inc, 1 add) | pad 3 | operand u64 (1 for inc)
 *   ACK     (3): (the seq field suffices)
 *   CONTROL (4): len u64 | blob
 * The Proxy backend's socket transport (Config.transport = 1) speaks it; the
 * codec is exported for tests and for a host that bridges frames itself. */
#define GINSIM_WIRE_MAGIC 0x474E4931u
#define GINSIM_WIRE_HEADER_BYTES 21
enum { GINSIM_WIRE_PUT = 1, GINSIM_WIRE_SIGNAL = 2, GINSIM_WIRE_ACK = 3, GINSIM_WIRE_CONTROL = 4 };
typedef struct ginsim_cuda_wire_frame {
  uint32_t type;             /* GINSIM_WIRE_* */
  uint32_t src_rank;
  uint16_t ctx;
  uint16_t pad;
  uint32_t window_or_signal; /* PUT: dst_window; SIGNAL: signal_id */
  uint64_t seq_or_watermark;
  uint64_t dst_offset;       /* PUT */
  uint32_t signal_add;       /* SIGNAL: 0 inc, 1 add */
  uint32_t reserved;
  uint64_t operand;          /* SIGNAL: the amount (encode ignores it for inc and writes 1) */
  uint64_t body_bytes;       /* PUT payload / CONTROL blob length */
} ginsim_cuda_wire_frame;
/* encode_put_frame / encode_signal_frame / encode_ack_frame /
 * encode_control_frame (wire.hpp:47-53): writes the frame (header + body)
 * into out; *len = its size.  USAGE when cap < *len (with *len set). */
int ginsim_cuda_wire_encode(const ginsim_cuda_wire_frame* f, const void* body, void* out, size_t cap, size_t* len);
/* FrameParser (wire.hpp:57-66): an incremental decoder over a byte stream;
 * frames may arrive split or coalesced.  next(): *ready = 1 and the frame
 * (its body copied to `body`) when one is whole; *ready = 0 when more bytes
 * are needed; MALFORMED_FRAME on a bad magic, type, padding or signal op;
 * USAGE (nothing consumed, f->body_bytes = the body size) when body_cap is
 * too small. */
typedef struct ginsim_cuda_wire_parser_s* ginsim_cuda_wire_parser_t;
int ginsim_cuda_wire_parser_create(ginsim_cuda_wire_parser_t* out);
int ginsim_cuda_wire_parser_feed(ginsim_cuda_wire_parser_t p, const void* data, size_t n);
int ginsim_cuda_wire_parser_next(ginsim_cuda_wire_parser_t p, ginsim_cuda_wire_frame* f, void* body, size_t body_cap,
                                 int* ready);
size_t ginsim_cuda_wire_parser_buffered(ginsim_cuda_wire_parser_t p);
int ginsim_cuda_wire_parser_destroy(ginsim_cuda_wire_parser_t p);

/* ---------------------------------------------------------------- descriptor codec
 * proj/core/src/descriptor.cpp:148-199 (encode_descriptor / decode_descriptor),
 * 64-byte little-endian layout of descriptor.hpp:13-27. */
typedef struct ginsim_cuda_descriptor {
  uint8_t opcode;   /* 1 PUT, 2 PUT_INLINE, 3 SIGNAL_ONLY */
  uint8_t flags;    /* bit0 HAS_SIGNAL, bit1 SIGNAL_IS_ADD, bit2 HAS_COUNTER */
  uint16_t team;
  uint32_t peer;
  uint32_t dst_window;
  uint32_t src_window; /* 0xFFFFFFFF = inline */
  uint64_t dst_offset;
  uint64_t src_offset_or_value;
  uint64_t bytes;
  uint32_t signal_id;
  uint32_t counter_id;
  uint64_t signal_operand;
} ginsim_cuda_descriptor;
/* INVALID_DESCRIPTOR when d violates an invariant (descriptor.cpp:32-60). */
int ginsim_cuda_descriptor_encode(const ginsim_cuda_descriptor* d, uint8_t out[64]);
/* MALFORMED_DESCRIPTOR on unknown opcode / nonzero reserved / bad fields. */
int ginsim_cuda_descriptor_decode(const uint8_t in[64], ginsim_cuda_descriptor* d);

/* ---------------------------------------------------------------- kernels
 * All launchers take an array of `n` comms driven by this process: n == 1
 * for one rank per process; n > 1 requires every comm on one device and runs
 * them as emulated ranks in ONE cooperative launch (blocks of different
 * ranks wait on one another, so they must be co-resident).  Streams are per
 * call (one per comm device). */

/* put+signal ping-pong (harness_bench.cpp:47-90, K14): rank 0 of the pair
 * puts `bytes` with SignalInc to rank 1 and waits for the echo, `iters`
 * timed iterations after `warmup`; a single persistent CTA per rank times
 * every round trip with %globaltimer into rtt_ns_out (device, iters u64,
 * written by rank 0).  window `send_win` / `recv_win` of >= bytes.  Cells
 * signal_id (rounds) and signal_id+1 (a launch handshake, so no ping can
 * precede the peer's host read of the round cell) are the ping-pong's own. */
int ginsim_cuda_pingpong(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1,
                         uint32_t send_win, uint32_t recv_win, uint64_t bytes, uint32_t iters,
                         uint32_t warmup, uint32_t signal_id, uint32_t threads, uint64_t* rtt_ns_out,
                         void* stream);

/* Raw NVLink round-trip floor: one thread per rank flips
 * a flag word in the peer's signal table and polls its own -- no put, no API.
 * mode 0 = st.release.sys / ld.acquire.sys polls, mode 1 = relaxed .sys (no
 * ordering), mode 2 = st.release.sys / relaxed polls + one acquire fence,
 * mode 3 = red.release.sys.add (the signal path) / relaxed polls + one fence.  rtt_ns_out as for ping-pong (iters u64, written by peer0).
 * Cells signal_id (the flag) and signal_id+1 (a launch handshake) must be
 * dedicated to it. */
int ginsim_cuda_rtt_floor(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1, uint32_t mode,
                          uint32_t iters, uint32_t warmup, uint32_t signal_id, uint64_t* rtt_ns_out, void* stream);

/* Windowed put bandwidth (bw_rank_program, harness_bench.cpp:92-129): rank
 * peer0 puts `window` messages of `bytes` into peer1's recv_win at w*bytes,
 * then flushes; ns_out[i] (device, iters u64) = time of timed iteration i
 * (window puts + flush) after `warmup`.  The puts of an iteration are split
 * over `ctas` CTAs (0 = auto: 256 KiB per CTA, at most one per SM). */
int ginsim_cuda_bw(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1, uint32_t send_win,
                   uint32_t recv_win, uint64_t bytes, uint32_t window, uint32_t iters, uint32_t warmup, uint32_t ctas,
                   uint64_t* ns_out, void* stream);

/* Roofline probe: copy `bytes` from this rank's src window into `peer`'s dst
 * window (peer == own rank: local HBM copy) `iters` times with the put path's
 * engines (0 = 128-bit LSU stores, 1 = TMA bulk copies through shared
 * memory); *ms_out = mean milliseconds per copy.  No signals. */
int ginsim_cuda_copy_bench(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                           uint64_t bytes, uint32_t engine, uint32_t ctas, uint32_t iters, float* ms_out,
                           void* stream);

/* Extended roofline probe: engine 0 = LSU 128-bit, 1 = TMA load+store with
 * `chunk`-byte stages, 2 = LSU 256-bit, 3 = copy engine (cudaMemcpyAsync over
 * the peer mapping), 4 = TMA store-only (write path alone, no reads),
 * 5 = TMA pull (bulk-load the peer's src window, store into this rank's dst
 * window), 6 = hybrid push (copy engine moves the last GINSIM_HYBRID_CE_PCT %
 * on a side stream while TMA copies the rest), 7 = LSU 256-bit pull. */
int ginsim_cuda_copy_bench_ex(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                              uint64_t bytes, uint32_t engine, uint32_t ctas, uint32_t chunk, uint32_t iters,
                              float* ms_out, void* stream);

/* Host-issued operation cost (the proxy agent's building blocks): n_ops
 * 64-bit stream memops (kind 0, `batch` per cuStreamBatchMemOp) or copies
 * (kind 1, cudaMemcpyAsync of `bytes` each) into `peer`'s dst window.
 * out[0] = device microseconds per op, out[1] = host microseconds per op. */
int ginsim_cuda_host_op_bench(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                              uint32_t kind, uint32_t n_ops, uint32_t batch, uint64_t bytes, float* out,
                              void* stream);

/* Launches a kernel that holds every SM (ctas_per_sm x 1024 threads per SM,
 * 1..2) until *release_word (host-mapped) becomes nonzero or timeout_ms
 * passes: the proxy agent's copies and memops must progress meanwhile. */
int ginsim_cuda_occupy(int device, uint32_t ctas_per_sm, const uint32_t* release_word, uint64_t timeout_ms,
                       void* stream);

/* One-sided all-to-all via put+signal: every rank puts
 * `bytes_per_peer` from send_win[dst*M] to dst's recv_win[src*M] and signals
 * `signal_id` on dst; then waits until the cell >= expected. */
int ginsim_cuda_alltoall(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t send_win,
                         uint32_t recv_win, uint64_t bytes_per_peer, uint32_t signal_id,
                         uint64_t expected, uint32_t ctas, void* stream);

/* Ordering stress (acceptance #1, acceptance.cpp:63-118): `channels` parallel
 * (ctx, rank -> right neighbour) channels, each `rounds` puts of `bytes` with
 * SignalAdd(1) into a 2-slot ring; receivers acquire the signal and verify
 * every byte, then return a credit.  VERIFICATION_FAILURE when a signal was
 * observed before the put it follows.  Windows: 2 * channels * bytes. */
int ginsim_cuda_ordering_stress(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t src_win, uint32_t dst_win,
                                uint64_t bytes, uint32_t channels, uint32_t rounds, void* stream);

/* Ring exchange (harness_ring.cpp:18-57) on the device: `rounds` rounds of
 * put+SignalInc to (r+1)%n, wait, verify the (rank, round) pattern, reset,
 * flush, barrier.  VERIFICATION_FAILURE through the device error word. */
int ginsim_cuda_ring(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t send_win,
                     uint32_t recv_win, uint64_t bytes, uint32_t rounds, void* stream);

/* The same ring over a registered team (team_id 0 = world): team rank i puts
 * to team rank (i+1) % |team| with SignalInc on `signal_id` and syncs a
 * BarrierSession over the team; non-members return at once.  The device
 * validates the op (submit_op, runtime.cpp:474-507): an out-of-range
 * signal_id raises INVALID_SIGNAL, an unregistered team RANK_OUT_OF_RANGE. */
int ginsim_cuda_team_ring(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t team_id, uint32_t send_win,
                          uint32_t recv_win, uint64_t bytes, uint32_t rounds, uint32_t signal_id, void* stream);

/* moe-ht circular-buffer flow control (harness_moe.cpp:283-382) on the
 * device: `channels` channels, `slots`-deep rings of 256-byte stamped slots,
 * `messages` per channel; head/tail signals and stage counters exactly as the
 * reference maps them through pool_select (runtime.hpp:51-58).  Each rank's
 * pool of comms is comms_pool[r*n_pool .. +n_pool) with windows recv/stage
 * registered in order (2 per comm).  One CTA per channel. */
int ginsim_cuda_moe_ht_ring(const ginsim_cuda_comm_t* comms_pool, uint32_t n, uint32_t n_pool,
                            uint32_t channels, uint32_t slots, uint32_t messages, uint64_t seed,
                            void* stream);

/* ---- NVLink SHARP barrier ----
 * comm_create binds one multicast granule on every rank when every device
 * reports CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED and no two ranks share a
 * device (GINSIM_NVLS=0 disables it).  *enabled = 1 when it is active. */
int ginsim_cuda_nvls_enabled(ginsim_cuda_comm_t comm, int* enabled);
/* `iters` back-to-back barriers, one thread per rank, each timed with
 * %globaltimer into ns_out (device, iters u64, rank 0 of the launch):
 * mode 0 = the reference's dissemination BarrierSession on reserved signal
 * cells (runtime.cpp:651-666), mode 1 = NVLS (one multimem.red arrival).
 * The device gin::BarrierSession picks the NVLS form by itself for the world
 * team whenever the comm bound the multicast object. */
int ginsim_cuda_barrier_bench(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t mode, uint32_t iters,
                              uint64_t* ns_out, void* stream);

/* ---- verification utility ----
 * Per-record digests of `count` consecutive records of `record_bytes` at the
 * device pointer `records` into out[count] (device memory):
 *   digest(rec) = sum_i mix64(w_i + i * 0xD1B54A32D192ED03) mod 2^64
 * over the record's little-endian u64 words (tail zero-padded), mix64 =
 * harness_moe.cpp:17-22.  The large-shape analogue of the reference's
 * in-program message verification (harness_moe.cpp:184-200, :227-242): the
 * CPU checker computes the digests it expects and compares arrays, so a
 * 3.76 GB window is verified without copying it to the host. */
int ginsim_cuda_digest(const void* records, uint64_t record_bytes, uint64_t count, uint64_t* out, void* stream);

/* Multicast signal broadcast: adds `amount` to broadcast
 * cell `id` (0..255, a namespace separate from the signal table) on EVERY
 * rank of the comm with one multimem.red through the NVLS mapping, issued on
 * `stream` (device: gin::signal_broadcast).  read_broadcast reads this rank's
 * copy.  USAGE when the comm has no multicast object. */
int ginsim_cuda_signal_broadcast(ginsim_cuda_comm_t comm, uint32_t id, uint64_t amount, void* stream);
int ginsim_cuda_read_broadcast(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value);

/* ---- DeepEP-style MoE dispatch / combine (harness_moe.cpp:105-250) ---- */
typedef struct ginsim_cuda_moe_config {
  uint32_t experts;  /* E, divisible by world */
  uint32_t top_k;    /* K */
  uint32_t tokens;   /* T per rank */
  uint32_t hidden;   /* elements per token (2-byte elements) */
  uint32_t mode;     /* 0 = u16 exact (reference arithmetic), 1 = bf16,
                        2 = fp8 dispatch: e4m3 codes + per-128 fp32 scales (hidden % 512 == 0,
                            direct TMA path), bf16 combine */
  uint32_t layout;   /* 0 = reference layout ((e_loc*n+src)*T+slot)*dmsg,
                        1 = compact per-source layout (src*T*K + prefix + slot)*dmsg,
                        2 = layout 1 with a per-rank dedup transport (one NVLink row per
                            (token, destination rank), fanned out at the destination) */
  uint32_t ctas;     /* CTAs per rank (0 = as many as fit) */
  uint32_t engine;   /* data mover: 0 = auto (TMA bulk copies when messages are
                        16-byte aligned), 1 = 128-bit LSU stores, 2 = TMA */
} ginsim_cuda_moe_config;

typedef struct ginsim_cuda_moe_s* ginsim_cuda_moe_t;

/* Registers (collectively) the dispatch-receive, count and combine-receive
 * windows of the config on `comm` (moe_ll_rank_program's window set,
 * harness_moe.cpp:122-130, minus the CPU staging windows the device path
 * does not need).  Window ids are returned for inspection. */
int ginsim_cuda_moe_create(ginsim_cuda_comm_t comm, const ginsim_cuda_moe_config* cfg, ginsim_cuda_moe_t* out);
/* moe_create for every rank of an in-process group from one caller thread. */
int ginsim_cuda_moe_create_all(const ginsim_cuda_comm_t* comms, uint32_t n, const ginsim_cuda_moe_config* cfg,
                               ginsim_cuda_moe_t* out);
/* Waits for the rank's device work (and, on the Proxy backend, for the agent
 * to drain every submitted descriptor), deregisters and frees the handle's
 * windows and scratch, and returns its signal-cell range for reuse by a later
 * moe_create (which zeroes the range between two barriers). */
int ginsim_cuda_moe_destroy(ginsim_cuda_moe_t moe);
/* The handle's signal cells: [first, first + span) = local expert cells
 * (e_local), the combine flag, the rows cell and the dedup chunk cells. */
int ginsim_cuda_moe_cells(ginsim_cuda_moe_t moe, uint32_t* first, uint32_t* span);
int ginsim_cuda_moe_windows(ginsim_cuda_moe_t moe, uint32_t* dispatch_win, uint32_t* count_win,
                            uint32_t* combine_win);

/* Synthetic workload of the reference (harness_moe.cpp:25-42), generated on
 * the device for rank `src`: x [T][hidden] (token_element in mode 0, the bf16
 * generator in mode 1), topk_idx [T][K] int32 (route_token, bit-exact), and
 * weights [T][K] (combine_weight: u16 in mode 0, float w/8 in mode 1). */
int ginsim_cuda_moe_generate(ginsim_cuda_moe_t moe, uint64_t seed, uint32_t src, void* x,
                             int32_t* topk_idx, void* weights, void* stream);

/* Dispatch: route every (t,k) row of x to its expert's owner with NVLink
 * puts into the owner's dispatch window at the reference slot order
 * (slot = per-expert count in (t,k) order, harness_moe.cpp:143-150), write
 * per-(expert,source) counts, release each expert with
 * SignalAdd((1<<32)+count) (:163-167), and return once every local expert
 * has been released by every source. */
int ginsim_cuda_moe_dispatch(const ginsim_cuda_moe_t* moes, uint32_t n, const void* const* x,
                             const int32_t* const* topk_idx, void* stream);

/* Combine: expert transform (u16: 3x+17e+1; bf16: x*s_e+c_e) fused with the
 * put back to the source's combine window at (token*K+k)*cmsg, per-(src,ctx)
 * SignalAdd(count) on the combine flag (:169-223), then the weighted top-k
 * reduction out[t] = sum_k w_k*y_k (u16 wraparound, or fp32 accumulate ->
 * bf16) once the flag reaches T*K (:227-242). */
int ginsim_cuda_moe_combine(const ginsim_cuda_moe_t* moes, uint32_t n, const void* const* weights,
                            void* const* out, void* stream);

/* Phase timeline of the last dispatch (kernel 0), combine send (1) and
 * combine reduce (2) launches: per CTA, 8 %globaltimer stamps (ns; unused = 0)
 * into out[1024*8]; *ctas = that kernel's grid.  Needs GINSIM_PROFILE_PHASES=1
 * when the moe handle was created.  Dispatch stamps: start, route tables done,
 * puts issued+drained, releases issued, experts acquired. */
int ginsim_cuda_moe_phase_times(ginsim_cuda_moe_t moe, uint32_t kernel, uint64_t* out, uint32_t* ctas);

/* Per-launch kernel count of the last dispatch/combine (for bench evidence). */
int ginsim_cuda_moe_last_launch(ginsim_cuda_moe_t moe, uint32_t* ctas, uint32_t* threads);

/* Transport the handle runs: 0 = direct NVLink stores, 1 = Proxy backend
 * with one-shot staging (LSU kernels; per-message puts when
 * GINSIM_PROXY_COALESCE=0), 2 = Proxy pipeline (chunked copy-engine puts
 * issued while the staging kernel runs; layout 1, modes 0/1). */
int ginsim_cuda_moe_transport(ginsim_cuda_moe_t moe, uint32_t* kind);

#ifdef __cplusplus
}
#endif
#endif /* GINSIM_CUDA_H */
