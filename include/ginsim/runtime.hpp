// ginsim/runtime.hpp — C++ host API of the B200 GIN hot path.
//
// Keeps the reference's host surface (proj/core/include/ginsim/types.hpp,
// runtime.hpp) so a ginsim program recompiles against GPU windows: Config /
// config_from_env, InProcGroup + comm_init, DevComm (window_register, cells,
// flush, snapshot_cells), Gin (put / put_value / signal / flush / waits),
// BarrierSession, Team, Window, CompletionAction, pool_select.  Everything is
// a thin header-only layer over the C ABI (include/ginsim_cuda.h); window
// bytes are DEVICE memory (ginsim::mem_alloc), ops execute on the GPU.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <functional>
#include <thread>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "../ginsim_cuda.h"
#include "errors.hpp"

namespace ginsim {

// ---------------------------------------------------------------- types.hpp:14-123
using RankId = uint32_t;
using TeamId = uint16_t;
using WindowId = uint32_t;
using SignalId = uint32_t;
using CounterId = uint32_t;
using ContextId = uint16_t;

inline constexpr WindowId kInlineWindow = 0xFFFFFFFFu;
inline constexpr uint64_t kMaxInlineBytes = 8;

enum class SignalKind : uint8_t { Inc = 0, Add = 1 };

struct SignalOp {
  SignalKind kind = SignalKind::Inc;
  uint64_t operand = 1;
  static SignalOp inc() { return {SignalKind::Inc, 1}; }
  static SignalOp add(uint64_t v) { return {SignalKind::Add, v}; }
  uint64_t amount() const { return kind == SignalKind::Inc ? 1 : operand; }
  friend bool operator==(const SignalOp&, const SignalOp&) = default;
};

struct CompletionAction {
  struct RemoteSignal {
    SignalId id = 0;
    SignalOp op = SignalOp::inc();
    friend bool operator==(const RemoteSignal&, const RemoteSignal&) = default;
  };
  std::optional<RemoteSignal> remote_signal;
  std::optional<CounterId> local_counter;

  static CompletionAction none() { return {}; }
  static CompletionAction signal(SignalId id, SignalOp op = SignalOp::inc()) {
    CompletionAction a;
    a.remote_signal = RemoteSignal{id, op};
    return a;
  }
  static CompletionAction counter(CounterId id) {
    CompletionAction a;
    a.local_counter = id;
    return a;
  }
  CompletionAction with_counter(CounterId id) const {
    CompletionAction a = *this;
    a.local_counter = id;
    return a;
  }
  friend bool operator==(const CompletionAction&, const CompletionAction&) = default;

  ginsim_cuda_action to_c() const {
    ginsim_cuda_action a{};
    a.signal_id = remote_signal ? (int32_t)remote_signal->id : -1;
    a.signal_add = remote_signal && remote_signal->op.kind == SignalKind::Add;
    a.operand = remote_signal ? remote_signal->op.operand : 1;
    a.counter_id = local_counter ? (int32_t)*local_counter : -1;
    return a;
  }
};

struct Team {
  TeamId id = 0;
  std::vector<RankId> members;
  static Team world(uint32_t world_size) {
    Team t;
    t.members.resize(world_size);
    for (uint32_t i = 0; i < world_size; ++i) t.members[i] = i;
    return t;
  }
  uint32_t size() const { return static_cast<uint32_t>(members.size()); }
};

inline RankId team_translate(const Team& team, uint32_t team_rank) {
  if (team_rank >= team.members.size()) {
    throw RankOutOfRange("team rank " + std::to_string(team_rank) + " out of range for team of " +
                         std::to_string(team.members.size()));
  }
  return team.members[team_rank];
}

class DevComm;

// A collectively registered DEVICE memory region (types.hpp:89-118).
class Window {
 public:
  Window() = default;
  Window(ginsim_cuda_comm_t c, WindowId id, RankId self, std::vector<uint64_t> sizes, std::span<std::byte> local)
      : comm_(c), id_(id), self_(self), sizes_(std::move(sizes)), local_(local) {}
  // types.hpp:92-93: a window description without a communicator (ranges,
  // sizes and the local slice only; peer_bytes needs a registered window)
  Window(WindowId id, RankId self, std::vector<uint64_t> sizes, std::span<std::byte> local)
      : id_(id), self_(self), sizes_(std::move(sizes)), local_(local) {
    if (self_ >= sizes_.size() || local_.size() != sizes_[self_])
      throw UnknownWindow("window " + std::to_string(id) + ": local region size mismatch");
  }
  // types.hpp:95-97: a registration still collecting the peers' sizes
  static Window pending(WindowId id, RankId self, std::span<std::byte> local) {
    Window w;
    w.id_ = id;
    w.self_ = self;
    w.local_ = local;
    return w;
  }
  WindowId id() const { return id_; }
  RankId self_rank() const { return self_; }
  bool complete() const { return !sizes_.empty(); }
  uint32_t rank_count() const { return static_cast<uint32_t>(sizes_.size()); }
  uint64_t size_of(RankId rank) const {
    if (!complete()) throw UnknownWindow("window " + std::to_string(id_) + " not fully registered yet");
    if (rank >= sizes_.size()) throw RankOutOfRange("rank " + std::to_string(rank) + " not registered in window");
    return sizes_[rank];
  }
  void check_range(RankId rank, uint64_t offset, uint64_t len) const {
    const uint64_t cap = size_of(rank);
    if (offset > cap || len > cap - offset) {
      throw OutOfBounds("window " + std::to_string(id_) + " rank " + std::to_string(rank) + ": [" +
                        std::to_string(offset) + ", +" + std::to_string(len) + ") exceeds capacity " +
                        std::to_string(cap));
    }
  }
  // Validated view of the local slice (device bytes).
  std::span<std::byte> local_bytes(uint64_t offset, uint64_t len) const {
    check_range(self_, offset, len);
    return local_.subspan(static_cast<size_t>(offset), static_cast<size_t>(len));
  }
  // Device address of `rank`'s region as mapped in this process (NVLink peer mapping).
  std::byte* peer_bytes(RankId rank) const {
    void* p = nullptr;
    check(ginsim_cuda_window_ptr(comm_, id_, rank, &p));
    return static_cast<std::byte*>(p);
  }

 private:
  ginsim_cuda_comm_t comm_ = nullptr;
  WindowId id_ = 0;
  RankId self_ = 0;
  std::vector<uint64_t> sizes_;
  std::span<std::byte> local_;
};

// types.hpp:119-123: the bytes of [offset, offset + len) in rank's region --
// validated for every rank, backing bytes only for the registering rank (the
// other ranks' regions are not local; the span is empty for those).
inline std::span<std::byte> window_resolve(Window& w, RankId rank, uint64_t offset, uint64_t len) {
  w.check_range(rank, offset, len);
  if (rank == w.self_rank()) return w.local_bytes(offset, len);
  return {};
}

// ---------------------------------------------------------------- runtime.hpp:26-58
enum class BackendKind { Direct, Proxy };
inline const char* to_string(BackendKind k) { return k == BackendKind::Direct ? "direct" : "proxy"; }
// runtime.hpp:26-29.  On B200 the "transport" is NVLink peer memory (or one
// GPU's HBM for emulated ranks) whatever the bootstrap; progress is always
// asynchronous (the device moves the bytes, the proxy agent is a thread):
// the fields are kept so reference code compiles, and are informational.
enum class TransportKind { Inproc, Socket, Nvlink };
enum class ProgressMode { Threaded, Manual };
inline const char* to_string(TransportKind k) {
  return k == TransportKind::Inproc ? "inproc" : (k == TransportKind::Socket ? "socket" : "nvlink");
}
enum class Opcode : uint8_t { Put = 1, PutInline = 2, SignalOnly = 3 };

// fabric.hpp:26-35.  The reference's simulated-fabric latency model.  On B200
// the fabric is real (NVLink, or one GPU's HBM for emulated ranks): the model
// is accepted so reference programs compile, and its seed is the CSV's seed
// column (write_csv); the delays are not applied.
struct LatencyModel {
  uint64_t base_delay_ns = 0;
  uint64_t jitter_ns = 0;
  uint32_t reorder_window = 0;
  uint64_t seed = 0;
  double line_rate_gbps = 0.0;
  friend bool operator==(const LatencyModel&, const LatencyModel&) = default;
};

struct Config {
  uint32_t n_contexts = 4;
  std::optional<BackendKind> backend;  // unset = direct
  uint32_t signal_cells = 256;
  uint32_t counter_cells = 256;
  uint32_t queue_depth = 1024;
  uint64_t timeout_ms = 30'000;
  // runtime.hpp:36-37 defaults; informational on B200 (see LatencyModel)
  LatencyModel latency{.base_delay_ns = 500, .jitter_ns = 0, .reorder_window = 0, .seed = 0x5EED,
                       .line_rate_gbps = 16.0};
  ProgressMode progress = ProgressMode::Threaded;  // informational on B200 (always asynchronous)
  int device = -1;  // B200: GPU of this rank (-1 = rank % device count)
  // unset = the fabric (NVLink peer mappings); Socket = the Proxy backend's
  // GIN1-over-TCP transport between the ranks' host agents (comm_init_socket)
  std::optional<TransportKind> transport;
  friend bool operator==(const Config&, const Config&) = default;

  ginsim_cuda_config to_c() const {
    ginsim_cuda_config c{};
    c.n_contexts = n_contexts;
    c.backend = backend.value_or(BackendKind::Direct) == BackendKind::Proxy ? 1u : 0u;
    c.signal_cells = signal_cells;
    c.counter_cells = counter_cells;
    c.queue_depth = queue_depth;
    c.timeout_ms = timeout_ms;
    c.transport = transport == TransportKind::Socket ? 1u : 0u;
    return c;
  }
};

inline Config config_from_env(Config base = {}) {
  ginsim_cuda_config c = base.to_c();
  check(ginsim_cuda_config_from_env(&c));
  base.backend = c.backend ? BackendKind::Proxy : BackendKind::Direct;
  base.queue_depth = c.queue_depth;
  base.timeout_ms = c.timeout_ms;
  if (!std::getenv("GINSIM_BACKEND")) base.backend.reset();
  if (std::getenv("GINSIM_TRANSPORT")) base.transport = c.transport ? TransportKind::Socket : TransportKind::Nvlink;
  // the latency-model variables (runtime.cpp:53-56), parsed as the reference
  // does (strtoull base 0, the whole string, UsageError otherwise)
  auto env_u64 = [](const char* name) -> std::optional<uint64_t> {
    const char* v = std::getenv(name);
    if (!v || !*v) return std::nullopt;
    char* end = nullptr;
    const uint64_t x = std::strtoull(v, &end, 0);
    if (end == v || *end != '\0') throw UsageError(std::string(name) + ": cannot parse '" + v + "' as an integer");
    return x;
  };
  if (auto v = env_u64("GINSIM_SEED")) base.latency.seed = *v;
  if (auto v = env_u64("GINSIM_LATENCY_NS")) base.latency.base_delay_ns = *v;
  if (auto v = env_u64("GINSIM_JITTER_NS")) base.latency.jitter_ns = *v;
  if (auto v = env_u64("GINSIM_REORDER")) base.latency.reorder_window = static_cast<uint32_t>(*v);
  return base;
}

struct PoolSelection {
  uint32_t comm_index;
  uint32_t context_index;
  friend bool operator==(const PoolSelection&, const PoolSelection&) = default;
};
constexpr PoolSelection pool_select(uint32_t id, uint32_t n_contexts = 4) { return {id / n_contexts, id % n_contexts}; }

inline constexpr uint32_t kBarrierSlots = 8;
inline constexpr uint32_t kBarrierSteps = 8;

// In-process rendezvous (runtime.hpp:68-121): ranks are host threads.
class InProcGroup {
 public:
  static std::shared_ptr<InProcGroup> create(uint32_t world_size) {
    ginsim_cuda_group_t g = nullptr;
    check(ginsim_cuda_inproc_group_create(world_size, &g));
    return std::shared_ptr<InProcGroup>(new InProcGroup(g, world_size));
  }
  ~InProcGroup() { ginsim_cuda_inproc_group_destroy(g_); }
  uint32_t world_size() const { return world_; }
  ginsim_cuda_group_t handle() const { return g_; }
  // runtime.hpp:81-83 (Manual-mode progress).  The device moves the bytes and
  // the proxy agents run on their own threads, so there is never work for the
  // host to pump: 0, as the reference returns once a group is quiescent.
  size_t pump_all() { return 0; }

 private:
  InProcGroup(ginsim_cuda_group_t g, uint32_t w) : g_(g), world_(w) {}
  ginsim_cuda_group_t g_;
  uint32_t world_;
};

// One rank's communicator (runtime.hpp:123-246).
class DevComm {
 public:
  // `keep` owns the bootstrap the comm registers windows over (an
  // InProcGroup, or comm_init_socket's rendezvous)
  DevComm(ginsim_cuda_comm_t c, std::shared_ptr<void> keep, Config cfg) : c_(c), group_(std::move(keep)), cfg_(cfg) {
    uint32_t b = 0;
    check(ginsim_cuda_comm_info(c_, &rank_, &world_, &device_, &b));
    backend_ = b ? BackendKind::Proxy : BackendKind::Direct;
    world_team_ = Team::world(world_);
  }
  ~DevComm() { ginsim_cuda_comm_destroy(c_); }
  DevComm(const DevComm&) = delete;
  DevComm& operator=(const DevComm&) = delete;

  RankId rank() const { return rank_; }
  uint32_t world_size() const { return world_; }
  int device() const { return device_; }
  const Config& config() const { return cfg_; }
  BackendKind backend() const { return backend_; }
  const Team& world_team() const { return world_team_; }
  TransportKind transport_kind() const { return cfg_.transport.value_or(TransportKind::Nvlink); }
  ProgressMode progress_mode() const { return cfg_.progress; }
  ginsim_cuda_comm_t handle() const { return c_; }

  // Collective (runtime.cpp:347-371): `local` are device bytes this rank owns.
  Window& window_register(std::span<std::byte> local) {
    WindowId id = 0;
    check(ginsim_cuda_window_register(c_, local.data(), local.size(), &id));
    std::vector<uint64_t> sizes(world_);
    for (RankId r = 0; r < world_; ++r) check(ginsim_cuda_window_size(c_, id, r, &sizes[r]));
    windows_.push_back(std::make_unique<Window>(c_, id, rank_, std::move(sizes), local));
    return *windows_.back();
  }
  Window& lookup_window(WindowId id) {
    for (auto& w : windows_)
      if (w->id() == id) return *w;
    throw UnknownWindow("window " + std::to_string(id) + " was never registered");
  }
  // B200 addition (no reference counterpart): release a window on this rank;
  // the id is reused by the next window_register (ginsim_cuda.h).
  void window_deregister(WindowId id) {
    check(ginsim_cuda_window_deregister(c_, id));
    windows_.erase(std::remove_if(windows_.begin(), windows_.end(), [&](const auto& w) { return w->id() == id; }),
                   windows_.end());
  }

  // Sub-teams (runtime.hpp:145-148, runtime.cpp:329-343).  World is id 0.
  const Team& register_team(Team team) {
    check(ginsim_cuda_register_team(c_, team.id, team.members.data(), static_cast<uint32_t>(team.members.size())));
    teams_.push_back(std::make_unique<Team>(std::move(team)));
    return *teams_.back();
  }
  const Team& team(TeamId id) const {
    if (id == 0) return world_team_;
    for (auto& t : teams_)
      if (t->id == id) return *t;
    throw UsageError("team " + std::to_string(id) + " not registered");
  }

  uint64_t read_signal(SignalId id) const {
    uint64_t v = 0;
    check(ginsim_cuda_read_signal(c_, id, &v));
    return v;
  }
  void wait_signal(SignalId id, uint64_t expected) { check(ginsim_cuda_wait_signal(c_, id, expected)); }
  void reset_signal(SignalId id) { check(ginsim_cuda_reset_signal(c_, id)); }
  uint64_t read_counter(CounterId id) const {
    uint64_t v = 0;
    check(ginsim_cuda_read_counter(c_, id, &v));
    return v;
  }
  void wait_counter(CounterId id, uint64_t expected) { check(ginsim_cuda_wait_counter(c_, id, expected)); }
  void reset_counter(CounterId id) { check(ginsim_cuda_reset_counter(c_, id)); }
  void flush(ContextId ctx) { check(ginsim_cuda_flush(c_, ctx, nullptr)); }

  // runtime.hpp:164-171.  Delivery needs no host pumping on B200 (the device
  // moves the bytes; the proxy agent runs on its own thread), so a local
  // progress pass only surfaces device-side failures; it returns 0.
  size_t pump_local() {
    check_failed();
    return 0;
  }
  // The simulator's clock; here the host's monotonic clock in ns.
  uint64_t virtual_now() const {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
  }
  // runtime.hpp:188-191: poll pred until it holds; Timeout after config().timeout_ms.
  void wait_until(const std::function<bool()>& pred, const char* what) {
    const auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(cfg_.timeout_ms);
    uint32_t idle = 0;
    while (!pred()) {
      check_failed();
      if (std::chrono::steady_clock::now() > deadline)
        throw Timeout(std::string(what) + ": exceeded " + std::to_string(cfg_.timeout_ms) + " ms");
      if (++idle < 128) std::this_thread::yield();
      else std::this_thread::sleep_for(std::chrono::microseconds(50));
    }
  }

  // runtime.hpp:180-183 / runtime.cpp:474-544: validate one op and route it to
  // the backend (team-relative peer; 1-8 byte inline values little-endian).
  void submit_op(ContextId ctx, const Team& team, uint32_t peer_team_rank, Opcode opcode, WindowId dst_window,
                 uint64_t dst_offset, WindowId src_window, uint64_t src_offset_or_value, uint64_t bytes,
                 const CompletionAction& action) {
    const RankId peer = team_translate(team, peer_team_rank);
    const ginsim_cuda_action a = action.to_c();
    switch (opcode) {
      case Opcode::Put:
        check(ginsim_cuda_put(c_, ctx, peer, dst_window, dst_offset, src_window, src_offset_or_value, bytes, &a,
                              nullptr));
        break;
      case Opcode::PutInline:
        check(ginsim_cuda_put_value(c_, ctx, peer, dst_window, dst_offset, src_offset_or_value, (uint32_t)bytes, &a,
                                    nullptr));
        break;
      case Opcode::SignalOnly: {
        if (!action.remote_signal) throw InvalidDescriptor("SIGNAL_ONLY op without a signal");
        ginsim_cuda_action extra = a;
        extra.signal_id = -1;
        check(ginsim_cuda_signal(c_, ctx, peer, action.remote_signal->id,
                                 action.remote_signal->op.kind == SignalKind::Add, action.remote_signal->op.operand,
                                 &extra, nullptr));
        break;
      }
    }
  }
  void check_failed() const {
    uint32_t code = 0;
    check(ginsim_cuda_device_error(c_, &code, 1));
    if (code) throw_status((int)code, "device-side error on rank " + std::to_string(rank_));
  }

  struct CellSnapshot {
    std::vector<uint64_t> signals;
    std::vector<uint64_t> counters;
    friend bool operator==(const CellSnapshot&, const CellSnapshot&) = default;
  };
  CellSnapshot snapshot_cells() const {
    CellSnapshot s;
    s.signals.resize(cfg_.signal_cells);
    s.counters.resize(cfg_.counter_cells);
    check(ginsim_cuda_snapshot_cells(c_, s.signals.data(), s.counters.data()));
    return s;
  }

 private:
  ginsim_cuda_comm_t c_;
  std::shared_ptr<void> group_;
  Config cfg_;
  RankId rank_ = 0;
  uint32_t world_ = 1;
  int device_ = 0;
  BackendKind backend_ = BackendKind::Direct;
  Team world_team_;
  std::vector<std::unique_ptr<Team>> teams_;
  std::vector<std::unique_ptr<Window>> windows_;
};

// comm_init (runtime.hpp:251-252): collective over the group's threads.
inline std::unique_ptr<DevComm> comm_init(std::shared_ptr<InProcGroup> group, RankId self, const Config& config) {
  if (!group) throw UsageError("comm_init requires a group");
  int ndev = 1;
  int device = config.device;
  if (device < 0) {
    ginsim_cuda_comm_t probe = nullptr;
    (void)probe;
    device = static_cast<int>(self);  // one GPU per rank; callers emulating ranks set Config::device
  }
  ginsim_cuda_bootstrap boot{};
  check(ginsim_cuda_inproc_bootstrap(group->handle(), self, &boot));
  const ginsim_cuda_config c = config.to_c();
  ginsim_cuda_comm_t h = nullptr;
  check(ginsim_cuda_comm_create(self, group->world_size(), device, &c, &boot, &h));
  (void)ndev;
  return std::make_unique<DevComm>(h, std::move(group), config);
}

// comm_init_socket (socket_transport.hpp:117-126): rank 0 hosts the
// rendezvous at host:port; every rank's Proxy agent then reaches the others
// with GIN1 frames over TCP (net.cu) -- the path toward peers outside the
// NVLink domain.  Requires the Proxy backend (unset = Proxy).
inline std::unique_ptr<DevComm> comm_init_socket(const std::string& host, uint16_t port, uint32_t world_size,
                                                 RankId self, const Config& config) {
  if (config.backend && *config.backend != BackendKind::Proxy)
    throw BackendMismatch("the socket transport runs on the Proxy backend");
  // socket_transport.cpp: the receiver threads are the transport's progress
  if (config.progress == ProgressMode::Manual)
    throw UsageError("the socket transport needs threaded progress (ProgressMode::Manual is in-process only)");
  Config cfg = config;
  cfg.backend = BackendKind::Proxy;
  cfg.transport = TransportKind::Socket;
  std::shared_ptr<ginsim_cuda_bootstrap> boot(new ginsim_cuda_bootstrap{}, [](ginsim_cuda_bootstrap* b) {
    ginsim_cuda_socket_bootstrap_destroy(b);
    delete b;
  });
  check(ginsim_cuda_socket_bootstrap_create(host.c_str(), port, world_size, self, cfg.timeout_ms, boot.get()));
  const ginsim_cuda_config c = cfg.to_c();
  ginsim_cuda_comm_t h = nullptr;
  check(ginsim_cuda_comm_create(self, world_size, cfg.device >= 0 ? cfg.device : static_cast<int>(self), &c, boot.get(),
                                &h));
  return std::make_unique<DevComm>(h, std::move(boot), cfg);
}

// reserve_loopback_port (socket_transport.hpp:128-129).
inline uint16_t reserve_loopback_port() {
  uint16_t p = 0;
  check(ginsim_cuda_reserve_loopback_port(&p));
  return p;
}

// Device memory for windows: cuMemCreate-backed, exportable to peers.
inline std::span<std::byte> mem_alloc(DevComm& comm, uint64_t bytes) {
  void* p = nullptr;
  check(ginsim_cuda_mem_alloc(comm.handle(), bytes, &p));
  return {static_cast<std::byte*>(p), static_cast<size_t>(bytes)};
}

// Per-context handle (runtime.hpp:260-306); host-issued ops run on the GPU.
class Gin {
 public:
  Gin(DevComm& comm, ContextId context_index) : comm_(comm), ctx_(context_index) {
    if (context_index >= comm.config().n_contexts) {
      throw InvalidContext("context " + std::to_string(context_index) + " out of range (" +
                           std::to_string(comm.config().n_contexts) + " configured)");
    }
  }
  DevComm& comm() { return comm_; }
  ContextId context() const { return ctx_; }

  void put(const Team& team, uint32_t peer, const Window& dst_window, uint64_t dst_offset, const Window& src_window,
           uint64_t src_offset, uint64_t bytes, const CompletionAction& action = {}) {
    const ginsim_cuda_action a = action.to_c();
    check(ginsim_cuda_put(comm_.handle(), ctx_, world_peer(team, peer), dst_window.id(), dst_offset, src_window.id(),
                          src_offset, bytes, &a, nullptr));
  }
  template <typename T>
  void put_value(const Team& team, uint32_t peer, const Window& dst_window, uint64_t dst_offset, T value,
                 const CompletionAction& action = {}) {
    static_assert(std::is_trivially_copyable_v<T> && sizeof(T) <= 8,
                  "inline values are at most 8 trivially copyable bytes");
    unsigned char raw[8] = {};
    std::memcpy(raw, &value, sizeof(T));
    uint64_t packed = 0;
    for (size_t i = 0; i < sizeof(T); ++i) packed |= static_cast<uint64_t>(raw[i]) << (8 * i);
    put_value_raw(team, peer, dst_window, dst_offset, packed, sizeof(T), action);
  }
  void put_value_raw(const Team& team, uint32_t peer, const Window& dst_window, uint64_t dst_offset, uint64_t le_value,
                     uint32_t width, const CompletionAction& action = {}) {
    const ginsim_cuda_action a = action.to_c();
    check(ginsim_cuda_put_value(comm_.handle(), ctx_, world_peer(team, peer), dst_window.id(), dst_offset, le_value,
                                width, &a, nullptr));
  }
  void signal(const Team& team, uint32_t peer, SignalId id, SignalOp op = SignalOp::inc(),
              const CompletionAction& action = {}) {
    const ginsim_cuda_action a = action.to_c();
    check(ginsim_cuda_signal(comm_.handle(), ctx_, world_peer(team, peer), id, op.kind == SignalKind::Add,
                             op.operand, &a, nullptr));
  }
  void flush() { comm_.flush(ctx_); }
  uint64_t read_signal(SignalId id) const { return comm_.read_signal(id); }
  void wait_signal(SignalId id, uint64_t expected) { comm_.wait_signal(id, expected); }
  void reset_signal(SignalId id) { comm_.reset_signal(id); }
  uint64_t read_counter(CounterId id) const { return comm_.read_counter(id); }
  void wait_counter(CounterId id, uint64_t expected) { comm_.wait_counter(id, expected); }
  void reset_counter(CounterId id) { comm_.reset_counter(id); }

 private:
  uint32_t world_peer(const Team& team, uint32_t peer) const {
    if (peer >= team.size()) {
      throw InvalidPeer("peer " + std::to_string(peer) + " outside team of " + std::to_string(team.size()));
    }
    return team.members[peer];
  }
  DevComm& comm_;
  ContextId ctx_;
};

// Dissemination barrier over reserved cells (runtime.hpp:312-327, runtime.cpp:651-666).
class BarrierSession {
 public:
  BarrierSession(Gin& gin, Team team, uint32_t slot) : gin_(gin), team_(std::move(team)), slot_(slot) {
    if (slot >= kBarrierSlots) throw UsageError("barrier slot " + std::to_string(slot) + " out of range");
    const RankId self = gin_.comm().rank();
    auto it = std::find(team_.members.begin(), team_.members.end(), self);
    if (it == team_.members.end()) {
      throw InvalidPeer("rank " + std::to_string(self) + " is not a member of the barrier team");
    }
    my_index_ = static_cast<uint32_t>(it - team_.members.begin());
  }
  void sync() {
    round_++;
    const uint32_t n = team_.size();
    if (n <= 1) return;
    uint32_t steps = 0;
    while ((1u << steps) < n) steps++;
    if (steps > kBarrierSteps) throw UsageError("team too large for the barrier signal region");
    const uint32_t base = gin_.comm().config().signal_cells - kBarrierSlots * kBarrierSteps + slot_ * kBarrierSteps;
    for (uint32_t k = 0; k < steps; ++k) {
      gin_.signal(team_, (my_index_ + (1u << k)) % n, base + k, SignalOp::inc());
      gin_.wait_signal(base + k, round_);
    }
  }
  uint64_t round() const { return round_; }

 private:
  Gin& gin_;
  Team team_;
  uint32_t slot_;
  uint32_t my_index_ = 0;
  uint64_t round_ = 0;
};

}  // namespace ginsim
