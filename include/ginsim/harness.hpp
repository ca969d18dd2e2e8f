// ginsim/harness.hpp -- the reference's harness over the B200 library
// (proj/core/include/ginsim/harness.hpp): LaunchOptions, launch, launch_pool
// (:13-30); RankState (:36-43); the ring exchange (:45-62,
// harness_ring.cpp:18-57); ping-pong / bandwidth programs, summarize and
// write_csv (:64-102, harness_bench.cpp:12-178).  The programs run the
// reference's host protocols unchanged over host windows (std::vector<std::byte>
// registered as in the reference: the library pins and maps the pages, the
// device moves the bytes).  They time with the host's monotonic clock (there
// is no virtual clock on hardware), so a row includes the host-issued op's
// launch; the device-resident loops are ginsim_cuda_pingpong / ginsim_cuda_bw
// (include/ginsim_cuda.h).  The MoE demos (run_moe_ll / run_moe_ht) are the
// device kernels behind ginsim_cuda_moe_* and ginsim_cuda_moe_ht_ring.
// One host thread per rank; each builds its communicator(s) with comm_init
// over an InProcGroup (TransportKind::Inproc) or comm_init_socket
// (TransportKind::Socket, the Proxy backend's GIN1 transport), runs the
// program, waits until every rank's program has returned, then tears its
// communicators down (a rank must not unmap its windows while a peer may
// still write them), and the first rank failure is rethrown after the join.
// Device: Config::device < 0 puts rank r on GPU r % device count.
#pragma once

#include <cuda_runtime.h>
#include <spawn.h>
#include <sys/wait.h>
#include <unistd.h>  // environ

#include <algorithm>
#include <chrono>
#include <cerrno>
#include <condition_variable>
#include <cstddef>
#include <cstring>
#include <exception>
#include <fstream>
#include <functional>
#include <initializer_list>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "ginsim/runtime.hpp"

namespace ginsim {

struct LaunchOptions {
  uint32_t ranks = 2;
  TransportKind transport = TransportKind::Inproc;  // Inproc or Socket (Nvlink is the Inproc fabric here)
  Config config;
  std::string host = "127.0.0.1";
  uint16_t port = 0;  // socket rendezvous; 0 picks a free loopback port (comm c of a pool: port + c)
};

namespace detail {
class Latch {
 public:
  explicit Latch(uint32_t n) : left_(n) {}
  void arrive_and_wait() {
    std::unique_lock<std::mutex> lk(mu_);
    if (--left_ == 0) {
      cv_.notify_all();
      return;
    }
    cv_.wait(lk, [&] { return left_ == 0; });
  }

 private:
  std::mutex mu_;
  std::condition_variable cv_;
  uint32_t left_;
};
}  // namespace detail

// Each rank gets `n_comms` communicators (channel counts beyond one comm's
// contexts, pool_select); socket mode uses ports port .. port + n_comms - 1.
inline void launch_pool(const LaunchOptions& opts, uint32_t n_comms,
                        const std::function<void(std::vector<DevComm*>&)>& program) {
  if (opts.ranks == 0 || opts.ranks > 8) throw UsageError("launch: ranks must be 1..8 (one NVSwitch domain)");
  if (n_comms == 0) throw UsageError("launch_pool: at least one communicator per rank");
  if (opts.transport == TransportKind::Socket && opts.config.backend && *opts.config.backend != BackendKind::Proxy)
    throw BackendMismatch("launch: the socket transport runs on the Proxy backend");
  std::vector<std::shared_ptr<InProcGroup>> groups;
  std::vector<uint16_t> ports;
  for (uint32_t c = 0; c < n_comms; ++c) {
    if (opts.transport == TransportKind::Socket)
      ports.push_back(opts.port ? static_cast<uint16_t>(opts.port + c) : reserve_loopback_port());
    else
      groups.push_back(InProcGroup::create(opts.ranks));
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) throw CudaError("launch: no CUDA device visible");
  detail::Latch programs_done(opts.ranks);
  std::mutex mu;
  std::exception_ptr first;
  std::vector<std::thread> threads;
  for (uint32_t r = 0; r < opts.ranks; ++r) {
    threads.emplace_back([&, r] {
      std::vector<std::unique_ptr<DevComm>> comms;
      try {
        Config cfg = opts.config;
        if (cfg.device < 0) cfg.device = static_cast<int>(r % static_cast<uint32_t>(ndev));
        for (uint32_t c = 0; c < n_comms; ++c)
          comms.push_back(opts.transport == TransportKind::Socket
                              ? comm_init_socket(opts.host, ports[c], opts.ranks, r, cfg)
                              : comm_init(groups[c], r, cfg));
        std::vector<DevComm*> raw;
        for (auto& c : comms) raw.push_back(c.get());
        program(raw);
      } catch (...) {
        std::lock_guard<std::mutex> lk(mu);
        if (!first) first = std::current_exception();
      }
      programs_done.arrive_and_wait();
      comms.clear();  // teardown once every rank's program has returned
    });
  }
  for (auto& t : threads) t.join();
  if (first) std::rethrow_exception(first);
}

// launch (harness.hpp:22-24): `program` once per rank.
inline void launch(const LaunchOptions& opts, const std::function<void(DevComm&)>& program) {
  launch_pool(opts, 1, [&](std::vector<DevComm*>& comms) { program(*comms[0]); });
}

// launch_processes (harness.hpp:32-34, harness_launch.cpp:77-119): `ranks`
// copies of `exe` with args + {"--rank", i}, then wait for all of them.
// ChildFailure names the first rank (in rank order) that exited nonzero or
// died on a signal, or a spawn that failed.  posix_spawn instead of fork +
// exec: the caller may already hold a CUDA context, and a forked child of a
// CUDA process must not touch the runtime before exec.
inline void launch_processes(const std::string& exe, const std::vector<std::string>& args, uint32_t ranks) {
  if (ranks == 0) throw UsageError("launch_processes: need at least one rank");
  std::vector<pid_t> pids(ranks, -1);
  std::string failure;
  for (uint32_t r = 0; r < ranks; ++r) {
    std::vector<std::string> argv_s{exe};
    argv_s.insert(argv_s.end(), args.begin(), args.end());
    argv_s.push_back("--rank");
    argv_s.push_back(std::to_string(r));
    std::vector<char*> argv;
    for (auto& a : argv_s) argv.push_back(a.data());
    argv.push_back(nullptr);
    const int rc = ::posix_spawn(&pids[r], exe.c_str(), nullptr, nullptr, argv.data(), environ);
    if (rc != 0) {
      pids[r] = -1;
      if (failure.empty()) failure = "rank " + std::to_string(r) + ": spawn of " + exe + " failed: " + std::strerror(rc);
      break;  // the ranks already running are still reaped below
    }
  }
  for (uint32_t r = 0; r < ranks; ++r) {
    if (pids[r] < 0) continue;
    int st = 0;
    pid_t w;
    do {
      w = ::waitpid(pids[r], &st, 0);
    } while (w < 0 && errno == EINTR);
    std::string why;
    if (w < 0)
      why = "waitpid failed: " + std::string(std::strerror(errno));
    else if (WIFEXITED(st) && WEXITSTATUS(st) != 0)
      why = "exited with status " + std::to_string(WEXITSTATUS(st));
    else if (WIFSIGNALED(st))
      why = "killed by signal " + std::to_string(WTERMSIG(st));
    if (!why.empty() && failure.empty()) failure = "rank " + std::to_string(r) + " " + why;
  }
  if (!failure.empty()) throw ChildFailure(failure);
}

// ------------------------------------------------------------ final state
// Everything a rank's program observes at the end (harness.hpp:36-43): two
// backends are equivalent when these match.
struct RankState {
  std::vector<std::vector<std::byte>> windows;
  DevComm::CellSnapshot cells;
  friend bool operator==(const RankState&, const RankState&) = default;
};
using FinalState = std::vector<RankState>;

// ------------------------------------------------------------ ring exchange
struct RingOptions {
  uint64_t bytes = 4096;
  uint32_t rounds = 10;
};

struct RingReport {
  uint32_t ranks = 0;
  uint32_t rounds = 0;
  FinalState state;
};

namespace detail {
// Unpin a program's host windows before its vectors go away (the caller owns
// window bytes; runtime.cu window_deregister).  Called after the program's
// closing barrier, when no peer can still write them.
inline void release(DevComm& comm, std::initializer_list<WindowId> ids) {
  for (WindowId id : ids) comm.window_deregister(id);
}

// the (sender, round, offset) tag every ring byte carries (harness_ring.cpp:12-14);
// receivers recompute it, nothing expected travels out of band
inline std::byte ring_tag(uint32_t sender, uint32_t round, uint64_t i) {
  return static_cast<std::byte>(sender * 131u + round * 31u + i * 7u + 1u);
}
}  // namespace detail

// One rank of the ring (harness_ring.cpp:18-57): per round, put + SignalInc of
// this rank's slice to the right neighbour, wait for the left neighbour's,
// verify it, reset the cell, flush (the source is reused next round) and
// barrier (no rank signals round + 1 before every rank has reset).
inline void ring_rank_program(DevComm& comm, const RingOptions& ring, RankState* out) {
  const uint32_t n = comm.world_size(), me = comm.rank();
  const uint64_t S = ring.bytes;
  const Team& world = comm.world_team();
  std::vector<std::byte> send(n * S), recv(n * S);
  Window& send_w = comm.window_register(send);
  Window& recv_w = comm.window_register(recv);
  Gin gin(comm, 0);
  BarrierSession barrier(gin, world, 0);
  const uint32_t right = (me + 1) % n, left = (me + n - 1) % n;
  for (uint32_t round = 0; round < ring.rounds; ++round) {
    std::byte* slice = send.data() + right * S;
    for (uint64_t i = 0; i < S; ++i) slice[i] = detail::ring_tag(me, round, i);
    gin.put(world, right, recv_w, me * S, send_w, right * S, S, CompletionAction::signal(0, SignalOp::inc()));
    gin.wait_signal(0, 1);
    const std::byte* got = recv.data() + left * S;
    for (uint64_t i = 0; i < S; ++i)
      if (got[i] != detail::ring_tag(left, round, i))
        throw VerificationFailure("ring: rank " + std::to_string(me) + " round " + std::to_string(round) +
                                  ": first mismatch at offset " + std::to_string(left * S + i));
    gin.reset_signal(0);
    gin.flush();
    barrier.sync();
  }
  if (out) {
    out->windows = {send, recv};
    out->cells = comm.snapshot_cells();
  }
  detail::release(comm, {recv_w.id(), send_w.id()});
}

inline RingReport run_ring(const LaunchOptions& opts, const RingOptions& ring) {
  if (opts.ranks < 2) throw UsageError("ring exchange needs at least 2 ranks");
  RingReport rep;
  rep.ranks = opts.ranks;
  rep.rounds = ring.rounds;
  rep.state.resize(opts.ranks);
  launch(opts, [&](DevComm& comm) { ring_rank_program(comm, ring, &rep.state[comm.rank()]); });
  return rep;
}

// ------------------------------------------------------------ microbenchmarks
struct BenchConfig {
  std::vector<uint64_t> sizes = default_sizes();
  uint32_t iters = 100;
  uint32_t warmup = 10;
  bool wall_clock = true;  // always wall clock on hardware (kept so reference code compiles)
  std::string csv_path;    // written when non-empty

  // 4 B .. 4 MiB in x2 steps (harness_bench.cpp:12-16)
  static std::vector<uint64_t> default_sizes() {
    std::vector<uint64_t> v;
    for (uint64_t s = 4; s <= (4ull << 20); s <<= 1) v.push_back(s);
    return v;
  }
};

struct BenchRow {
  uint64_t size_bytes = 0;
  uint32_t iters = 0;
  uint64_t p50_ns = 0;
  uint64_t p99_ns = 0;
  double mean_ns = 0;
};

// p50 = s[n/2], p99 = s[min(n-1, 99n/100)] of the sorted samples, and the mean
// (harness_bench.cpp:20-32; Python summarize).
inline BenchRow summarize(uint64_t size, std::vector<uint64_t> samples) {
  BenchRow row;
  row.size_bytes = size;
  row.iters = static_cast<uint32_t>(samples.size());
  if (samples.empty()) return row;
  std::sort(samples.begin(), samples.end());
  const size_t n = samples.size();
  row.p50_ns = samples[n / 2];
  row.p99_ns = samples[std::min(n - 1, n * 99 / 100)];
  double total = 0;
  for (uint64_t s : samples) total += static_cast<double>(s);
  row.mean_ns = total / static_cast<double>(n);
  return row;
}

namespace detail {
inline uint64_t mono_ns() {
  return static_cast<uint64_t>(std::chrono::duration_cast<std::chrono::nanoseconds>(
                                   std::chrono::steady_clock::now().time_since_epoch())
                                   .count());
}
inline uint64_t max_size(const BenchConfig& b) { return *std::max_element(b.sizes.begin(), b.sizes.end()); }
}  // namespace detail

// Rank 0 times put + SignalInc round trips against rank 1's echo; signal 0
// counts pings at rank 1 and pongs at rank 0 and is reset between sizes
// (harness_bench.cpp:46-88).  Rows on rank 0 only.
inline std::vector<BenchRow> pingpong_rank_program(DevComm& comm, const BenchConfig& bench) {
  const Team& world = comm.world_team();
  const uint32_t me = comm.rank();
  const uint64_t cap = detail::max_size(bench);
  std::vector<std::byte> send(cap), recv(cap);
  Window& send_w = comm.window_register(send);
  Window& recv_w = comm.window_register(recv);
  Gin gin(comm, 0);
  BarrierSession barrier(gin, world, 0);
  std::vector<BenchRow> rows;
  for (uint64_t size : bench.sizes) {
    for (uint64_t i = 0; i < size; ++i) send[i] = static_cast<std::byte>(i * 31 + me);
    barrier.sync();
    std::vector<uint64_t> samples;
    samples.reserve(bench.iters);
    for (uint32_t k = 1; k <= bench.warmup + bench.iters; ++k) {
      if (me == 0) {
        const uint64_t t0 = detail::mono_ns();
        gin.put(world, 1, recv_w, 0, send_w, 0, size, CompletionAction::signal(0, SignalOp::inc()));
        gin.wait_signal(0, k);
        const uint64_t dt = detail::mono_ns() - t0;
        if (k > bench.warmup) samples.push_back(dt);
      } else {
        gin.wait_signal(0, k);
        gin.put(world, 0, recv_w, 0, send_w, 0, size, CompletionAction::signal(0, SignalOp::inc()));
      }
    }
    gin.flush();
    barrier.sync();  // both ranks idle: the ping counter can be reset
    gin.reset_signal(0);
    barrier.sync();
    if (me == 0) rows.push_back(summarize(size, std::move(samples)));
  }
  detail::release(comm, {recv_w.id(), send_w.id()});
  return rows;
}

// Rank 0 issues `window` puts then one flush per sample (local completion of
// the batch); rank 1 is released by a signal per size (harness_bench.cpp:90-128).
inline std::vector<BenchRow> bw_rank_program(DevComm& comm, const BenchConfig& bench, uint32_t window) {
  const Team& world = comm.world_team();
  const uint32_t me = comm.rank();
  const uint64_t cap = detail::max_size(bench);
  std::vector<std::byte> send(cap), recv(uint64_t{window} * cap);
  Window& send_w = comm.window_register(send);
  Window& recv_w = comm.window_register(recv);
  Gin gin(comm, 0);
  BarrierSession barrier(gin, world, 0);
  std::vector<BenchRow> rows;
  for (uint64_t size : bench.sizes) {
    barrier.sync();
    if (me == 0) {
      std::vector<uint64_t> samples;
      for (uint32_t k = 0; k < bench.warmup + bench.iters; ++k) {
        const uint64_t t0 = detail::mono_ns();
        for (uint32_t w = 0; w < window; ++w) gin.put(world, 1, recv_w, uint64_t{w} * size, send_w, 0, size);
        gin.flush();
        const uint64_t dt = detail::mono_ns() - t0;
        if (k >= bench.warmup) samples.push_back(dt);
      }
      gin.signal(world, 1, 0, SignalOp::inc());
      rows.push_back(summarize(size, std::move(samples)));
    } else {
      gin.wait_signal(0, 1);
      gin.reset_signal(0);
    }
    barrier.sync();
  }
  detail::release(comm, {recv_w.id(), send_w.id()});
  return rows;
}

// The reference's benchmark CSV (harness_bench.cpp:167-178); the seed column
// is the config's latency seed, as in the reference.
inline void write_csv(const std::string& path, const LaunchOptions& opts, const std::vector<BenchRow>& rows) {
  const uint64_t seed = opts.config.latency.seed;
  std::ofstream f(path);
  if (!f) throw UsageError("cannot write CSV to " + path);
  f << "size_bytes,iters,p50_ns,p99_ns,mean_ns,backend,transport,seed\n";
  const char* backend = to_string(opts.config.backend.value_or(BackendKind::Direct));
  const char* transport = to_string(opts.transport);
  for (const BenchRow& r : rows)
    f << r.size_bytes << ',' << r.iters << ',' << r.p50_ns << ',' << r.p99_ns << ',' << r.mean_ns << ',' << backend
      << ',' << transport << ',' << seed << '\n';
}

namespace detail {
inline void check_bench(const LaunchOptions& opts, const BenchConfig& bench) {
  if (opts.ranks != 2) throw UsageError("point-to-point benchmarks need exactly 2 ranks");
  if (bench.sizes.empty() || !std::is_sorted(bench.sizes.begin(), bench.sizes.end()))
    throw UsageError("bench sizes must be ascending and non-empty");
  if (bench.iters == 0) throw UsageError("bench iterations must be positive");
}
inline std::vector<BenchRow> run_p2p(const LaunchOptions& opts, const BenchConfig& bench,
                                     const std::function<std::vector<BenchRow>(DevComm&)>& body) {
  check_bench(opts, bench);
  std::vector<BenchRow> rows;
  std::mutex mu;
  launch(opts, [&](DevComm& comm) {
    std::vector<BenchRow> mine = body(comm);
    if (comm.rank() == 0) {
      std::lock_guard<std::mutex> lk(mu);
      rows = std::move(mine);
    }
  });
  if (!bench.csv_path.empty()) write_csv(bench.csv_path, opts, rows);
  return rows;
}
}  // namespace detail

// Exactly 2 ranks; rows from rank 0 (harness.hpp:84-89).
inline std::vector<BenchRow> run_pingpong(const LaunchOptions& opts, const BenchConfig& bench) {
  return detail::run_p2p(opts, bench, [&](DevComm& c) { return pingpong_rank_program(c, bench); });
}
inline std::vector<BenchRow> run_bw(const LaunchOptions& opts, const BenchConfig& bench, uint32_t window = 16) {
  if (window == 0) throw UsageError("bandwidth window must be positive");
  return detail::run_p2p(opts, bench, [&](DevComm& c) { return bw_rank_program(c, bench, window); });
}

}  // namespace ginsim
