// ginsim/harness.hpp -- the reference's launch helpers over the B200 library:
// LaunchOptions, launch, launch_pool (proj/core/include/ginsim/harness.hpp:13-30).
// One host thread per rank; each builds its communicator(s) with comm_init
// over an InProcGroup (TransportKind::Inproc) or comm_init_socket
// (TransportKind::Socket, the Proxy backend's GIN1 transport), runs the
// program, waits until every rank's program has returned, then tears its
// communicators down (a rank must not unmap its windows while a peer may
// still write them), and the first rank failure is rethrown after the join.
// Device: Config::device < 0 puts rank r on GPU r % device count.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <exception>
#include <functional>
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

}  // namespace ginsim
