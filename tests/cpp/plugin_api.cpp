// The reference's plugin boundary (proj/core/include/ginsim/plugin.hpp:64-144,
// direct_backend.hpp:17-63) driven through include/ginsim/plugin.hpp over the
// C ABI, on both backends, plus sub-team registration (runtime.hpp:145-148):
//   ./plugin_api        host-only checks (no GPU)
//   ./plugin_api gpu    2 ranks (threads) sharing cuda:0:
//     proxy  : reg_mr -> iput_signal -> test -> retire (the CompletionAction
//              comes back exactly once; UnknownHandle afterwards), iput with a
//              remote signal rejected, inline iput, create_context is a
//              BackendMismatch;
//     direct : create_context -> post (put + signal + counter) -> poll ->
//              outstanding == 0; iput is a BackendMismatch;
//     teams  : register_team({1, 0}) then Gin ops over the team's ranks.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "ginsim/plugin.hpp"

#define EXPECT(c)                                                           \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::fprintf(stderr, "FAILED %s at %s:%d\n", #c, __FILE__, __LINE__); \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static void host_checks() {
  const auto s = ginsim::PutSource::inline_bytes(0xDEADBEEF).to_c();
  EXPECT(s.is_inline == 1 && s.inline_value == 0xDEADBEEF);
  const auto w = ginsim::PutSource::window(ginsim::MrHandle{3}, 64).to_c();
  EXPECT(w.is_inline == 0 && w.mr == 3 && w.offset == 64);
  ginsim_cuda_action a{7, 1, 5, 2, 0};
  const auto act = ginsim::action_from_c(a);
  EXPECT(act.remote_signal && act.remote_signal->id == 7 && act.remote_signal->op.amount() == 5);
  EXPECT(act.local_counter && *act.local_counter == 2);
  std::printf("host checks ok\n");
}

static void run(ginsim::BackendKind backend) {
  constexpr uint32_t kRanks = 2;
  constexpr uint64_t kBytes = 1 << 16;
  auto group = ginsim::InProcGroup::create(kRanks);
  std::vector<std::thread> ts;
  std::vector<int> ok(kRanks, 0);
  for (uint32_t r = 0; r < kRanks; ++r) {
    ts.emplace_back([&, r] {
      ginsim::Config cfg;
      cfg.device = 0;
      cfg.backend = backend;
      auto comm = ginsim::comm_init(group, r, cfg);
      auto sbuf = ginsim::mem_alloc(*comm, kBytes);
      auto rbuf = ginsim::mem_alloc(*comm, kBytes);
      ginsim::Window& send = comm->window_register(sbuf);
      ginsim::Window& recv = comm->window_register(rbuf);
      std::vector<uint8_t> host(kBytes);
      for (uint64_t i = 0; i < kBytes; ++i) host[i] = (uint8_t)(r * 37 + i * 11 + 5);
      cudaMemcpy(sbuf.data(), host.data(), kBytes, cudaMemcpyHostToDevice);
      ginsim::Gin gin(*comm, 0);
      ginsim::BarrierSession barrier(gin, comm->world_team(), 0);
      barrier.sync();
      const uint32_t peer = (r + 1) % kRanks, left = (r + kRanks - 1) % kRanks;
      ginsim::FabricPlugin plugin(*comm, backend);
      if (backend == ginsim::BackendKind::Proxy) {
        plugin.set_call_log_enabled(true);
        const auto mr_s = plugin.reg_mr(send.id());
        const auto mr_r = plugin.reg_mr(recv.id());
        EXPECT(plugin.reg_mr(send.id()) == mr_s);  // idempotent
        EXPECT(plugin.is_registered(recv.id()));
        EXPECT(throws<ginsim::UnknownWindow>([&] { plugin.reg_mr(99); }));
        const auto req = plugin.iput_signal(ginsim::PutSource::window(mr_s, 0), mr_r, 0, kBytes, peer, 1, 4,
                                            ginsim::SignalOp::add(3), ginsim::CompletionAction::counter(2));
        EXPECT(plugin.outstanding_requests() == 1);
        auto t0 = std::chrono::steady_clock::now();
        while (!plugin.test(req)) {
          EXPECT(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(20));
          std::this_thread::yield();
        }
        EXPECT(plugin.test(req));  // idempotent once true
        const auto done = plugin.retire(req);
        EXPECT(done.local_counter && *done.local_counter == 2 && !done.remote_signal);
        EXPECT(throws<ginsim::UnknownHandle>([&] { plugin.retire(req); }));
        EXPECT(throws<ginsim::UnknownHandle>([&] { plugin.test(req + 1000); }));
        EXPECT(plugin.outstanding_requests() == 0);
        EXPECT(comm->read_counter(2) == 1);
        // iput carries no remote signal (plugin.cpp:85-88)
        EXPECT(throws<ginsim::Error>([&] {
          plugin.iput(ginsim::PutSource::window(mr_s, 0), mr_r, 0, 8, peer, 0, ginsim::CompletionAction::signal(1));
        }));
        // an inline iput (<= 8 bytes in the descriptor)
        const auto req2 =
            plugin.iput(ginsim::PutSource::inline_bytes(0x0102030405060708ull), mr_r, kBytes - 8, 8, peer, 0, {});
        while (!plugin.test(req2)) std::this_thread::yield();
        plugin.retire(req2);
        // the posting trace: iput_signal, (rejected) iput, inline iput -- in order, from this thread
        const auto log = plugin.call_log();
        EXPECT(log.size() == 2 && log[0].op == 's' && log[0].bytes == kBytes && log[0].peer == peer &&
               log[0].ctx == 1 && log[1].op == 'p' && log[1].bytes == 8 && log[0].issuer == log[1].issuer);
        EXPECT(throws<ginsim::BackendMismatch>([&] { plugin.create_context(0); }));
      } else {
        EXPECT(throws<ginsim::BackendMismatch>([&] {
          plugin.iput(ginsim::PutSource::window(ginsim::MrHandle{send.id()}, 0), ginsim::MrHandle{recv.id()}, 0, 8,
                      peer, 0, {});
        }));
        EXPECT(throws<ginsim::InvalidContext>([&] { plugin.create_context(9); }));
        ginsim::DirectContext& dc = plugin.create_context(1);
        EXPECT(&plugin.create_context(1) == &dc);
        ginsim::ResolvedOp op;
        op.opcode = ginsim::Opcode::Put;
        op.peer = peer;
        op.dst_window = recv.id();
        op.src_window = send.id();
        op.bytes = kBytes;
        op.action = ginsim::CompletionAction::signal(4, ginsim::SignalOp::add(3)).with_counter(2);
        dc.post(op);
        ginsim::ResolvedOp iv;
        iv.opcode = ginsim::Opcode::PutInline;
        iv.peer = peer;
        iv.dst_window = recv.id();
        iv.dst_offset = kBytes - 8;
        iv.src_offset_or_value = 0x0102030405060708ull;
        iv.bytes = 8;
        dc.post(iv);
        size_t retired = 0;
        auto t0 = std::chrono::steady_clock::now();
        while (dc.outstanding() > 0) {
          retired += dc.poll();
          EXPECT(std::chrono::steady_clock::now() - t0 < std::chrono::seconds(20));
        }
        EXPECT(retired == 2 && dc.poll() == 0);
        EXPECT(comm->read_counter(2) == 1);
      }
      std::printf("rank %u: %s ops posted, waiting for the peer's signal\n", r,
                  backend == ginsim::BackendKind::Proxy ? "proxy" : "direct");
      comm->wait_signal(4, 3);
      barrier.sync();
      cudaDeviceSynchronize();
      cudaMemcpy(host.data(), rbuf.data(), kBytes, cudaMemcpyDeviceToHost);
      for (uint64_t i = 0; i < kBytes - 8; ++i) EXPECT(host[i] == (uint8_t)(left * 37 + i * 11 + 5));
      for (int i = 0; i < 8; ++i) EXPECT(host[kBytes - 8 + i] == 8 - i);
      // sub-team {1, 0}: team rank 0 is world rank 1 (runtime.cpp:329-343)
      const ginsim::Team& t = comm->register_team(ginsim::Team{5, {1, 0}});
      EXPECT(&comm->team(5) == &t);
      EXPECT(throws<ginsim::UsageError>([&] { comm->register_team(ginsim::Team{5, {0}}); }));
      EXPECT(throws<ginsim::InvalidPeer>([&] { comm->register_team(ginsim::Team{6, {0, 7}}); }));
      std::printf("rank %u: data checked, team ops\n", r);
      const uint32_t team_peer = r == 1 ? 1u : 0u;  // the other rank, in team-relative numbering
      gin.put_value(t, team_peer, recv, 0, (uint32_t)(0xC0DE0000u + r), ginsim::CompletionAction::signal(6));
      try {
        comm->wait_signal(6, 1);
      } catch (const ginsim::Timeout&) {
        uint64_t d = 0, cp = 0, busy = 0, wall = 0;
        if (backend == ginsim::BackendKind::Proxy) ginsim_cuda_proxy_stats(comm->handle(), &d, &cp, &busy, &wall);
        uint32_t raw = 0;
        cudaMemcpy(&raw, rbuf.data(), 4, cudaMemcpyDeviceToHost);
        std::printf("rank %u: TIMEOUT cell6=%llu data=%08x descriptors=%llu copies=%llu\n", r,
                    (unsigned long long)comm->read_signal(6), raw, (unsigned long long)d, (unsigned long long)cp);
        throw;
      }
      uint32_t v = 0;
      cudaMemcpy(&v, rbuf.data(), 4, cudaMemcpyDeviceToHost);
      EXPECT(v == 0xC0DE0000u + left);
      gin.flush();
      barrier.sync();
      comm->check_failed();
      ok[r] = 1;
    });
  }
  for (auto& t : ts) t.join();
  EXPECT(ok[0] && ok[1]);
  std::printf("%s plugin ok\n", backend == ginsim::BackendKind::Proxy ? "proxy" : "direct");
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);  // progress lines survive an abort
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "gpu") {
    run(ginsim::BackendKind::Direct);
    run(ginsim::BackendKind::Proxy);
  }
  return 0;
}
