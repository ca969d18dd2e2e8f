// A ginsim program written against the reference's C++ host surface
// (proj/core/include/ginsim/{types,runtime}.hpp), built against this repo's
// include/ginsim/runtime.hpp + libginsim_b200.so -- the drop-in boundary.
//   ./ring_ref_api        host-only checks (no GPU needed)
//   ./ring_ref_api gpu    + the Listing-2 ring (harness_ring.cpp:18-57) on
//                           2 ranks (threads) sharing cuda:0
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <thread>
#include <vector>

#include "ginsim/runtime.hpp"

#define EXPECT(c)                                                        \
  do {                                                                   \
    if (!(c)) {                                                          \
      std::fprintf(stderr, "FAILED %s at %s:%d\n", #c, __FILE__, __LINE__); \
      std::exit(1);                                                      \
    }                                                                    \
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
  // pool_select (test_runtime.cpp:73-77)
  EXPECT((ginsim::pool_select(0) == ginsim::PoolSelection{0, 0}));
  EXPECT((ginsim::pool_select(7) == ginsim::PoolSelection{1, 3}));
  EXPECT((ginsim::pool_select(23) == ginsim::PoolSelection{5, 3}));
  // SignalOp / CompletionAction (types.hpp:27-72)
  EXPECT(ginsim::SignalOp::inc().amount() == 1);
  EXPECT(ginsim::SignalOp::add(41).amount() == 41);
  const auto a = ginsim::CompletionAction::signal(9, ginsim::SignalOp::add(1)).with_counter(3);
  const ginsim_cuda_action c = a.to_c();
  EXPECT(c.signal_id == 9 && c.signal_add == 1 && c.operand == 1 && c.counter_id == 3);
  // Team translation errors (types.cpp:16-22)
  const auto team = ginsim::Team::world(4);
  EXPECT(ginsim::team_translate(team, 3) == 3);
  EXPECT(throws<ginsim::RankOutOfRange>([&] { ginsim::team_translate(team, 4); }));
  // Config defaults (runtime.hpp:29-44)
  const ginsim::Config cfg;
  EXPECT(cfg.n_contexts == 4 && cfg.signal_cells == 256 && cfg.counter_cells == 256 && cfg.queue_depth == 1024);
  // descriptor golden bytes through the C ABI (test_descriptor.cpp:60-79)
  ginsim_cuda_descriptor d{};
  d.opcode = 1;
  d.flags = 0x03;
  d.peer = 1;
  d.dst_window = 2;
  d.dst_offset = 0x40;
  d.src_window = 7;
  d.src_offset_or_value = 0x100;
  d.bytes = 14352;
  d.signal_id = 9;
  d.signal_operand = 1;
  uint8_t raw[64];
  EXPECT(ginsim_cuda_descriptor_encode(&d, raw) == GINSIM_OK);
  EXPECT(raw[0] == 0x01 && raw[1] == 0x03 && raw[4] == 1 && raw[8] == 2 && raw[12] == 7);
  // an inline put over 8 bytes is rejected with the reference's exception type
  d.opcode = 2;
  d.src_window = 0xFFFFFFFFu;
  d.bytes = 9;
  EXPECT(throws<ginsim::InvalidDescriptor>([&] { ginsim::check(ginsim_cuda_descriptor_encode(&d, raw)); }));
  std::printf("host checks ok\n");
}

// harness_ring.cpp:18-57 over 2 ranks: put + SignalInc to the right
// neighbour, wait, verify the (rank, round) bytes, reset, flush, barrier.
static void ring_gpu() {
  constexpr uint32_t kRanks = 2, kRounds = 5;
  constexpr uint64_t kBytes = 4096;
  auto group = ginsim::InProcGroup::create(kRanks);
  std::vector<std::thread> ts;
  std::vector<int> ok(kRanks, 0);
  for (uint32_t r = 0; r < kRanks; ++r) {
    ts.emplace_back([&, r] {
      ginsim::Config cfg;
      cfg.device = 0;  // ranks emulated on one B200
      auto comm = ginsim::comm_init(group, r, cfg);
      auto sbuf = ginsim::mem_alloc(*comm, kBytes);
      auto rbuf = ginsim::mem_alloc(*comm, kBytes);
      ginsim::Window& send = comm->window_register(sbuf);
      ginsim::Window& recv = comm->window_register(rbuf);
      ginsim::Gin gin(*comm, 0);
      ginsim::BarrierSession barrier(gin, comm->world_team(), 0);
      std::vector<uint8_t> host(kBytes);
      for (uint32_t round = 0; round < kRounds; ++round) {
        for (uint64_t i = 0; i < kBytes; ++i) host[i] = (uint8_t)(r * 131 + round * 31 + i * 7 + 1);
        cudaMemcpy(sbuf.data(), host.data(), kBytes, cudaMemcpyHostToDevice);
        const uint32_t right = (r + 1) % kRanks, left = (r + kRanks - 1) % kRanks;
        gin.put(comm->world_team(), right, recv, 0, send, 0, kBytes, ginsim::CompletionAction::signal(0));
        gin.wait_signal(0, 1);
        cudaMemcpy(host.data(), rbuf.data(), kBytes, cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < kBytes; ++i) EXPECT(host[i] == (uint8_t)(left * 131 + round * 31 + i * 7 + 1));
        gin.reset_signal(0);
        gin.flush();
        barrier.sync();
      }
      // put_value little-endian at the target (test_runtime.cpp:175-199)
      gin.put_value(comm->world_team(), (r + 1) % kRanks, recv, 16, (uint32_t)0xDEADBEEFu,
                    ginsim::CompletionAction::signal(1));
      gin.wait_signal(1, 1);
      uint8_t v[4];
      cudaMemcpy(v, rbuf.data() + 16, 4, cudaMemcpyDeviceToHost);
      EXPECT(v[0] == 0xEF && v[1] == 0xBE && v[2] == 0xAD && v[3] == 0xDE);
      // out-of-bounds puts raise the reference's exception type (types.cpp:52-60)
      EXPECT(throws<ginsim::OutOfBounds>(
          [&] { gin.put(comm->world_team(), (r + 1) % kRanks, recv, kBytes - 7, send, 0, 8); }));
      // DevComm::submit_op / wait_until / pump_local (runtime.hpp:164-191)
      comm->submit_op(0, comm->world_team(), (r + 1) % kRanks, ginsim::Opcode::PutInline, recv.id(), 24,
                      ginsim::kInlineWindow, 0x0A0B, 2, ginsim::CompletionAction::signal(2));
      comm->wait_until([&] { return comm->read_signal(2) >= 1; }, "submit_op signal");
      EXPECT(comm->pump_local() == 0);
      EXPECT(comm->virtual_now() > 0 && comm->transport_kind() == ginsim::TransportKind::Nvlink);
      EXPECT(throws<ginsim::RankOutOfRange>([&] {
        comm->submit_op(0, comm->world_team(), 9, ginsim::Opcode::Put, recv.id(), 0, send.id(), 0, 8, {});
      }));
      barrier.sync();
      comm->check_failed();
      ok[r] = 1;
    });
  }
  for (auto& t : ts) t.join();
  EXPECT(ok[0] && ok[1]);
  std::printf("ring ok\n");
}

int main(int argc, char** argv) {
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "gpu") ring_gpu();
  return 0;
}
