// Host-API compatibility: a ginsim host program whose windows are plain
// std::vector<std::byte> buffers, as the reference's own programs register
// them (harness_ring.cpp:18-57 registers std::vector send/recv buffers and
// reads/writes them directly), running unchanged over the B200 library:
// window_register pins and maps the host pages (cudaHostRegister), the put /
// signal path moves the bytes on the GPU, and the host fills and verifies the
// windows with ordinary loads and stores.
//   ./host_windows gpu     4 ranks (threads) on cuda:0, both backends
#include <cstdio>
#include <cstdlib>
#include <string>
#include <thread>
#include <vector>

#include "ginsim/runtime.hpp"

#define EXPECT(c)                                                           \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::fprintf(stderr, "FAILED %s at %s:%d\n", #c, __FILE__, __LINE__); \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

static uint8_t pattern(uint32_t sender, uint32_t round, uint64_t i) {
  return (uint8_t)(sender * 29 + round * 7 + i * 3 + 11);
}

static void ring(ginsim::BackendKind backend) {
  constexpr uint32_t kRanks = 4, kRounds = 6;
  constexpr uint64_t kBytes = 8192;
  auto group = ginsim::InProcGroup::create(kRanks);
  std::vector<std::thread> ts;
  std::vector<int> ok(kRanks, 0);
  for (uint32_t r = 0; r < kRanks; ++r) {
    ts.emplace_back([&, r] {
      ginsim::Config cfg;
      cfg.device = 0;
      cfg.backend = backend;
      auto comm = ginsim::comm_init(group, r, cfg);
      // the reference's way: plain host vectors as window memory
      std::vector<std::byte> send_buf(kRanks * kBytes), recv_buf(kRanks * kBytes);
      ginsim::Window& send = comm->window_register(send_buf);
      ginsim::Window& recv = comm->window_register(recv_buf);
      ginsim::Gin gin(*comm, 0);
      ginsim::BarrierSession barrier(gin, comm->world_team(), 0);
      const uint32_t right = (r + 1) % kRanks, left = (r + kRanks - 1) % kRanks;
      for (uint32_t round = 0; round < kRounds; ++round) {
        for (uint64_t i = 0; i < kBytes; ++i) send_buf[right * kBytes + i] = (std::byte)pattern(r, round, i);
        gin.put(comm->world_team(), right, recv, r * kBytes, send, right * kBytes, kBytes,
                ginsim::CompletionAction::signal(0));
        gin.wait_signal(0, 1);
        for (uint64_t i = 0; i < kBytes; ++i) EXPECT(recv_buf[left * kBytes + i] == (std::byte)pattern(left, round, i));
        gin.reset_signal(0);
        gin.flush();
        barrier.sync();
      }
      // an inline value lands little-endian in the peer's host window
      gin.put_value(comm->world_team(), right, recv, 8, (uint32_t)(0xFEED0000u + r), ginsim::CompletionAction::signal(1));
      gin.wait_signal(1, 1);
      const uint32_t want = 0xFEED0000u + left;
      for (int b = 0; b < 4; ++b) EXPECT(recv_buf[8 + b] == (std::byte)((want >> (8 * b)) & 0xFF));
      barrier.sync();
      // unpin the host pages before the vectors go away (the caller owns window bytes)
      comm->window_deregister(recv.id());
      comm->window_deregister(send.id());
      comm->check_failed();
      ok[r] = 1;
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < kRanks; ++r) EXPECT(ok[r]);
  std::printf("%s host-window ring ok\n", backend == ginsim::BackendKind::Proxy ? "proxy" : "direct");
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 1 && std::string(argv[1]) == "gpu") {
    ring(ginsim::BackendKind::Direct);
    ring(ginsim::BackendKind::Proxy);
  } else {
    std::printf("host checks ok\n");
  }
  return 0;
}
