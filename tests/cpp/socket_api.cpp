// comm_init_socket (the reference's socket flavour of a communicator,
// proj/core/include/ginsim/socket_transport.hpp:117-129) over the B200 library:
// rank 0 hosts the rendezvous on a loopback port from reserve_loopback_port,
// every rank's Proxy agent reaches the others with GIN1 frames over TCP.
//   ./socket_api        host-only checks (no GPU): the Config carries the transport
//   ./socket_api gpu    3 ranks (threads) on cuda:0: a put + SignalAdd ring with
//                       a local counter, inline values, a dissemination barrier,
//                       transport_kind() == Socket; a Direct-backend request is a
//                       BackendMismatch
#include <cuda_runtime.h>

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

static void host_checks() {
  ginsim::Config cfg;
  EXPECT(cfg.to_c().transport == 0);
  cfg.transport = ginsim::TransportKind::Socket;
  EXPECT(cfg.to_c().transport == 1);
  EXPECT(ginsim::reserve_loopback_port() > 0);
  std::printf("host checks ok\n");
}

static void ring() {
  constexpr uint32_t kRanks = 3, kRounds = 4;
  constexpr uint64_t kBytes = 1 << 16;
  const uint16_t port = ginsim::reserve_loopback_port();
  std::vector<std::thread> ts;
  std::vector<int> ok(kRanks, 0);
  for (uint32_t r = 0; r < kRanks; ++r) {
    ts.emplace_back([&, r] {
      ginsim::Config cfg;
      cfg.device = 0;
      cfg.timeout_ms = 20000;
      auto comm = ginsim::comm_init_socket("127.0.0.1", port, kRanks, r, cfg);
      EXPECT(comm->transport_kind() == ginsim::TransportKind::Socket);
      EXPECT(comm->backend() == ginsim::BackendKind::Proxy);
      auto sbuf = ginsim::mem_alloc(*comm, kRanks * kBytes);
      auto rbuf = ginsim::mem_alloc(*comm, kRanks * kBytes + 64);  // + a word for the inline values
      ginsim::Window& send = comm->window_register(sbuf);
      ginsim::Window& recv = comm->window_register(rbuf);
      ginsim::Gin gin(*comm, r % 2);
      ginsim::BarrierSession barrier(gin, comm->world_team(), 0);
      const uint32_t right = (r + 1) % kRanks, left = (r + kRanks - 1) % kRanks;
      std::vector<uint8_t> host(kBytes);
      for (uint32_t round = 0; round < kRounds; ++round) {
        for (uint64_t i = 0; i < kBytes; ++i) host[i] = (uint8_t)(r * 31 + round * 7 + i * 5 + 1);
        cudaMemcpy(sbuf.data() + right * kBytes, host.data(), kBytes, cudaMemcpyHostToDevice);
        gin.put(comm->world_team(), right, recv, r * kBytes, send, right * kBytes, kBytes,
                ginsim::CompletionAction::signal(0, ginsim::SignalOp::add(2)).with_counter(1));
        gin.put_value(comm->world_team(), right, recv, kRanks * kBytes, (uint32_t)(0xC0DE0000u + r * 16 + round),
                      ginsim::CompletionAction::signal(1));
        gin.flush();  // local completion: the peer acked the frames
        EXPECT(comm->read_counter(1) == round + 1);
        comm->wait_signal(0, 2 * (round + 1));
        comm->wait_signal(1, round + 1);
        cudaMemcpy(host.data(), rbuf.data() + left * kBytes, kBytes, cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < kBytes; ++i) EXPECT(host[i] == (uint8_t)(left * 31 + round * 7 + i * 5 + 1));
        uint32_t v = 0;
        cudaMemcpy(&v, rbuf.data() + kRanks * kBytes, 4, cudaMemcpyDeviceToHost);
        EXPECT(v == 0xC0DE0000u + left * 16 + round);
        barrier.sync();
      }
      comm->check_failed();
      ok[r] = 1;
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < kRanks; ++r) EXPECT(ok[r]);
  // the socket transport needs the Proxy backend
  bool refused = false;
  try {
    ginsim::Config d;
    d.backend = ginsim::BackendKind::Direct;
    ginsim::comm_init_socket("127.0.0.1", ginsim::reserve_loopback_port(), 1, 0, d);
  } catch (const ginsim::BackendMismatch&) {
    refused = true;
  }
  EXPECT(refused);
  std::printf("socket ring ok\n");
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "gpu") ring();
  return 0;
}
