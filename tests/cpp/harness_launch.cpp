// ginsim::launch / launch_pool (include/ginsim/harness.hpp; the reference's
// proj/core/include/ginsim/harness.hpp:13-30) over the B200 library.
//   ./harness_launch        host-only checks: option validation, LaunchOptions defaults
//   ./harness_launch gpu    3 ranks (threads) on cuda:0 through launch (Inproc) -- a put + signal ring
//                           -- and launch_pool (2 comms per rank); a rank failure is rethrown
#include <cstdio>
#include <cstdlib>
#include <string>

#include "ginsim/harness.hpp"

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
  ginsim::LaunchOptions o;
  EXPECT(o.ranks == 2 && o.transport == ginsim::TransportKind::Inproc && o.port == 0 && o.host == "127.0.0.1");
  o.ranks = 0;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::launch(o, [](ginsim::DevComm&) {}); }));
  o.ranks = 9;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::launch(o, [](ginsim::DevComm&) {}); }));
  o.ranks = 2;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::launch_pool(o, 0, [](std::vector<ginsim::DevComm*>&) {}); }));
  o.transport = ginsim::TransportKind::Socket;
  o.config.backend = ginsim::BackendKind::Direct;
  EXPECT(throws<ginsim::BackendMismatch>([&] { ginsim::launch(o, [](ginsim::DevComm&) {}); }));
  std::printf("host checks ok\n");
}

static void gpu() {
  ginsim::LaunchOptions o;
  o.ranks = 3;
  o.config.device = 0;
  o.config.timeout_ms = 20000;
  constexpr uint64_t kBytes = 4096;
  ginsim::launch(o, [&](ginsim::DevComm& comm) {
    auto buf = ginsim::mem_alloc(comm, 2 * kBytes);
    ginsim::Window& w = comm.window_register(buf);
    ginsim::Gin gin(comm, 0);
    const uint32_t right = (comm.rank() + 1) % comm.world_size();
    gin.put_value(comm.world_team(), right, w, kBytes, 0xA0u + comm.rank(), ginsim::CompletionAction::signal(0));
    comm.wait_signal(0, 1);
    uint32_t v = 0;
    cudaMemcpy(&v, buf.data() + kBytes, 4, cudaMemcpyDeviceToHost);
    EXPECT(v == 0xA0u + (comm.rank() + comm.world_size() - 1) % comm.world_size());
  });
  ginsim::launch_pool(o, 2, [&](std::vector<ginsim::DevComm*>& comms) {
    EXPECT(comms.size() == 2 && comms[0]->rank() == comms[1]->rank());
  });
  // the first rank failure comes back after every rank joined
  EXPECT(throws<ginsim::UsageError>([&] {
    ginsim::launch(o, [](ginsim::DevComm& comm) {
      if (comm.rank() == 1) throw ginsim::UsageError("rank 1 fails");
    });
  }));
  std::printf("launch ok\n");
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "gpu") gpu();
  return 0;
}
