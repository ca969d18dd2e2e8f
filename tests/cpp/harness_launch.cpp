// ginsim::launch / launch_pool (include/ginsim/harness.hpp; the reference's
// proj/core/include/ginsim/harness.hpp:13-30) over the B200 library.
//   ./harness_launch        host-only checks: option validation, LaunchOptions defaults
//   ./harness_launch gpu    3 ranks (threads) on cuda:0 through launch (Inproc) -- a put + signal ring
//                           -- and launch_pool (2 comms per rank); a rank failure is rethrown;
//                           the reference's harness programs over host windows: run_ring (3 ranks,
//                           both backends; the final states agree), run_pingpong / run_bw + CSV
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
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

  // summarize (harness_bench.cpp:20-32): p50 = s[n/2], p99 = s[min(n-1, 99n/100)]
  std::vector<uint64_t> s;
  for (uint64_t i = 200; i >= 1; --i) s.push_back(i * 10);
  const ginsim::BenchRow row = ginsim::summarize(64, s);
  EXPECT(row.size_bytes == 64 && row.iters == 200 && row.p50_ns == 1010 && row.p99_ns == 1990);
  EXPECT(row.mean_ns == 1005.0);
  EXPECT(ginsim::summarize(8, {}).iters == 0 && ginsim::summarize(8, {}).p50_ns == 0);
  EXPECT(ginsim::summarize(8, {7}).p50_ns == 7 && ginsim::summarize(8, {7}).p99_ns == 7);
  // default sizes: 4 B .. 4 MiB, x2 (harness_bench.cpp:12-16)
  const auto sizes = ginsim::BenchConfig::default_sizes();
  EXPECT(sizes.size() == 21 && sizes.front() == 4 && sizes.back() == (4ull << 20));
  // the reference's CSV schema (harness_bench.cpp:167-178)
  ginsim::LaunchOptions co;
  co.config.backend = ginsim::BackendKind::Proxy;
  EXPECT(co.config.latency.seed == 0x5EED && co.config.latency.base_delay_ns == 500);  // runtime.hpp:36-37
  co.config.latency.seed = 3;
  // config_from_env applies the latency variables (runtime.cpp:53-56)
  setenv("GINSIM_SEED", "0x2A", 1);
  setenv("GINSIM_REORDER", "8", 1);
  const ginsim::Config env = ginsim::config_from_env();
  EXPECT(env.latency.seed == 42 && env.latency.reorder_window == 8 && env.latency.base_delay_ns == 500);
  setenv("GINSIM_JITTER_NS", "12x", 1);
  EXPECT(throws<ginsim::UsageError>([] { ginsim::config_from_env(); }));
  unsetenv("GINSIM_SEED");
  unsetenv("GINSIM_REORDER");
  unsetenv("GINSIM_JITTER_NS");
  const char* path = "harness_launch_test.csv";
  ginsim::write_csv(path, co, {row, ginsim::summarize(128, {5, 6, 7})});
  std::ifstream in(path);
  std::stringstream ss;
  ss << in.rdbuf();
  EXPECT(ss.str() == "size_bytes,iters,p50_ns,p99_ns,mean_ns,backend,transport,seed\n"
                     "64,200,1010,1990,1005,proxy,inproc,3\n"
                     "128,3,6,7,6,proxy,inproc,3\n");
  std::remove(path);
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::write_csv("/nonexistent-dir/x.csv", co, {}); }));
  // argument checks before any device work (harness_ring.cpp:59-60, harness_bench.cpp:131-137)
  ginsim::LaunchOptions one;
  one.ranks = 1;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_ring(one, {}); }));
  ginsim::BenchConfig b;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_pingpong(one, b); }));
  ginsim::LaunchOptions three;
  three.ranks = 3;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_bw(three, b); }));
  ginsim::LaunchOptions two;
  b.sizes = {64, 8};
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_pingpong(two, b); }));
  b.sizes = {};
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_bw(two, b); }));
  b.sizes = {8};
  b.iters = 0;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_pingpong(two, b); }));
  b.iters = 4;
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::run_bw(two, b, 0); }));

  // launch_processes (harness_launch.cpp:77-119): argv = exe, args..., --rank, i
  EXPECT(throws<ginsim::UsageError>([&] { ginsim::launch_processes("/bin/sh", {"-c", "exit 0"}, 0); }));
  ginsim::launch_processes("/bin/sh", {"-c", "test \"$1\" = --rank && test \"$2\" -lt 4", "sh"}, 4);
  std::string what;
  try {
    ginsim::launch_processes("/bin/sh", {"-c", "exit $(( $2 >= 2 ? 10 + $2 : 0 ))", "sh"}, 4);
  } catch (const ginsim::ChildFailure& e) {
    what = e.what();
  }
  EXPECT(what.find("rank 2 exited with status 12") != std::string::npos);
  what.clear();
  try {
    ginsim::launch_processes("/bin/sh", {"-c", "test $2 = 1 && kill -9 $$; exit 0", "sh"}, 3);
  } catch (const ginsim::ChildFailure& e) {
    what = e.what();
  }
  EXPECT(what.find("rank 1 killed by signal 9") != std::string::npos);
  EXPECT(throws<ginsim::ChildFailure>([&] { ginsim::launch_processes("/nonexistent/exe", {}, 2); }));
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

  // the reference's harness programs over host windows
  ginsim::RingOptions ring;
  ring.bytes = 1000;
  ring.rounds = 4;
  const ginsim::RingReport direct = ginsim::run_ring(o, ring);
  ginsim::LaunchOptions op = o;
  op.config.backend = ginsim::BackendKind::Proxy;
  const ginsim::RingReport proxy = ginsim::run_ring(op, ring);
  EXPECT(direct.ranks == 3 && direct.rounds == 4 && direct.state.size() == 3);
  EXPECT(direct.state == proxy.state);  // backend equivalence (acceptance #6)
  ginsim::LaunchOptions o2 = o;
  o2.ranks = 2;
  ginsim::BenchConfig bc;
  bc.sizes = {8, 4096, 65536};
  bc.iters = 20;
  bc.warmup = 2;
  bc.csv_path = "harness_launch_pingpong.csv";
  const auto pp = ginsim::run_pingpong(o2, bc);
  EXPECT(pp.size() == 3 && pp[0].iters == 20 && pp[0].p50_ns > 0 && pp[0].p50_ns <= pp[0].p99_ns);
  std::ifstream csv(bc.csv_path);
  std::string header;
  std::getline(csv, header);
  EXPECT(header == "size_bytes,iters,p50_ns,p99_ns,mean_ns,backend,transport,seed");
  std::remove(bc.csv_path.c_str());
  bc.csv_path.clear();
  const auto bw = ginsim::run_bw(o2, bc, 4);
  EXPECT(bw.size() == 3 && bw[2].size_bytes == 65536 && bw[2].iters == 20);
  std::printf("harness programs ok\n");
}

int main(int argc, char** argv) {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  host_checks();
  if (argc > 1 && std::string(argv[1]) == "gpu") gpu();
  return 0;
}
