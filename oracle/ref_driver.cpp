// ref_driver.cpp — ORACLE HARNESS (test infrastructure only).
//
// Links the UNMODIFIED reference library (oracle/_ref/libginsim_ref.a, built
// from /root/reference/proj/core/src by oracle/build_ref.sh) and drives its
// public API: run_moe_ll (proj/core/src/harness_moe.cpp:252), run_moe_ht
// (:384), run_pingpong / run_bw (harness_bench.cpp:156,161), run_ring
// (harness_ring.cpp:59) and the descriptor codec / DescriptorRing.  Used to
// generate tests/golden/ fixtures and as bench.py's CPU reference arm.
// Prints one JSON object per invocation on stdout.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "ginsim/descriptor.hpp"
#include "ginsim/harness.hpp"
#include "ginsim/proxy_backend.hpp"
#include "ginsim/runtime.hpp"
#include "ginsim/wire.hpp"

using namespace ginsim;
using clk = std::chrono::steady_clock;

namespace {

uint64_t arg_u64(int argc, char** argv, const char* name, uint64_t dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return std::strtoull(argv[i + 1], nullptr, 0);
  return dflt;
}
std::string arg_str(int argc, char** argv, const char* name, const char* dflt) {
  for (int i = 1; i + 1 < argc; ++i)
    if (std::strcmp(argv[i], name) == 0) return argv[i + 1];
  return dflt;
}

LaunchOptions options(int argc, char** argv) {
  LaunchOptions o;
  o.ranks = static_cast<uint32_t>(arg_u64(argc, argv, "--ranks", 2));
  o.config.backend =
      arg_str(argc, argv, "--backend", "direct") == "proxy" ? BackendKind::Proxy : BackendKind::Direct;
  o.config.latency = LatencyModel{};  // zero delay, no line-rate term: wall-clock CPU cost only
  o.config.timeout_ms = 600'000;
  return o;
}

void dump(const std::string& path, const void* p, size_t n) {
  std::ofstream f(path, std::ios::binary);
  f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
}

double secs(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double>(b - a).count();
}

// Restatement of proj/tests/test_descriptor.cpp:24-55 (random_valid), compiled
// by the same g++ so argument evaluation order matches the reference's tests.
Descriptor random_valid(std::mt19937_64& rng) {
  auto u64 = [&] { return rng(); };
  auto u32 = [&] { return static_cast<uint32_t>(rng()); };
  CompletionAction action;
  switch (rng() % 4) {
    case 0: break;
    case 1: action.remote_signal = {u32() % 4096, SignalOp::inc()}; break;
    case 2: action.remote_signal = {u32() % 4096, SignalOp::add(u64())}; break;
    case 3:
      action.remote_signal = {u32() % 4096, SignalOp::add(u64())};
      action.local_counter = u32() % 4096;
      break;
  }
  if (rng() % 2) action.local_counter = u32() % 4096;
  switch (rng() % 3) {
    case 0:
      return make_put_descriptor(static_cast<TeamId>(rng()), u32(), u32(), u64(),
                                 u32() & 0x7FFFFFFF, u64(), u64(), action);
    case 1:
      return make_put_inline_descriptor(static_cast<TeamId>(rng()), u32(), u32(), u64(), u64(),
                                        rng() % 9, action);
    default: {
      SignalOp op = (rng() % 2) ? SignalOp::add(u64()) : SignalOp::inc();
      CompletionAction rest;
      rest.local_counter = action.local_counter;
      return make_signal_descriptor(static_cast<TeamId>(rng()), u32(), u32() % 4096, op, rest);
    }
  }
}

int cmd_moe_ll(int argc, char** argv) {
  LaunchOptions o = options(argc, argv);
  MoeConfig cfg;
  cfg.experts = static_cast<uint32_t>(arg_u64(argc, argv, "--experts", 256));
  cfg.top_k = static_cast<uint32_t>(arg_u64(argc, argv, "--topk", 8));
  cfg.tokens_per_rank = static_cast<uint32_t>(arg_u64(argc, argv, "--tokens", 128));
  cfg.hidden = static_cast<uint32_t>(arg_u64(argc, argv, "--hidden", 7168));
  cfg.seed = arg_u64(argc, argv, "--seed", 1);
  const uint64_t reps = arg_u64(argc, argv, "--reps", 1);
  const std::string dir = arg_str(argc, argv, "--dump", "");
  double best = 1e30, total = 0;
  MoeReport rep;
  for (uint64_t i = 0; i < reps; ++i) {
    auto t0 = clk::now();
    rep = run_moe_ll(o, cfg);
    auto t1 = clk::now();
    best = std::min(best, secs(t0, t1));
    total += secs(t0, t1);
  }
  if (!dir.empty()) {
    for (uint32_t r = 0; r < o.ranks; ++r) {
      const RankState& s = rep.state[r];
      dump(dir + "/rank" + std::to_string(r) + "_dispatch.bin", s.windows[0].data(), s.windows[0].size());
      dump(dir + "/rank" + std::to_string(r) + "_combine.bin", s.windows[1].data(), s.windows[1].size());
      dump(dir + "/rank" + std::to_string(r) + "_signals.bin", s.cells.signals.data(),
           s.cells.signals.size() * 8);
      dump(dir + "/rank" + std::to_string(r) + "_counters.bin", s.cells.counters.data(),
           s.cells.counters.size() * 8);
    }
  }
  std::printf(
      "{\"cmd\":\"moe-ll\",\"ranks\":%u,\"experts\":%u,\"topk\":%u,\"tokens\":%u,\"hidden\":%u,"
      "\"seed\":%llu,\"backend\":\"%s\",\"reps\":%llu,\"best_s\":%.6f,\"mean_s\":%.6f,"
      "\"dispatch_msg\":%llu,\"combine_msg\":%llu,\"tokens_routed\":%llu,\"threads\":%u}\n",
      o.ranks, cfg.experts, cfg.top_k, cfg.tokens_per_rank, cfg.hidden,
      (unsigned long long)cfg.seed, to_string(*o.config.backend), (unsigned long long)reps, best,
      total / reps, (unsigned long long)rep.dispatch_message_bytes,
      (unsigned long long)rep.combine_message_bytes, (unsigned long long)rep.tokens_routed,
      2 * o.ranks);
  return 0;
}

int cmd_moe_ht(int argc, char** argv) {
  LaunchOptions o = options(argc, argv);
  MoeConfig cfg;
  cfg.mode = MoeMode::HighThroughput;
  cfg.channels = static_cast<uint32_t>(arg_u64(argc, argv, "--channels", 24));
  cfg.slots = static_cast<uint32_t>(arg_u64(argc, argv, "--slots", 4));
  cfg.messages = static_cast<uint32_t>(arg_u64(argc, argv, "--messages", 64));
  cfg.seed = arg_u64(argc, argv, "--seed", 1);
  auto t0 = clk::now();
  HtReport rep = run_moe_ht(o, cfg);
  auto t1 = clk::now();
  std::printf("{\"cmd\":\"moe-ht\",\"ranks\":%u,\"channels\":%llu,\"messages_delivered\":%llu,"
              "\"wall_s\":%.6f}\n",
              o.ranks, (unsigned long long)rep.channels,
              (unsigned long long)rep.messages_delivered, secs(t0, t1));
  return 0;
}

int cmd_bench(int argc, char** argv, bool pingpong) {
  LaunchOptions o = options(argc, argv);
  o.ranks = 2;
  BenchConfig b;
  b.iters = static_cast<uint32_t>(arg_u64(argc, argv, "--iters", 200));
  b.warmup = static_cast<uint32_t>(arg_u64(argc, argv, "--warmup", 20));
  b.wall_clock = true;
  const uint64_t lo = arg_u64(argc, argv, "--min", 8), hi = arg_u64(argc, argv, "--max", 4u << 20);
  b.sizes.clear();
  for (uint64_t s = lo; s <= hi; s *= 2) b.sizes.push_back(s);
  auto rows = pingpong ? run_pingpong(o, b) : run_bw(o, b, 16);
  std::printf("{\"cmd\":\"%s\",\"backend\":\"%s\",\"rows\":[", pingpong ? "pingpong" : "bw",
              to_string(*o.config.backend));
  for (size_t i = 0; i < rows.size(); ++i) {
    std::printf("%s{\"size\":%llu,\"iters\":%u,\"p50_ns\":%llu,\"p99_ns\":%llu,\"mean_ns\":%.1f}",
                i ? "," : "", (unsigned long long)rows[i].size_bytes, rows[i].iters,
                (unsigned long long)rows[i].p50_ns, (unsigned long long)rows[i].p99_ns,
                rows[i].mean_ns);
  }
  std::printf("]}\n");
  return 0;
}

int cmd_ring(int argc, char** argv) {
  LaunchOptions o = options(argc, argv);
  RingOptions ro;
  ro.bytes = arg_u64(argc, argv, "--bytes", 4096);
  ro.rounds = static_cast<uint32_t>(arg_u64(argc, argv, "--rounds", 10));
  const std::string dir = arg_str(argc, argv, "--dump", "");
  auto t0 = clk::now();
  RingReport rep = run_ring(o, ro);
  auto t1 = clk::now();
  if (!dir.empty()) {
    for (uint32_t r = 0; r < o.ranks; ++r) {
      const RankState& s = rep.state[r];
      dump(dir + "/ring_rank" + std::to_string(r) + "_send.bin", s.windows[0].data(), s.windows[0].size());
      dump(dir + "/ring_rank" + std::to_string(r) + "_recv.bin", s.windows[1].data(), s.windows[1].size());
      dump(dir + "/ring_rank" + std::to_string(r) + "_signals.bin", s.cells.signals.data(),
           s.cells.signals.size() * 8);
    }
  }
  std::printf("{\"cmd\":\"ring\",\"ranks\":%u,\"bytes\":%llu,\"rounds\":%u,\"wall_s\":%.6f}\n",
              o.ranks, (unsigned long long)ro.bytes, ro.rounds, secs(t0, t1));
  return 0;
}

int cmd_descriptors(int argc, char** argv) {
  const uint64_t seed = arg_u64(argc, argv, "--seed", 0xD15C0);
  const uint64_t count = arg_u64(argc, argv, "--count", 10000);
  const std::string out = arg_str(argc, argv, "--out", "descriptors.bin");
  std::mt19937_64 rng(seed);
  std::vector<std::byte> all;
  all.reserve(count * kDescriptorBytes);
  for (uint64_t i = 0; i < count; ++i) {
    Descriptor d = random_valid(rng);
    EncodedDescriptor b = encode_descriptor(d);
    if (!(decode_descriptor(b) == d)) {
      std::fprintf(stderr, "reference round trip failed at %llu\n", (unsigned long long)i);
      return 1;
    }
    all.insert(all.end(), b.begin(), b.end());
  }
  dump(out, all.data(), all.size());
  std::printf("{\"cmd\":\"descriptors\",\"seed\":%llu,\"count\":%llu}\n",
              (unsigned long long)seed, (unsigned long long)count);
  return 0;
}

// DescriptorRing + decode throughput (the survey's ringbench).
int cmd_ringbench(int argc, char** argv) {
  const uint32_t producers = static_cast<uint32_t>(arg_u64(argc, argv, "--producers", 1));
  const uint64_t per = arg_u64(argc, argv, "--count", 1'000'000);
  const uint64_t cap = arg_u64(argc, argv, "--capacity", 1024);
  DescriptorRing ring(cap);
  const EncodedDescriptor enc = encode_descriptor(
      make_put_descriptor(0, 1, 2, 0x40, 7, 0x100, 14352, CompletionAction::signal(9, SignalOp::add(1))));
  auto t0 = clk::now();
  std::vector<std::thread> ts;
  for (uint32_t p = 0; p < producers; ++p)
    ts.emplace_back([&] {
      for (uint64_t i = 0; i < per; ++i) ring.submit(enc);
    });
  EncodedDescriptor out;
  uint64_t got = 0, sum = 0;
  while (got < per * producers) {
    if (ring.pop(out)) {
      sum += decode_descriptor(out).bytes;
      ++got;
    }
  }
  for (auto& t : ts) t.join();
  auto t1 = clk::now();
  std::printf("{\"cmd\":\"ringbench\",\"producers\":%u,\"descriptors\":%llu,\"wall_s\":%.6f,"
              "\"desc_per_s\":%.1f,\"checksum\":%llu}\n",
              producers, (unsigned long long)got, secs(t0, t1), got / secs(t0, t1),
              (unsigned long long)sum);
  return 0;
}

}  // namespace

// GIN1 frames encoded by the reference (wire.cpp) for a seeded set of
// fields: {"frames": [{"type", "src", "ctx", "seq", "id", "offset", "add",
// "operand", "body", "hex"}]}.  tests/golden/wire.json pins the B200 codec.
int cmd_wire(int argc, char** argv) {
  const uint64_t n = arg_u64(argc, argv, "--count", 64);
  std::mt19937_64 rng(arg_u64(argc, argv, "--seed", 7));
  auto hex = [](const std::vector<std::byte>& v) {
    static const char* d = "0123456789abcdef";
    std::string s;
    for (std::byte b : v) {
      const uint8_t x = std::to_integer<uint8_t>(b);
      s += d[x >> 4];
      s += d[x & 15];
    }
    return s;
  };
  std::printf("{\"frames\":[");
  for (uint64_t i = 0; i < n; ++i) {
    const uint32_t type = 1 + (uint32_t)(i % 4);
    const uint32_t src = (uint32_t)(rng() % 8);
    const uint16_t ctx = (uint16_t)(rng() % 5);
    const uint64_t seq = (i % 3 == 0) ? rng() : rng() % 1000;
    const uint32_t id = (uint32_t)(rng() % 300);
    const uint64_t off = (i % 5 == 0) ? rng() : rng() % 65536;
    const bool add = rng() & 1;
    const uint64_t operand = add ? ((i % 7 == 0) ? rng() : rng() % 100) : 1;
    const size_t blen = (type == 1 || type == 4) ? (size_t)(i % 9 == 0 ? 0 : rng() % 40) : 0;
    std::vector<std::byte> body(blen);
    for (auto& b : body) b = std::byte{(uint8_t)(rng() & 0xFF)};
    std::vector<std::byte> f;
    if (type == 1) f = encode_put_frame(src, ctx, seq, id, off, body);
    else if (type == 2) f = encode_signal_frame(src, ctx, seq, id, add ? SignalOp::add(operand) : SignalOp::inc());
    else if (type == 3) f = encode_ack_frame(src, ctx, seq);
    else f = encode_control_frame(src, body);
    std::printf("%s{\"type\":%u,\"src\":%u,\"ctx\":%u,\"seq\":%llu,\"id\":%u,\"offset\":%llu,\"add\":%d,"
                "\"operand\":%llu,\"body\":\"%s\",\"hex\":\"%s\"}",
                i ? "," : "", type, src, (unsigned)ctx, (unsigned long long)seq, id, (unsigned long long)off, add ? 1 : 0,
                (unsigned long long)operand, hex(body).c_str(), hex(f).c_str());
  }
  std::printf("]}\n");
  return 0;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ginsim_ref_driver moe-ll|moe-ht|pingpong|bw|ring|descriptors|ringbench|wire ...\n");
    return 2;
  }
  const std::string cmd = argv[1];
  try {
    if (cmd == "moe-ll") return cmd_moe_ll(argc, argv);
    if (cmd == "moe-ht") return cmd_moe_ht(argc, argv);
    if (cmd == "pingpong") return cmd_bench(argc, argv, true);
    if (cmd == "bw") return cmd_bench(argc, argv, false);
    if (cmd == "ring") return cmd_ring(argc, argv);
    if (cmd == "descriptors") return cmd_descriptors(argc, argv);
    if (cmd == "ringbench") return cmd_ringbench(argc, argv);
    if (cmd == "wire") return cmd_wire(argc, argv);
  } catch (const std::exception& e) {
    std::printf("{\"error\":\"%s\"}\n", e.what());
    return 1;
  }
  std::fprintf(stderr, "unknown command %s\n", cmd.c_str());
  return 2;
}
