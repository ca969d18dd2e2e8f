// The host agent's two byte codecs under AddressSanitizer + UBSan (no GPU):
// the GIN1 frame codec (csrc/wire.cpp) and the 64-byte descriptor codec
// (csrc/descriptor.cpp) are compiled from their sources together with this
// harness (tests/test_cpp_api.py builds it with -fsanitize=address,undefined).
//   * frames: 8,000 random frames of every type round-trip through the
//     parser fed in random pieces; random garbage and single-byte corruptions
//     of valid streams either parse, wait for more bytes, or raise
//     MALFORMED_FRAME -- never read out of bounds or loop forever;
//   * descriptors: random field values round-trip when valid; random 64-byte
//     images decode or raise MALFORMED_DESCRIPTOR.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../paper_2511_15076_b200/csrc/runtime_internal.h"
#include "../../paper_2511_15076_b200/csrc/wire.h"

namespace ginsim_b200 {
// the two runtime symbols the codecs use (runtime.cu is not linked here)
[[noreturn]] void fail(int code, const std::string& msg) { throw GinError(code, msg); }
void set_last_error(const char*) {}
int descriptor_check(const ginsim_cuda_descriptor* d);
void descriptor_encode(const ginsim_cuda_descriptor* d, uint8_t out[64]);
void descriptor_decode(const uint8_t in[64], ginsim_cuda_descriptor* d);
}  // namespace ginsim_b200

using namespace ginsim_b200;

#define EXPECT(c)                                                           \
  do {                                                                      \
    if (!(c)) {                                                             \
      std::fprintf(stderr, "FAILED %s at %s:%d\n", #c, __FILE__, __LINE__); \
      std::exit(1);                                                         \
    }                                                                       \
  } while (0)

static std::vector<uint8_t> random_frame(std::mt19937_64& rng, wire::Frame& f) {
  f = wire::Frame{};
  f.type = (uint8_t)(1 + rng() % 4);
  f.src = (uint32_t)rng();
  f.ctx = f.type == wire::kControl ? 0 : (uint16_t)rng();
  f.seq = f.type == wire::kControl ? 0 : rng();
  std::vector<uint8_t> out(64);
  size_t h = 0;
  if (f.type == wire::kPut || f.type == wire::kControl) {
    f.body.resize(rng() % 3 == 0 ? 0 : rng() % 300);
    for (auto& b : f.body) b = (uint8_t)rng();
  }
  switch (f.type) {
    case wire::kPut:
      f.id = (uint32_t)rng();
      f.offset = rng();
      h = wire::encode_put_prefix(out.data(), f.src, f.ctx, f.seq, f.id, f.offset, f.body.size());
      break;
    case wire::kSignal:
      f.id = (uint32_t)rng();
      f.add = rng() & 1;
      f.operand = f.add ? rng() : 1;
      h = wire::encode_signal(out.data(), f.src, f.ctx, f.seq, f.id, f.add, f.operand);
      break;
    case wire::kAck:
      h = wire::encode_ack(out.data(), f.src, f.ctx, f.seq);
      break;
    default:
      h = wire::encode_control_prefix(out.data(), f.src, f.body.size());
  }
  out.resize(h);
  out.insert(out.end(), f.body.begin(), f.body.end());
  return out;
}

static void frames() {
  std::mt19937_64 rng(0x6171);
  std::vector<wire::Frame> want(8000);
  std::vector<uint8_t> stream;
  for (auto& f : want) {
    const auto b = random_frame(rng, f);
    stream.insert(stream.end(), b.begin(), b.end());
  }
  wire::Parser p;
  size_t i = 0, got = 0;
  wire::Frame f;
  while (i < stream.size()) {
    const size_t n = std::min<size_t>(stream.size() - i, 1 + rng() % 700);
    p.feed(stream.data() + i, n);
    i += n;
    while (p.next(f)) {
      const wire::Frame& w = want[got++];
      EXPECT(f.type == w.type && f.src == w.src && f.ctx == w.ctx && f.seq == w.seq && f.id == w.id);
      EXPECT(f.offset == w.offset && f.add == w.add && f.operand == w.operand && f.body == w.body);
    }
  }
  EXPECT(got == want.size() && p.buffered() == 0);
  // garbage: random bytes, and valid streams with one corrupted byte
  size_t malformed = 0, waiting = 0;
  for (int trial = 0; trial < 3000; ++trial) {
    std::vector<uint8_t> g;
    if (trial % 2) {
      g.resize(rng() % 200);
      for (auto& b : g) b = (uint8_t)rng();
      if (g.size() >= 4 && rng() % 2) {  // a valid magic in front makes the parser look further
        g[0] = 0x31, g[1] = 0x49, g[2] = 0x4E, g[3] = 0x47;
      }
    } else {
      wire::Frame tmp;
      g = random_frame(rng, tmp);
      g[rng() % g.size()] ^= (uint8_t)(1u << (rng() % 8));
    }
    wire::Parser q;
    q.feed(g.data(), g.size());
    try {
      for (int k = 0; k < 8 && q.next(f); ++k) {
      }
      ++waiting;
    } catch (const GinError& e) {
      EXPECT(e.code == GINSIM_E_MALFORMED_FRAME);
      ++malformed;
    }
  }
  EXPECT(malformed > 0 && waiting > 0);
  std::printf("frames ok (%zu frames, %zu malformed / %zu incomplete garbage streams)\n", got, malformed, waiting);
}

static void descriptors() {
  std::mt19937_64 rng(0xD15C);
  size_t valid = 0, invalid = 0, decoded = 0, rejected = 0;
  for (int t = 0; t < 60000; ++t) {
    ginsim_cuda_descriptor d{};
    d.opcode = (uint8_t)(1 + rng() % 3);
    d.flags = (uint8_t)(rng() % 8);
    d.team = (uint16_t)(rng() % 4);
    d.peer = (uint32_t)(rng() % 8);
    d.dst_window = rng() % 4 ? (uint32_t)(rng() % 64) : 0;
    d.src_window = rng() % 2 ? GIN_INLINE_WINDOW : (uint32_t)(rng() % 64);
    d.dst_offset = rng() % 3 ? rng() % 100000 : 0;
    d.src_offset_or_value = rng() % 3 ? rng() : 0;
    d.bytes = rng() % 3 ? rng() % 16 : rng() % 100000;
    d.signal_id = (d.flags & GIN_FLAG_HAS_SIGNAL) ? (uint32_t)(rng() % 256) : 0;
    d.counter_id = (d.flags & GIN_FLAG_HAS_COUNTER) ? (uint32_t)(rng() % 256) : 0;
    d.signal_operand = (d.flags & GIN_FLAG_HAS_SIGNAL) ? ((d.flags & GIN_FLAG_SIGNAL_IS_ADD) ? rng() % 100 : 1) : 0;
    if (descriptor_check(&d) != 0) {
      ++invalid;
      continue;
    }
    ++valid;
    uint8_t img[64];
    descriptor_encode(&d, img);
    ginsim_cuda_descriptor e{};
    descriptor_decode(img, &e);
    EXPECT(std::memcmp(&d, &e, sizeof(d)) == 0);
  }
  for (int t = 0; t < 60000; ++t) {
    uint8_t img[64];
    for (auto& b : img) b = (uint8_t)rng();
    if (t % 3 == 0) std::memset(img + 16, 0, 48);  // mostly-zero images reach the field checks
    ginsim_cuda_descriptor e{};
    try {
      descriptor_decode(img, &e);
      ++decoded;
    } catch (const GinError& err) {
      EXPECT(err.code == GINSIM_E_MALFORMED_DESCRIPTOR || err.code == GINSIM_E_INVALID_DESCRIPTOR);
      ++rejected;
    }
  }
  EXPECT(valid > 1000 && invalid > 1000 && rejected > 0);
  std::printf("descriptors ok (%zu valid round trips, %zu invalid; %zu random images decoded, %zu rejected)\n", valid,
              invalid, decoded, rejected);
}

int main() {
  std::setvbuf(stdout, nullptr, _IONBF, 0);
  frames();
  descriptors();
  return 0;
}
