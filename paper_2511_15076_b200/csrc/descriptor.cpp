// descriptor.cpp — the proxy path's 64-byte wire unit.
//
// Layout and invariants of proj/core/include/ginsim/descriptor.hpp:13-27 and
// proj/core/src/descriptor.cpp:32-60 (check), :148-166 (encode),
// :168-199 (decode).  Host and B200 are both little-endian, so the encoded
// image is the plain struct image the GPU producer stores with eight 64-bit
// words (gin_device.cuh, Gin::submit); this codec is what the host agent runs.
#include <cstring>
#include <string>

#include "runtime_internal.h"

namespace ginsim_b200 {

// Returns 0 when well-formed, else the reason index (see reasons below).
int descriptor_check(const ginsim_cuda_descriptor* d) {
  const bool is_inline = d->src_window == GIN_INLINE_WINDOW;
  switch (d->opcode) {
    case GIN_OP_PUT:
      if (is_inline) return 1;
      break;
    case GIN_OP_PUT_INLINE:
      if (!is_inline) return 2;
      if (d->bytes > 8) return 3;
      break;
    case GIN_OP_SIGNAL_ONLY:
      if (d->bytes != 0) return 4;
      if (!(d->flags & GIN_FLAG_HAS_SIGNAL)) return 5;
      if (!is_inline) return 6;
      if (d->dst_window || d->dst_offset || d->src_offset_or_value) return 7;
      break;
    default:
      return 8;
  }
  if (d->flags & ~(GIN_FLAG_HAS_SIGNAL | GIN_FLAG_SIGNAL_IS_ADD | GIN_FLAG_HAS_COUNTER)) return 9;
  if (d->flags & GIN_FLAG_HAS_SIGNAL) {
    if (!(d->flags & GIN_FLAG_SIGNAL_IS_ADD) && d->signal_operand != 1) return 10;
  } else {
    if (d->flags & GIN_FLAG_SIGNAL_IS_ADD) return 11;
    if (d->signal_id || d->signal_operand) return 12;
  }
  if (!(d->flags & GIN_FLAG_HAS_COUNTER) && d->counter_id) return 13;
  return 0;
}

static const char* reason(int why, uint8_t opcode) {
  static thread_local std::string s;
  switch (why) {
    case 1: return "PUT with inline src_window";
    case 2: return "PUT_INLINE requires inline src_window sentinel";
    case 3: return "inline payload over 8 bytes";
    case 4: return "SIGNAL_ONLY with nonzero bytes";
    case 5: return "SIGNAL_ONLY without HAS_SIGNAL";
    case 6: return "SIGNAL_ONLY carries no source window";
    case 7: return "SIGNAL_ONLY with nonzero transfer fields";
    case 8: s = "unknown opcode " + std::to_string(opcode); return s.c_str();
    case 9: return "reserved flag bits set";
    case 10: return "Inc signal with operand != 1";
    case 11: return "SIGNAL_IS_ADD without HAS_SIGNAL";
    case 12: return "signal fields set without HAS_SIGNAL";
    case 13: return "counter_id set without HAS_COUNTER";
    case 14: return "reserved word not zero";
    default: return "invalid descriptor";
  }
}

template <typename T>
static inline void put_le(uint8_t* b, int off, T v) {
  for (size_t i = 0; i < sizeof(T); ++i) b[off + i] = (uint8_t)((uint64_t)v >> (8 * i));
}
template <typename T>
static inline T get_le(const uint8_t* b, int off) {
  uint64_t v = 0;
  for (size_t i = 0; i < sizeof(T); ++i) v |= (uint64_t)b[off + i] << (8 * i);
  return (T)v;
}

void descriptor_encode(const ginsim_cuda_descriptor* d, uint8_t out[64]) {
  if (int why = descriptor_check(d)) fail(GINSIM_E_INVALID_DESCRIPTOR, reason(why, d->opcode));
  std::memset(out, 0, 64);
  put_le<uint8_t>(out, 0, d->opcode);
  put_le<uint8_t>(out, 1, d->flags);
  put_le<uint16_t>(out, 2, d->team);
  put_le<uint32_t>(out, 4, d->peer);
  put_le<uint32_t>(out, 8, d->dst_window);
  put_le<uint32_t>(out, 12, d->src_window);
  put_le<uint64_t>(out, 16, d->dst_offset);
  put_le<uint64_t>(out, 24, d->src_offset_or_value);
  put_le<uint64_t>(out, 32, d->bytes);
  put_le<uint32_t>(out, 40, d->signal_id);
  put_le<uint32_t>(out, 44, d->counter_id);
  put_le<uint64_t>(out, 48, d->signal_operand);
}

void descriptor_decode(const uint8_t in[64], ginsim_cuda_descriptor* d) {
  const uint8_t op = in[0];
  if (op < GIN_OP_PUT || op > GIN_OP_SIGNAL_ONLY) fail(GINSIM_E_MALFORMED_DESCRIPTOR, reason(8, op));
  d->opcode = op;
  d->flags = get_le<uint8_t>(in, 1);
  d->team = get_le<uint16_t>(in, 2);
  d->peer = get_le<uint32_t>(in, 4);
  d->dst_window = get_le<uint32_t>(in, 8);
  d->src_window = get_le<uint32_t>(in, 12);
  d->dst_offset = get_le<uint64_t>(in, 16);
  d->src_offset_or_value = get_le<uint64_t>(in, 24);
  d->bytes = get_le<uint64_t>(in, 32);
  d->signal_id = get_le<uint32_t>(in, 40);
  d->counter_id = get_le<uint32_t>(in, 44);
  d->signal_operand = get_le<uint64_t>(in, 48);
  if (get_le<uint64_t>(in, 56) != 0) fail(GINSIM_E_MALFORMED_DESCRIPTOR, reason(14, op));
  if (int why = descriptor_check(d)) fail(GINSIM_E_MALFORMED_DESCRIPTOR, reason(why, op));
}

}  // namespace ginsim_b200

// The codec's C ABI (include/ginsim_cuda.h), next to the codec so the host
// codecs build standalone (the sanitizer tests compile them from source).
using namespace ginsim_b200;

extern "C" {

int ginsim_cuda_descriptor_encode(const ginsim_cuda_descriptor* d, uint8_t out[64]) {
  GIN_API_BEGIN
  if (!d || !out) fail(GINSIM_E_USAGE, "descriptor_encode: null argument");
  descriptor_encode(d, out);
  GIN_API_END
}

int ginsim_cuda_descriptor_decode(const uint8_t in[64], ginsim_cuda_descriptor* d) {
  GIN_API_BEGIN
  if (!in || !d) fail(GINSIM_E_USAGE, "descriptor_decode: null argument");
  descriptor_decode(in, d);
  GIN_API_END
}

}  // extern "C"
