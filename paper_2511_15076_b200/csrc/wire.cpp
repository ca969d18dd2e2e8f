// wire.cpp -- GIN1 frame codec (wire.h) and its C ABI (ginsim_cuda_wire_*).
// Byte layout: proj/core/include/ginsim/wire.hpp:12-21; the parser's checks
// follow proj/core/src/wire.cpp:89-141 (bad magic, unknown type, nonzero
// padding, unknown signal op).  Pinned against frames the reference itself
// encodes (tests/golden/wire.json, oracle/ref_driver.cpp `wire`).
#include "wire.h"

#include <cstring>
#include <string>

#include "runtime_internal.h"

namespace ginsim_b200 {
namespace wire {

static inline void put_le(uint8_t* p, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
static inline uint64_t get_le(const uint8_t* p, int n) {
  uint64_t v = 0;
  for (int i = n - 1; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

static size_t encode_header(uint8_t* p, Type type, uint32_t src, uint16_t ctx, uint64_t seq) {
  put_le(p, kMagic, 4);
  p[4] = (uint8_t)type;
  put_le(p + 5, src, 4);
  put_le(p + 9, ctx, 2);
  put_le(p + 11, 0, 2);
  put_le(p + 13, seq, 8);
  return kHeaderBytes;
}

size_t encode_put_prefix(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t seq, uint32_t dst_window,
                         uint64_t dst_offset, uint64_t len) {
  uint8_t* p = out + encode_header(out, kPut, src, ctx, seq);
  put_le(p, dst_window, 4);
  put_le(p + 4, dst_offset, 8);
  put_le(p + 12, len, 8);
  return kPutPrefixBytes;
}

size_t encode_signal(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t watermark, uint32_t signal_id, bool add,
                     uint64_t operand) {
  uint8_t* p = out + encode_header(out, kSignal, src, ctx, watermark);
  put_le(p, signal_id, 4);
  p[4] = add ? 1 : 0;
  p[5] = p[6] = p[7] = 0;
  put_le(p + 8, add ? operand : 1ull, 8);  // an inc always carries 1
  return kSignalBytes;
}

size_t encode_ack(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t seq) {
  return encode_header(out, kAck, src, ctx, seq);
}

size_t encode_control_prefix(uint8_t* out, uint32_t src, uint64_t len) {
  uint8_t* p = out + encode_header(out, kControl, src, 0, 0);
  put_le(p, len, 8);
  return kControlPrefixBytes;
}

void Parser::feed(const void* data, size_t n) {
  if (head_ && head_ * 2 >= buf_.size()) {  // drop the consumed prefix once it dominates
    buf_.erase(buf_.begin(), buf_.begin() + (ptrdiff_t)head_);
    head_ = 0;
  }
  const uint8_t* d = static_cast<const uint8_t*>(data);
  buf_.insert(buf_.end(), d, d + n);
}

uint64_t Parser::front_body_bytes() const {
  const size_t avail = buffered();
  const uint8_t* b = buf_.data() + head_;
  if (avail < kHeaderBytes || get_le(b, 4) != kMagic) return 0;  // (next() reports the garbage)
  if (b[4] == kPut && avail >= kPutPrefixBytes) return get_le(b + kHeaderBytes + 12, 8);
  if (b[4] == kControl && avail >= kControlPrefixBytes) return get_le(b + kHeaderBytes, 8);
  return 0;
}

bool Parser::next(Frame& f) {
  const size_t avail = buffered();
  const uint8_t* b = buf_.data() + head_;
  if (avail < kHeaderBytes) return false;
  if (get_le(b, 4) != kMagic) fail(GINSIM_E_MALFORMED_FRAME, "GIN1 frame: bad magic");
  const uint8_t type = b[4];
  if (type < kPut || type > kControl) fail(GINSIM_E_MALFORMED_FRAME, "GIN1 frame: unknown type " + std::to_string(type));
  if (get_le(b + 11, 2) != 0) fail(GINSIM_E_MALFORMED_FRAME, "GIN1 frame: header padding not zero");
  size_t need = kHeaderBytes;
  uint64_t body = 0;
  const uint8_t* q = b + kHeaderBytes;
  switch (type) {
    case kPut:
      if (avail < kPutPrefixBytes) return false;
      body = get_le(q + 12, 8);
      need = kPutPrefixBytes;
      break;
    case kSignal:
      if (avail < kSignalBytes) return false;
      if (q[4] > 1) fail(GINSIM_E_MALFORMED_FRAME, "GIN1 frame: unknown signal op " + std::to_string(q[4]));
      need = kSignalBytes;
      break;
    case kControl:
      if (avail < kControlPrefixBytes) return false;
      body = get_le(q, 8);
      need = kControlPrefixBytes;
      break;
    default:
      break;
  }
  if (avail - need < body) return false;
  f.type = type;
  f.src = (uint32_t)get_le(b + 5, 4);
  f.ctx = (uint16_t)get_le(b + 9, 2);
  f.seq = get_le(b + 13, 8);
  f.id = 0;
  f.offset = 0;
  f.add = false;
  f.operand = 0;
  if (type == kPut) {
    f.id = (uint32_t)get_le(q, 4);
    f.offset = get_le(q + 4, 8);
  } else if (type == kSignal) {
    f.id = (uint32_t)get_le(q, 4);
    f.add = q[4] == 1;
    f.operand = get_le(q + 8, 8);
  }
  f.body.assign(b + need, b + need + body);
  head_ += need + body;
  return true;
}

}  // namespace wire
}  // namespace ginsim_b200

using namespace ginsim_b200;

struct ginsim_cuda_wire_parser_s {
  wire::Parser p;
};

extern "C" {

int ginsim_cuda_wire_encode(const ginsim_cuda_wire_frame* f, const void* body, void* out, size_t cap, size_t* len) {
  GIN_API_BEGIN
  if (!f || !len) fail(GINSIM_E_USAGE, "wire_encode: null frame or length");
  uint8_t hdr[64];
  size_t h = 0;
  uint64_t nbody = 0;
  switch (f->type) {
    case wire::kPut:
      nbody = f->body_bytes;
      h = wire::encode_put_prefix(hdr, f->src_rank, f->ctx, f->seq_or_watermark, f->window_or_signal, f->dst_offset,
                                  nbody);
      break;
    case wire::kSignal:
      if (f->signal_add > 1) fail(GINSIM_E_USAGE, "wire_encode: signal op must be 0 (inc) or 1 (add)");
      h = wire::encode_signal(hdr, f->src_rank, f->ctx, f->seq_or_watermark, f->window_or_signal, f->signal_add == 1,
                              f->operand);
      break;
    case wire::kAck:
      h = wire::encode_ack(hdr, f->src_rank, f->ctx, f->seq_or_watermark);
      break;
    case wire::kControl:
      nbody = f->body_bytes;
      h = wire::encode_control_prefix(hdr, f->src_rank, nbody);
      break;
    default:
      fail(GINSIM_E_USAGE, "wire_encode: frame type must be 1..4");
  }
  *len = h + nbody;
  if (nbody && !body) fail(GINSIM_E_USAGE, "wire_encode: null body");
  if (!out || cap < *len) fail(GINSIM_E_USAGE, "wire_encode: output buffer holds " + std::to_string(cap) +
                                                   " bytes, the frame needs " + std::to_string(*len));
  std::memcpy(out, hdr, h);
  if (nbody) std::memcpy(static_cast<uint8_t*>(out) + h, body, nbody);
  GIN_API_END
}

int ginsim_cuda_wire_parser_create(ginsim_cuda_wire_parser_t* out) {
  GIN_API_BEGIN
  if (!out) fail(GINSIM_E_USAGE, "wire_parser_create: null output");
  *out = new ginsim_cuda_wire_parser_s;
  GIN_API_END
}

int ginsim_cuda_wire_parser_feed(ginsim_cuda_wire_parser_t p, const void* data, size_t n) {
  GIN_API_BEGIN
  if (!p || (n && !data)) fail(GINSIM_E_USAGE, "wire_parser_feed: null parser or data");
  p->p.feed(data, n);
  GIN_API_END
}

int ginsim_cuda_wire_parser_next(ginsim_cuda_wire_parser_t p, ginsim_cuda_wire_frame* f, void* body, size_t body_cap,
                                 int* ready) {
  GIN_API_BEGIN
  if (!p || !f || !ready) fail(GINSIM_E_USAGE, "wire_parser_next: null argument");
  *ready = 0;
  const uint64_t need = p->p.front_body_bytes();
  if (need > body_cap) {
    f->body_bytes = need;
    fail(GINSIM_E_USAGE, "wire_parser_next: body buffer holds " + std::to_string(body_cap) + " bytes, the frame carries " +
                             std::to_string(need));
  }
  wire::Frame fr;
  if (!p->p.next(fr)) return GINSIM_OK;
  std::memset(f, 0, sizeof(*f));
  f->type = fr.type;
  f->src_rank = fr.src;
  f->ctx = fr.ctx;
  f->seq_or_watermark = fr.seq;
  f->window_or_signal = fr.id;
  f->dst_offset = fr.offset;
  f->signal_add = fr.add ? 1u : 0u;
  f->operand = fr.operand;
  f->body_bytes = fr.body.size();
  if (!fr.body.empty()) std::memcpy(body, fr.body.data(), fr.body.size());
  *ready = 1;
  GIN_API_END
}

size_t ginsim_cuda_wire_parser_buffered(ginsim_cuda_wire_parser_t p) { return p ? p->p.buffered() : 0; }

int ginsim_cuda_wire_parser_destroy(ginsim_cuda_wire_parser_t p) {
  delete p;
  return GINSIM_OK;
}

}  // extern "C"
