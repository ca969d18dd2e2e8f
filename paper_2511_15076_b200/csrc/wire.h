// wire.h -- the GIN1 frame codec used by the Proxy backend's socket transport
// (the reference's framing, proj/core/include/ginsim/wire.hpp:12-67).
//
// One frame per message, little-endian:
//   header (21 B): magic u32 0x474E4931 "GIN1" | type u8 | src u32 | ctx u16 |
//                  pad u16 = 0 | seq_or_watermark u64
//   Put     (+20 B): dst_window u32 | dst_offset u64 | len u64 | payload[len]
//   Signal  (+16 B): signal_id u32 | op u8 (0 inc, 1 add) | pad 3 | operand u64 (1 for inc)
//   Ack     (+0 B)
//   Control (+8 B):  len u64 | blob[len]
// The encoders write into caller memory (a frame header goes in front of a
// payload that already sits in a pinned staging buffer, so the sender never
// copies the payload); the parser accepts a byte stream split or coalesced
// at any point and raises MALFORMED_FRAME on a bad magic, type, padding or
// signal op.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

namespace ginsim_b200 {
namespace wire {

constexpr uint32_t kMagic = 0x474E4931u;
constexpr size_t kHeaderBytes = 21;
constexpr size_t kPutPrefixBytes = kHeaderBytes + 20;
constexpr size_t kSignalBytes = kHeaderBytes + 16;
constexpr size_t kAckBytes = kHeaderBytes;
constexpr size_t kControlPrefixBytes = kHeaderBytes + 8;
enum Type : uint8_t { kPut = 1, kSignal = 2, kAck = 3, kControl = 4 };

struct Frame {
  uint8_t type = 0;
  uint32_t src = 0;
  uint16_t ctx = 0;
  uint64_t seq = 0;       // put: sequence number; signal: watermark; ack: acknowledged sequence
  uint32_t id = 0;        // put: destination window; signal: signal id
  uint64_t offset = 0;    // put: destination offset
  bool add = false;       // signal: SignalAdd (else SignalInc)
  uint64_t operand = 0;   // signal: amount (1 for inc)
  std::vector<uint8_t> body;  // put payload / control blob
};

// Each returns the bytes written; the put / control prefixes are followed by
// the len body bytes on the wire.
size_t encode_put_prefix(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t seq, uint32_t dst_window,
                         uint64_t dst_offset, uint64_t len);
size_t encode_signal(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t watermark, uint32_t signal_id, bool add,
                     uint64_t operand);
size_t encode_ack(uint8_t* out, uint32_t src, uint16_t ctx, uint64_t seq);
size_t encode_control_prefix(uint8_t* out, uint32_t src, uint64_t len);

class Parser {
 public:
  void feed(const void* data, size_t n);
  // true and f filled when a whole frame was buffered; false when more bytes
  // are needed.  Throws (fail, GINSIM_E_MALFORMED_FRAME) on garbage.
  bool next(Frame& f);
  // The body size of the frame at the front once its fixed part is buffered
  // (put / control), else 0; lets a caller size its buffer before next().
  uint64_t front_body_bytes() const;
  size_t buffered() const { return buf_.size() - head_; }

 private:
  std::vector<uint8_t> buf_;
  size_t head_ = 0;
};

}  // namespace wire
}  // namespace ginsim_b200
