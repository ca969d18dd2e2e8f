// ginsim/wire.hpp -- the reference's GIN1 framing interface
// (proj/core/include/ginsim/wire.hpp:12-67) over this library's codec
// (ginsim_cuda_wire_*, csrc/wire.cpp: the frames the Proxy backend's socket
// transport exchanges between the ranks' agents, csrc/net.cu).  Reference
// sources that encode or parse frames compile against it unchanged; a bad
// magic, type, padding or signal op is the reference's MalformedFrame.
#pragma once

#include <cstddef>
#include <cstdint>
#include <optional>
#include <span>
#include <utility>
#include <vector>

#include "ginsim/runtime.hpp"

namespace ginsim {

inline constexpr uint32_t kFrameMagic = GINSIM_WIRE_MAGIC;  // "GIN1"
inline constexpr size_t kFrameHeaderBytes = GINSIM_WIRE_HEADER_BYTES;

enum class FrameType : uint8_t {
  Put = GINSIM_WIRE_PUT,
  Signal = GINSIM_WIRE_SIGNAL,
  Ack = GINSIM_WIRE_ACK,
  Control = GINSIM_WIRE_CONTROL,
};

// wire.hpp:33-45: one decoded frame; src_rank is the frame's sender
struct ParsedFrame {
  FrameType type = FrameType::Control;
  RankId src_rank = 0;
  ContextId ctx = 0;
  uint64_t seq_or_watermark = 0;
  WindowId dst_window = 0;
  uint64_t dst_offset = 0;
  std::vector<std::byte> payload;  // Put
  SignalId signal_id = 0;
  SignalOp op;
  std::vector<std::byte> blob;  // Control
};

namespace detail {
inline std::vector<std::byte> encode_frame(const ginsim_cuda_wire_frame& f, std::span<const std::byte> body) {
  size_t len = 0;
  // the first call sizes the frame (USAGE with *len set), the second writes it
  (void)ginsim_cuda_wire_encode(&f, body.data(), nullptr, 0, &len);
  std::vector<std::byte> out(len);
  check(ginsim_cuda_wire_encode(&f, body.data(), out.data(), out.size(), &len));
  out.resize(len);
  return out;
}
inline ginsim_cuda_wire_frame frame_of(uint32_t type, RankId src, ContextId ctx, uint64_t seq) {
  ginsim_cuda_wire_frame f{};
  f.type = type;
  f.src_rank = src;
  f.ctx = ctx;
  f.seq_or_watermark = seq;
  f.operand = 1;
  return f;
}
}  // namespace detail

// wire.hpp:47-53
inline std::vector<std::byte> encode_put_frame(RankId src, ContextId ctx, uint64_t seq, WindowId dst_window,
                                               uint64_t dst_offset, std::span<const std::byte> payload) {
  ginsim_cuda_wire_frame f = detail::frame_of(GINSIM_WIRE_PUT, src, ctx, seq);
  f.window_or_signal = dst_window;
  f.dst_offset = dst_offset;
  f.body_bytes = payload.size();
  return detail::encode_frame(f, payload);
}
inline std::vector<std::byte> encode_signal_frame(RankId src, ContextId ctx, uint64_t watermark, SignalId id,
                                                  SignalOp op) {
  ginsim_cuda_wire_frame f = detail::frame_of(GINSIM_WIRE_SIGNAL, src, ctx, watermark);
  f.window_or_signal = id;
  f.signal_add = op.kind == SignalKind::Add ? 1u : 0u;
  f.operand = op.kind == SignalKind::Add ? op.operand : 1;
  return detail::encode_frame(f, {});
}
inline std::vector<std::byte> encode_ack_frame(RankId src, ContextId ctx, uint64_t seq) {
  return detail::encode_frame(detail::frame_of(GINSIM_WIRE_ACK, src, ctx, seq), {});
}
inline std::vector<std::byte> encode_control_frame(RankId src, std::span<const std::byte> blob) {
  ginsim_cuda_wire_frame f = detail::frame_of(GINSIM_WIRE_CONTROL, src, 0, 0);
  f.body_bytes = blob.size();
  return detail::encode_frame(f, blob);
}

// wire.hpp:55-66: incremental decoder over a byte stream; frames may arrive
// split or coalesced.  next() is empty until a whole frame is buffered.
class FrameParser {
 public:
  FrameParser() { check(ginsim_cuda_wire_parser_create(&p_)); }
  ~FrameParser() {
    if (p_) ginsim_cuda_wire_parser_destroy(p_);
  }
  FrameParser(FrameParser&& o) noexcept : p_(o.p_) { o.p_ = nullptr; }
  FrameParser& operator=(FrameParser&& o) noexcept {
    std::swap(p_, o.p_);
    return *this;
  }
  FrameParser(const FrameParser&) = delete;
  FrameParser& operator=(const FrameParser&) = delete;

  void feed(std::span<const std::byte> data) { check(ginsim_cuda_wire_parser_feed(p_, data.data(), data.size())); }

  std::optional<ParsedFrame> next() {
    ginsim_cuda_wire_frame f{};
    int ready = 0;
    std::vector<std::byte> body(body_hint_);
    int rc = ginsim_cuda_wire_parser_next(p_, &f, body.data(), body.size(), &ready);
    if (rc == GINSIM_E_USAGE && f.body_bytes > body.size()) {  // body larger than the buffer: nothing consumed
      body.resize(f.body_bytes);
      rc = ginsim_cuda_wire_parser_next(p_, &f, body.data(), body.size(), &ready);
    }
    check(rc);
    if (!ready) return std::nullopt;
    body.resize(f.body_bytes);
    ParsedFrame out;
    out.type = static_cast<FrameType>(f.type);
    out.src_rank = f.src_rank;
    out.ctx = f.ctx;
    out.seq_or_watermark = f.seq_or_watermark;
    if (out.type == FrameType::Put) {
      out.dst_window = f.window_or_signal;
      out.dst_offset = f.dst_offset;
      out.payload = std::move(body);
    } else if (out.type == FrameType::Signal) {
      out.signal_id = f.window_or_signal;
      out.op = f.signal_add ? SignalOp::add(f.operand) : SignalOp::inc();
    } else if (out.type == FrameType::Control) {
      out.blob = std::move(body);
    }
    return out;
  }

  size_t buffered() const { return ginsim_cuda_wire_parser_buffered(p_); }

 private:
  static constexpr size_t body_hint_ = 4096;
  ginsim_cuda_wire_parser_t p_ = nullptr;
};

}  // namespace ginsim
