// ginsim/descriptor.hpp -- the reference's 64-byte descriptor interface
// (proj/core/include/ginsim/descriptor.hpp:13-94) over this library's codec
// (ginsim_cuda_descriptor_encode / _decode, csrc/descriptor.cpp: the same
// bytes the GPU producers write into the Proxy rings, gin_device.cuh).
// Reference sources that build, validate, encode or decode descriptors
// compile against it unchanged; errors are the reference's exception types
// (InvalidDescriptor from validate / encode, MalformedDescriptor from decode).
#pragma once

#include <array>
#include <cstddef>
#include <cstdint>
#include <span>

#include "ginsim/runtime.hpp"

namespace ginsim {

inline constexpr size_t kDescriptorBytes = 64;
using EncodedDescriptor = std::array<std::byte, kDescriptorBytes>;

namespace descriptor_flags {
inline constexpr uint8_t kHasSignal = 1u << 0;
inline constexpr uint8_t kSignalIsAdd = 1u << 1;
inline constexpr uint8_t kHasCounter = 1u << 2;
inline constexpr uint8_t kAll = kHasSignal | kSignalIsAdd | kHasCounter;
}  // namespace descriptor_flags

// descriptor.hpp:48-76: one operation and its completion actions, decoded
struct Descriptor {
  Opcode opcode = Opcode::Put;
  uint8_t flags = 0;
  TeamId team = 0;
  RankId peer = 0;
  WindowId dst_window = 0;
  WindowId src_window = 0;
  uint64_t dst_offset = 0;
  uint64_t src_offset_or_value = 0;
  uint64_t bytes = 0;
  SignalId signal_id = 0;
  CounterId counter_id = 0;
  uint64_t signal_operand = 0;

  bool has_signal() const { return (flags & descriptor_flags::kHasSignal) != 0; }
  bool signal_is_add() const { return (flags & descriptor_flags::kSignalIsAdd) != 0; }
  bool has_counter() const { return (flags & descriptor_flags::kHasCounter) != 0; }
  bool is_inline() const { return src_window == kInlineWindow; }
  SignalOp signal_op() const { return signal_is_add() ? SignalOp::add(signal_operand) : SignalOp::inc(); }
  CompletionAction action() const {
    CompletionAction a;
    if (has_signal()) a.remote_signal = CompletionAction::RemoteSignal{signal_id, signal_op()};
    if (has_counter()) a.local_counter = counter_id;
    return a;
  }
  friend bool operator==(const Descriptor&, const Descriptor&) = default;
};

namespace detail {
inline ginsim_cuda_descriptor to_c(const Descriptor& d) {
  ginsim_cuda_descriptor c{};
  c.opcode = static_cast<uint8_t>(d.opcode);
  c.flags = d.flags;
  c.team = d.team;
  c.peer = d.peer;
  c.dst_window = d.dst_window;
  c.src_window = d.src_window;
  c.dst_offset = d.dst_offset;
  c.src_offset_or_value = d.src_offset_or_value;
  c.bytes = d.bytes;
  c.signal_id = d.signal_id;
  c.counter_id = d.counter_id;
  c.signal_operand = d.signal_operand;
  return c;
}
inline Descriptor from_c(const ginsim_cuda_descriptor& c) {
  Descriptor d;
  d.opcode = static_cast<Opcode>(c.opcode);
  d.flags = c.flags;
  d.team = c.team;
  d.peer = c.peer;
  d.dst_window = c.dst_window;
  d.src_window = c.src_window;
  d.dst_offset = c.dst_offset;
  d.src_offset_or_value = c.src_offset_or_value;
  d.bytes = c.bytes;
  d.signal_id = c.signal_id;
  d.counter_id = c.counter_id;
  d.signal_operand = c.signal_operand;
  return d;
}
// the action's fields in normalized form (unused fields stay zero, Inc carries operand 1)
inline void set_action(Descriptor& d, const CompletionAction& a) {
  if (a.remote_signal) {
    d.flags |= descriptor_flags::kHasSignal;
    d.signal_id = a.remote_signal->id;
    const bool add = a.remote_signal->op.kind == SignalKind::Add;
    if (add) d.flags |= descriptor_flags::kSignalIsAdd;
    d.signal_operand = add ? a.remote_signal->op.operand : 1;
  }
  if (a.local_counter) {
    d.flags |= descriptor_flags::kHasCounter;
    d.counter_id = *a.local_counter;
  }
}
}  // namespace detail

// Builders (descriptor.hpp:78-82): normalized descriptors, so encode/decode
// round trips compare equal.
inline Descriptor make_put_descriptor(TeamId team, RankId peer, WindowId dst_window, uint64_t dst_offset,
                                      WindowId src_window, uint64_t src_offset, uint64_t bytes,
                                      const CompletionAction& action) {
  Descriptor d;
  d.opcode = Opcode::Put;
  d.team = team;
  d.peer = peer;
  d.dst_window = dst_window;
  d.dst_offset = dst_offset;
  d.src_window = src_window;
  d.src_offset_or_value = src_offset;
  d.bytes = bytes;
  detail::set_action(d, action);
  return d;
}

inline Descriptor make_put_inline_descriptor(TeamId team, RankId peer, WindowId dst_window, uint64_t dst_offset,
                                             uint64_t value, uint64_t bytes, const CompletionAction& action) {
  Descriptor d = make_put_descriptor(team, peer, dst_window, dst_offset, kInlineWindow, value, bytes, action);
  d.opcode = Opcode::PutInline;
  return d;
}

// The op's own signal wins over a signal in `action` (only its counter is kept).
inline Descriptor make_signal_descriptor(TeamId team, RankId peer, SignalId id, SignalOp op,
                                         const CompletionAction& action = {}) {
  Descriptor d;
  d.opcode = Opcode::SignalOnly;
  d.team = team;
  d.peer = peer;
  d.src_window = kInlineWindow;
  CompletionAction a = action;
  a.remote_signal = CompletionAction::RemoteSignal{id, op};
  detail::set_action(d, a);
  if (op.kind != SignalKind::Add) d.flags &= static_cast<uint8_t>(~descriptor_flags::kSignalIsAdd);
  return d;
}

// Deterministic 64-byte encoding (descriptor.hpp:88-89); InvalidDescriptor when
// d violates an invariant.
inline EncodedDescriptor encode_descriptor(const Descriptor& d) {
  const ginsim_cuda_descriptor c = detail::to_c(d);
  EncodedDescriptor out{};
  check(ginsim_cuda_descriptor_encode(&c, reinterpret_cast<uint8_t*>(out.data())));
  return out;
}

// descriptor.hpp:84-86: InvalidDescriptor when d violates an invariant.
inline void validate_descriptor(const Descriptor& d) { (void)encode_descriptor(d); }

// descriptor.hpp:91-93: MalformedDescriptor on an unknown opcode, reserved
// bits or words, fields inconsistent with the flags, or a wrong length.
inline Descriptor decode_descriptor(std::span<const std::byte> buf) {
  if (buf.size() != kDescriptorBytes)
    throw MalformedDescriptor("descriptor must be 64 bytes, got " + std::to_string(buf.size()));
  ginsim_cuda_descriptor c{};
  check(ginsim_cuda_descriptor_decode(reinterpret_cast<const uint8_t*>(buf.data()), &c));
  return detail::from_c(c);
}
inline Descriptor decode_descriptor(const EncodedDescriptor& buf) {
  return decode_descriptor(std::span<const std::byte>(buf.data(), buf.size()));
}

}  // namespace ginsim
