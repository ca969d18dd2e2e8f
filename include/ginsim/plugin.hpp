// ginsim/plugin.hpp — the reference's backend boundary (proj/core/include/
// ginsim/plugin.hpp:17-144, direct_backend.hpp:17-63) as a header-only layer
// over the C ABI's plugin entry points (include/ginsim_cuda.h), so code
// written against FabricPlugin / DirectContext drives the B200 backends:
//   proxy semantics: reg_mr, iput, iput_signal, test, retire -- the op runs on
//     the comm's host agent (copy engine + stream-memop signal/counter);
//   direct semantics: create_context -> DirectContext::post / poll /
//     outstanding -- the op runs as NVLink stores on the context's stream.
// The plugin's semantics are the comm's backend (as the reference's runtime
// constructs it, runtime.cpp:197-213).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <vector>

#include "runtime.hpp"

namespace ginsim {

struct MrHandle {
  WindowId window = 0;
  friend bool operator==(const MrHandle&, const MrHandle&) = default;
};

using RequestId = uint64_t;

struct PutSource {
  MrHandle mr;
  uint64_t offset = 0;
  std::optional<uint64_t> inline_value;
  static PutSource window(MrHandle mr, uint64_t offset) { return {mr, offset, std::nullopt}; }
  static PutSource inline_bytes(uint64_t value) { return {{}, 0, value}; }
  ginsim_cuda_put_source to_c() const {
    ginsim_cuda_put_source s{};
    s.is_inline = inline_value.has_value();
    s.mr = mr.window;
    s.offset = offset;
    s.inline_value = inline_value.value_or(0);
    return s;
  }
};

// plugin.hpp:48-55 (the posting trace; the issuer is a hash of the thread id)
struct PluginCall {
  char op = '?';  // 'p' iput, 's' iput_signal
  ContextId ctx = 0;
  RankId peer = 0;
  uint64_t bytes = 0;
  uint64_t issuer = 0;
};

// direct_backend.hpp:17-27
struct ResolvedOp {
  Opcode opcode = Opcode::Put;
  RankId peer = 0;
  WindowId dst_window = 0;
  uint64_t dst_offset = 0;
  WindowId src_window = kInlineWindow;
  uint64_t src_offset_or_value = 0;
  uint64_t bytes = 0;
  CompletionAction action;
};

inline CompletionAction action_from_c(const ginsim_cuda_action& a) {
  CompletionAction r;
  if (a.signal_id >= 0)
    r.remote_signal = CompletionAction::RemoteSignal{(SignalId)a.signal_id,
                                                     a.signal_add ? SignalOp::add(a.operand) : SignalOp::inc()};
  if (a.counter_id >= 0) r.local_counter = (CounterId)a.counter_id;
  return r;
}

class DirectContext {
 public:
  explicit DirectContext(ginsim_cuda_direct_ctx_t h, ContextId index) : h_(h), index_(index) {}
  ContextId index() const { return index_; }
  void post(const ResolvedOp& op) {
    ginsim_cuda_resolved_op c{};
    c.opcode = static_cast<uint32_t>(op.opcode);
    c.peer = op.peer;
    c.dst_window = op.dst_window;
    c.src_window = op.src_window;
    c.dst_offset = op.dst_offset;
    c.src_offset_or_value = op.src_offset_or_value;
    c.bytes = op.bytes;
    c.action = op.action.to_c();
    check(ginsim_cuda_direct_post(h_, &c));
  }
  size_t poll() {
    uint64_t n = 0;
    check(ginsim_cuda_direct_poll(h_, &n));
    return static_cast<size_t>(n);
  }
  uint64_t outstanding() const {
    uint64_t n = 0;
    check(ginsim_cuda_direct_outstanding(h_, &n));
    return n;
  }

 private:
  ginsim_cuda_direct_ctx_t h_;
  ContextId index_;
};

class FabricPlugin {
 public:
  FabricPlugin(DevComm& comm, BackendKind semantics) : semantics_(semantics) {
    check(ginsim_cuda_plugin_create(comm.handle(), semantics == BackendKind::Proxy ? 1u : 0u, &h_));
    contexts_.resize(comm.config().n_contexts);
  }
  ~FabricPlugin() { ginsim_cuda_plugin_destroy(h_); }
  FabricPlugin(const FabricPlugin&) = delete;
  FabricPlugin& operator=(const FabricPlugin&) = delete;

  BackendKind semantics() const { return semantics_; }

  MrHandle reg_mr(WindowId id) {
    uint32_t mr = 0;
    check(ginsim_cuda_plugin_reg_mr(h_, id, &mr));
    return MrHandle{mr};
  }
  bool is_registered(WindowId id) const {
    int r = 0;
    check(ginsim_cuda_plugin_is_registered(h_, id, &r));
    return r != 0;
  }

  RequestId iput(const PutSource& src, MrHandle dst, uint64_t dst_offset, uint64_t bytes, RankId peer, ContextId ctx,
                 const CompletionAction& action) {
    const ginsim_cuda_put_source s = src.to_c();
    const ginsim_cuda_action a = action.to_c();
    RequestId id = 0;
    check(ginsim_cuda_plugin_iput(h_, &s, dst.window, dst_offset, bytes, peer, ctx, &a, &id));
    return id;
  }
  RequestId iput_signal(const PutSource& src, MrHandle dst, uint64_t dst_offset, uint64_t bytes, RankId peer,
                        ContextId ctx, SignalId signal, SignalOp op, const CompletionAction& action) {
    const ginsim_cuda_put_source s = src.to_c();
    const ginsim_cuda_action a = action.to_c();
    RequestId id = 0;
    check(ginsim_cuda_plugin_iput_signal(h_, &s, dst.window, dst_offset, bytes, peer, ctx, signal,
                                         op.kind == SignalKind::Add, op.operand, &a, &id));
    return id;
  }
  bool test(RequestId id) const {
    int done = 0;
    check(ginsim_cuda_plugin_test(h_, id, &done));
    return done != 0;
  }
  CompletionAction retire(RequestId id) {
    ginsim_cuda_action a{};
    check(ginsim_cuda_plugin_retire(h_, id, &a));
    return action_from_c(a);
  }
  size_t outstanding_requests() const {
    uint64_t n = 0;
    check(ginsim_cuda_plugin_outstanding(h_, &n));
    return static_cast<size_t>(n);
  }

  void set_call_log_enabled(bool on) { check(ginsim_cuda_plugin_set_call_log(h_, on ? 1 : 0)); }
  std::vector<PluginCall> call_log() const {
    uint32_t n = 0;
    check(ginsim_cuda_plugin_call_log(h_, nullptr, 0, &n));
    std::vector<ginsim_cuda_plugin_call> raw(n);
    check(ginsim_cuda_plugin_call_log(h_, raw.data(), n, &n));
    std::vector<PluginCall> out;
    for (uint32_t i = 0; i < std::min<uint32_t>(n, (uint32_t)raw.size()); ++i)
      out.push_back(PluginCall{raw[i].op, (ContextId)raw[i].ctx, raw[i].peer, raw[i].bytes, raw[i].issuer});
    return out;
  }

  DirectContext& create_context(ContextId ctx) {
    ginsim_cuda_direct_ctx_t d = nullptr;
    check(ginsim_cuda_plugin_create_context(h_, ctx, &d));
    if (!contexts_[ctx]) contexts_[ctx] = std::make_unique<DirectContext>(d, ctx);
    return *contexts_[ctx];
  }

 private:
  ginsim_cuda_plugin_t h_ = nullptr;
  BackendKind semantics_;
  std::vector<std::unique_ptr<DirectContext>> contexts_;
};

}  // namespace ginsim
