// plugin.cu — the FabricPlugin boundary (proj/core/include/ginsim/plugin.hpp:
// 64-144, proj/core/src/plugin.cpp:18-172, direct_backend.cpp:7-57) over the
// B200 runtime, so a host runtime written against the reference's plugin
// interface can drive the GPU backends.
//
//   Proxy semantics (the host data path a progress agent drives):
//     reg_mr / iput / iput_signal / test / retire / outstanding_requests.
//     iput hands the op to the comm's host agent, which moves it on the copy
//     engines (cudaMemcpyAsync into the peer's VMM mapping) and applies the
//     signal / counter with stream memops after the copy (proxy.cu).  The
//     RequestId names (context, host ticket); test() is true once the agent's
//     completion event for that ticket has fired.  Requests are tracked until
//     retire() returns their CompletionAction, exactly once.
//   Direct semantics (submitters post inline):
//     create_context -> DirectContext; post(ResolvedOp) launches the one-warp
//     device op on the context's stream (NVLink stores + red.release.sys
//     signal + counter bump on the device), poll() retires the ops the stream
//     has executed, outstanding() counts the rest.
//
// The plugin's semantics must match the comm's backend (the reference creates
// the plugin from the comm's BackendKind, runtime.cpp:197-213); calls of the
// other semantics raise BackendMismatch as in plugin.cpp:38-43.
#include <algorithm>
#include <deque>
#include <functional>
#include <map>
#include <set>
#include <thread>

#include "runtime_internal.h"

namespace ginsim_b200 {

struct PluginRequest {
  uint32_t ctx = 0;
  uint64_t ticket = 0;
  ginsim_cuda_action action{};
  bool done = false;
};

}  // namespace ginsim_b200

struct ginsim_cuda_direct_ctx_s;

struct ginsim_cuda_plugin_s {
  ginsim_cuda_comm_t comm = nullptr;
  uint32_t semantics = 0;
  std::mutex mu;
  bool log_calls = false;                          // plugin.cpp:174-188 (posting trace for tests)
  std::vector<ginsim_cuda_plugin_call> calls;
  std::set<uint32_t> mrs;
  std::map<uint64_t, ginsim_b200::PluginRequest> requests;
  uint64_t next_request = 1;
  std::vector<ginsim_cuda_direct_ctx_s*> contexts;
};

struct ginsim_cuda_direct_ctx_s {
  ginsim_cuda_plugin_s* plugin = nullptr;
  uint32_t index = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::deque<cudaEvent_t> in_flight;  // one event per posted op, in post order
  std::vector<cudaEvent_t> spare;
};

using namespace ginsim_b200;

namespace {

// record_call (plugin.cpp:185-188): 'p' iput, 's' iput_signal / signalling post
void record_call(ginsim_cuda_plugin_t p, char op, uint32_t ctx, uint32_t peer, uint64_t bytes) {
  std::lock_guard<std::mutex> lk(p->mu);
  if (!p->log_calls) return;
  ginsim_cuda_plugin_call c{};
  c.op = op;
  c.ctx = ctx;
  c.peer = peer;
  c.bytes = bytes;
  c.issuer = (uint64_t)std::hash<std::thread::id>{}(std::this_thread::get_id());
  p->calls.push_back(c);
}

void require_semantics(ginsim_cuda_plugin_t p, uint32_t k, const char* op) {
  if (p->semantics != k)
    fail(GINSIM_E_BACKEND_MISMATCH, std::string(op) + " called on a " + (p->semantics ? "proxy" : "direct") +
                                        "-semantics backend");
}

void require_mr(ginsim_cuda_plugin_t p, uint32_t w, const char* role) {
  if (!p->mrs.count(w))
    fail(GINSIM_E_UNKNOWN_WINDOW, std::string(role) + " window " + std::to_string(w) + " not registered with backend");
}

uint64_t track(ginsim_cuda_plugin_t p, uint32_t ctx, uint64_t ticket, const ginsim_cuda_action* a) {
  PluginRequest r;
  r.ctx = ctx;
  r.ticket = ticket;
  if (a) r.action = *a;
  else r.action = ginsim_cuda_action{-1, 0, 1, -1, 0};
  const uint64_t id = p->next_request++;
  p->requests.emplace(id, r);
  return id;
}

uint64_t iput_common(ginsim_cuda_plugin_t p, const ginsim_cuda_put_source* src, uint32_t dst_mr, uint64_t dst_offset,
                     uint64_t bytes, uint32_t peer, uint32_t ctx, const ginsim_cuda_action* sig_action,
                     const ginsim_cuda_action* completion) {
  Comm* c = &p->comm->impl;
  std::lock_guard<std::mutex> lk(p->mu);
  if (!src) fail(GINSIM_E_USAGE, "iput: null source");
  // the op's action: the remote signal (iput_signal only) + the local counter
  ginsim_cuda_action a{-1, 0, 1, -1, 0};
  if (sig_action) a = *sig_action;
  if (completion) a.counter_id = completion->counter_id;
  uint64_t ticket;
  if (src->is_inline) {
    if (bytes > 8) fail(GINSIM_E_INVALID_DESCRIPTOR, "inline payload over 8 bytes");
    require_mr(p, dst_mr, "destination");
    ticket = bytes ? host_op(c, ctx, GIN_OP_PUT_INLINE, peer, dst_mr, dst_offset, GIN_INLINE_WINDOW,
                             src->inline_value, bytes, &a, nullptr)
                   : host_op(c, ctx, GIN_OP_PUT, peer, dst_mr, dst_offset, dst_mr, 0, 0, &a, nullptr);
  } else {
    if (bytes) {
      require_mr(p, src->mr, "source");
      require_mr(p, dst_mr, "destination");
    }
    ticket = host_op(c, ctx, GIN_OP_PUT, peer, dst_mr, dst_offset, src->mr, src->offset, bytes, &a, nullptr);
  }
  ginsim_cuda_action tracked = completion ? *completion : ginsim_cuda_action{-1, 0, 1, -1, 0};
  return track(p, ctx, ticket, &tracked);
}

void retire_done(ginsim_cuda_direct_ctx_t d, size_t* n) {
  while (!d->in_flight.empty()) {
    const cudaError_t q = cudaEventQuery(d->in_flight.front());
    if (q == cudaErrorNotReady) break;
    GIN_CUDA(q);
    d->spare.push_back(d->in_flight.front());
    d->in_flight.pop_front();
    if (n) ++*n;
  }
}

}  // namespace

extern "C" {

int ginsim_cuda_plugin_create(ginsim_cuda_comm_t comm, uint32_t semantics, ginsim_cuda_plugin_t* out) {
  GIN_API_BEGIN
  if (!comm || !out) fail(GINSIM_E_USAGE, "plugin_create: null argument");
  if (semantics > 1) fail(GINSIM_E_USAGE, "semantics must be 0 (direct) or 1 (proxy)");
  if (semantics != comm->impl.cfg.backend)
    fail(GINSIM_E_BACKEND_MISMATCH, "plugin semantics must match the comm's backend");
  auto* p = new ginsim_cuda_plugin_s;
  p->comm = comm;
  p->semantics = semantics;
  p->contexts.assign(comm->impl.cfg.n_contexts, nullptr);
  *out = p;
  GIN_API_END
}

int ginsim_cuda_plugin_destroy(ginsim_cuda_plugin_t p) {
  GIN_API_BEGIN
  if (!p) return GINSIM_OK;
  DeviceGuard g(p->comm->impl.device);
  for (auto* d : p->contexts) {
    if (!d) continue;
    cudaStreamSynchronize(d->stream);
    for (auto e : d->in_flight) cudaEventDestroy(e);
    for (auto e : d->spare) cudaEventDestroy(e);
    cudaStreamDestroy(d->stream);
    delete d;
  }
  delete p;
  GIN_API_END
}

int ginsim_cuda_plugin_reg_mr(ginsim_cuda_plugin_t p, uint32_t window_id, uint32_t* mr) {
  GIN_API_BEGIN
  if (!p) fail(GINSIM_E_USAGE, "reg_mr: null plugin");
  Comm* c = &p->comm->impl;
  if (!c->window_live(window_id))
    fail(GINSIM_E_UNKNOWN_WINDOW, "window " + std::to_string(window_id) + " is not registered");
  std::lock_guard<std::mutex> lk(p->mu);
  p->mrs.insert(window_id);  // idempotent: the handle is the window id
  if (mr) *mr = window_id;
  GIN_API_END
}

int ginsim_cuda_plugin_is_registered(ginsim_cuda_plugin_t p, uint32_t window_id, int* out) {
  GIN_API_BEGIN
  if (!p || !out) fail(GINSIM_E_USAGE, "plugin_is_registered: null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  *out = p->mrs.count(window_id) ? 1 : 0;
  GIN_API_END
}

int ginsim_cuda_plugin_iput(ginsim_cuda_plugin_t p, const ginsim_cuda_put_source* src, uint32_t dst_mr,
                            uint64_t dst_offset, uint64_t bytes, uint32_t peer, uint32_t ctx,
                            const ginsim_cuda_action* action, uint64_t* request) {
  GIN_API_BEGIN
  if (!p || !request) fail(GINSIM_E_USAGE, "iput: null argument");
  require_semantics(p, 1, "iput");
  if (action && action->signal_id >= 0) fail(GINSIM_E_GENERIC, "iput does not carry a remote signal; use iput_signal");
  record_call(p, 'p', ctx, peer, bytes);
  *request = iput_common(p, src, dst_mr, dst_offset, bytes, peer, ctx, nullptr, action);
  GIN_API_END
}

int ginsim_cuda_plugin_iput_signal(ginsim_cuda_plugin_t p, const ginsim_cuda_put_source* src, uint32_t dst_mr,
                                   uint64_t dst_offset, uint64_t bytes, uint32_t peer, uint32_t ctx,
                                   uint32_t signal_id, uint32_t signal_add, uint64_t operand,
                                   const ginsim_cuda_action* action, uint64_t* request) {
  GIN_API_BEGIN
  if (!p || !request) fail(GINSIM_E_USAGE, "iput_signal: null argument");
  require_semantics(p, 1, "iput_signal");
  record_call(p, 's', ctx, peer, bytes);
  ginsim_cuda_action sig{(int32_t)signal_id, signal_add, signal_add ? operand : 1ull, -1, 0};
  *request = iput_common(p, src, dst_mr, dst_offset, bytes, peer, ctx, &sig, action);
  GIN_API_END
}

int ginsim_cuda_plugin_test(ginsim_cuda_plugin_t p, uint64_t request, int* done) {
  GIN_API_BEGIN
  if (!p || !done) fail(GINSIM_E_USAGE, "test: null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->requests.find(request);
  if (it == p->requests.end())
    fail(GINSIM_E_UNKNOWN_HANDLE, "request " + std::to_string(request) + " unknown or retired");
  if (!it->second.done) it->second.done = proxy_host_done(&p->comm->impl, it->second.ctx, it->second.ticket);
  *done = it->second.done ? 1 : 0;  // idempotent once true
  GIN_API_END
}

int ginsim_cuda_plugin_retire(ginsim_cuda_plugin_t p, uint64_t request, ginsim_cuda_action* action) {
  GIN_API_BEGIN
  if (!p) fail(GINSIM_E_USAGE, "retire: null plugin");
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->requests.find(request);
  if (it == p->requests.end())
    fail(GINSIM_E_UNKNOWN_HANDLE, "request " + std::to_string(request) + " unknown or retired");
  if (!it->second.done) it->second.done = proxy_host_done(&p->comm->impl, it->second.ctx, it->second.ticket);
  if (!it->second.done) fail(GINSIM_E_GENERIC, "retiring request " + std::to_string(request) + " before completion");
  if (action) *action = it->second.action;
  p->requests.erase(it);
  GIN_API_END
}

int ginsim_cuda_plugin_outstanding(ginsim_cuda_plugin_t p, uint64_t* n) {
  GIN_API_BEGIN
  if (!p || !n) fail(GINSIM_E_USAGE, "plugin_outstanding: null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  *n = p->requests.size();
  GIN_API_END
}

int ginsim_cuda_plugin_set_call_log(ginsim_cuda_plugin_t p, int enabled) {
  GIN_API_BEGIN
  if (!p) fail(GINSIM_E_USAGE, "plugin_set_call_log: null plugin");
  std::lock_guard<std::mutex> lk(p->mu);
  p->log_calls = enabled != 0;
  p->calls.clear();
  GIN_API_END
}

int ginsim_cuda_plugin_call_log(ginsim_cuda_plugin_t p, ginsim_cuda_plugin_call* out, uint32_t max_calls, uint32_t* n) {
  GIN_API_BEGIN
  if (!p || (max_calls && !out)) fail(GINSIM_E_USAGE, "plugin_call_log: null argument");
  std::lock_guard<std::mutex> lk(p->mu);
  const uint32_t k = (uint32_t)std::min<size_t>(max_calls, p->calls.size());
  for (uint32_t i = 0; i < k; ++i) out[i] = p->calls[i];
  if (n) *n = (uint32_t)p->calls.size();
  GIN_API_END
}

int ginsim_cuda_plugin_create_context(ginsim_cuda_plugin_t p, uint32_t ctx, ginsim_cuda_direct_ctx_t* out) {
  GIN_API_BEGIN
  if (!p || !out) fail(GINSIM_E_USAGE, "create_context: null argument");
  require_semantics(p, 0, "create_context");
  if (ctx >= p->contexts.size())
    fail(GINSIM_E_INVALID_CONTEXT, "context " + std::to_string(ctx) + " out of range (" +
                                       std::to_string(p->contexts.size()) + " configured)");
  std::lock_guard<std::mutex> lk(p->mu);
  if (!p->contexts[ctx]) {
    auto* d = new ginsim_cuda_direct_ctx_s;
    d->plugin = p;
    d->index = ctx;
    DeviceGuard g(p->comm->impl.device);
    GIN_CUDA(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    p->contexts[ctx] = d;
  }
  *out = p->contexts[ctx];
  GIN_API_END
}

int ginsim_cuda_direct_post(ginsim_cuda_direct_ctx_t d, const ginsim_cuda_resolved_op* op) {
  GIN_API_BEGIN
  if (!d || !op) fail(GINSIM_E_USAGE, "direct_post: null argument");
  Comm* c = &d->plugin->comm->impl;
  record_call(d->plugin, op->action.signal_id >= 0 ? 's' : 'p', d->index, op->peer, op->bytes);
  std::lock_guard<std::mutex> lk(d->mu);
  const ginsim_cuda_action* a = &op->action;
  switch (op->opcode) {
    case GIN_OP_PUT:
      host_op(c, d->index, GIN_OP_PUT, op->peer, op->dst_window, op->dst_offset, op->src_window,
              op->src_offset_or_value, op->bytes, a, d->stream);
      break;
    case GIN_OP_PUT_INLINE:
      host_op(c, d->index, GIN_OP_PUT_INLINE, op->peer, op->dst_window, op->dst_offset, GIN_INLINE_WINDOW,
              op->src_offset_or_value, op->bytes, a, d->stream);
      break;
    case GIN_OP_SIGNAL_ONLY:
      if (a->signal_id < 0) fail(GINSIM_E_INVALID_DESCRIPTOR, "SIGNAL_ONLY op without a signal");
      if ((uint32_t)a->signal_id >= c->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal out of range");
      host_op(c, d->index, GIN_OP_SIGNAL_ONLY, op->peer, 0, 0, GIN_INLINE_WINDOW, 0, 0, a, d->stream);
      break;
    default:
      fail(GINSIM_E_INVALID_DESCRIPTOR, "unknown opcode " + std::to_string(op->opcode));
  }
  DeviceGuard g(c->device);
  cudaEvent_t e;
  if (!d->spare.empty()) {
    e = d->spare.back();
    d->spare.pop_back();
  } else {
    GIN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  GIN_CUDA(cudaEventRecord(e, d->stream));
  d->in_flight.push_back(e);
  GIN_API_END
}

int ginsim_cuda_direct_poll(ginsim_cuda_direct_ctx_t d, uint64_t* retired) {
  GIN_API_BEGIN
  if (!d) fail(GINSIM_E_USAGE, "direct_poll: null context");
  std::lock_guard<std::mutex> lk(d->mu);
  size_t n = 0;
  retire_done(d, &n);
  if (retired) *retired = n;
  GIN_API_END
}

int ginsim_cuda_direct_outstanding(ginsim_cuda_direct_ctx_t d, uint64_t* n) {
  GIN_API_BEGIN
  if (!d || !n) fail(GINSIM_E_USAGE, "direct_outstanding: null argument");
  std::lock_guard<std::mutex> lk(d->mu);
  *n = d->in_flight.size();
  GIN_API_END
}

}  // extern "C"
