// proxy.cu — the Proxy backend's host agent (the paper's CPU proxy thread,
// PAPER.md:651-669; reference ProxyBackend, proj/core/src/proxy_backend.cpp).
//
//   GPU producer (gin_device.cuh, Gin::submit): ticket from a device counter,
//     wait until the agent has consumed ticket - capacity (a host-written
//     counter), write the 64-byte descriptor into pinned host memory, publish
//     slot.seq = ticket + 1 (proxy_backend.cpp:19-29).
//   Host consumer (this file): drain <= 64 descriptors per ring per pass
//     (proxy_backend.hpp:67-68, cpp:64-113), decode (descriptor.cpp), and post
//     through the plugin's iput / iput_signal analogue: cudaMemcpyAsync for
//     the payload (peer VMM mapping, copy engine) followed, in stream order,
//     by cuStreamWriteValue64 stores for the signal cells.  Up to 4 CUDA
//     streams, peer p on stream p % streams: every op toward one peer (any
//     context) is ordered on one stream -- stronger than the reference's
//     per-(ctx, peer) channel order -- and copies toward different peers
//     overlap each other's per-op overheads.  Because one stream owns each
//     peer's signal sub-cells, the running values the agent writes land in
//     issue order and a cell never moves backwards.  Local counters (and the
//     device-visible flush words) are written once per pass on stream 0 after
//     it has waited for every other stream the pass used, so they too have a
//     single in-order writer.  Ranks emulated on one device share the device's
//     hardware queues (CUDA_DEVICE_MAX_CONNECTIONS, default 8): a stream
//     aliased onto the queue of a spinning MoE kernel would stall the agent
//     behind it, so each of their agents keeps a single stream.
//
// Signals without SM atomics: rank d's cell id is the sum over sources s of a
// sub-cell [s][id] that only s writes (gin_types.h).  The agent is the single
// writer of its rank's sub-cells in proxy mode, so it keeps the running value
// on the host and writes it with a stream memop after the put's copy -- the
// signal is ordered after every earlier put of the channel (fabric.cpp:63-79)
// and no kernel is launched, so a persistent user kernel that occupies every
// SM can never starve the agent.  Counters (local completion,
// proxy_backend.cpp:95-110) are written at the end of the pass whose copies
// completed them.
#include <sched.h>
#include <time.h>

#include <algorithm>
#include <chrono>
#include <cstring>

#include "runtime_internal.h"

namespace ginsim_b200 {

static uint64_t now_ns() {
  timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (uint64_t)ts.tv_sec * 1000000000ull + (uint64_t)ts.tv_nsec;
}

struct ProxyAgent {
  Comm* c = nullptr;
  uint32_t n_ctx = 0, cap = 0;
  std::vector<GinRingSlot*> slots;       // pinned host, device-mapped
  uint64_t* consumed_host = nullptr;     // pinned host, device-mapped: [ctx] tickets consumed
  std::vector<uint64_t> tail;            // next ticket to consume per ctx
  std::vector<cudaStream_t> streams;     // peer p -> streams[p % size]
  std::thread th;
  std::atomic<bool> stop{false};

  // running cell values this agent owns
  std::mutex sig_mu;                     // sig_value: agent thread vs proxy_reset_cells
  std::vector<uint64_t> sig_value;       // [peer][cell] sub-cell (peer, my rank)
  std::vector<uint64_t> ctr_value;       // [cell]

  // inline payload staging (pinned), recycled by pass
  static constexpr uint32_t kStage = 8192;
  uint64_t* stage = nullptr;
  uint32_t stage_next = 0;

  // completion tracking: one event per pass with work
  struct Pass {
    std::vector<cudaEvent_t> evs;        // one per context stream with work
    std::vector<uint64_t> host_done;     // per ctx host tickets complete after this pass
    std::vector<uint32_t> counters;      // counter ids completed by this pass
    uint32_t stage_begin;                // staging entries [stage_begin, stage_next) of this pass
  };
  std::deque<Pass> inflight;
  std::vector<cudaEvent_t> free_events;

  // host-submitted ops
  std::mutex hq_mu;
  std::deque<std::pair<uint32_t, std::array<uint8_t, 64>>> host_queue;
  std::vector<uint64_t> host_submitted;            // per ctx (under hq_mu)
  std::vector<std::atomic<uint64_t>> host_completed;
  std::vector<uint64_t> host_taken;                // per ctx, agent thread only
  std::vector<std::atomic<uint32_t>> counter_pending;

  std::atomic<uint64_t> n_desc{0}, n_copies{0}, busy_ns{0};

  // GINSIM_PROXY_TRACE=1: timing events around every copy (diagnostics)
  struct CopyTrace {
    uint64_t bytes, issue_ns;
    uint32_t ctx;
    cudaEvent_t e0, e1;
  };
  bool trace = false;
  std::mutex trace_mu;
  std::vector<CopyTrace> traces;
  uint64_t t_start = 0;
  std::string failure;
  std::atomic<bool> failed{false};

  // socket transport (Config.transport = 1): every peer but this rank is
  // reached through GIN1 frames (net.cu); peers posted to in this pass
  NetPtr net;
  std::vector<uint8_t> net_touched;

  ProxyAgent(Comm* comm)
      : c(comm),
        host_completed(comm->cfg.n_contexts),
        counter_pending(comm->cfg.counter_cells) {}

  cudaEvent_t get_event() {
    if (!free_events.empty()) {
      cudaEvent_t e = free_events.back();
      free_events.pop_back();
      return e;
    }
    cudaEvent_t e;
    GIN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    return e;
  }

  // Stream memory operations (signals, counters, aligned inline values) are
  // gathered and issued with one cuStreamBatchMemOp per run of consecutive
  // memops; a copy in between flushes them first, so stream order == the
  // ring's ticket order (the watermark rule, fabric.cpp:63-79).
  // (A memop costs ~1.2-1.4 us of stream time on B200 even batched,
  // tools/host_op_probe.py, so workloads should need few of them.)
  std::vector<std::vector<CUstreamBatchMemOpParams>> memops;  // per stream
  std::vector<uint8_t> touched;                               // stream used in this pass
  std::vector<uint8_t> ctr_touched;                           // counter completed in this pass
  static constexpr size_t kMaxBatch = 128;

  // Copy streams 0..S-1 (peer p on p % S); memop queue S is the completion
  // stream when there are several copy streams, else stream 0 doubles as it.
  cudaStream_t comp_stream = nullptr;
  uint32_t stream_index(uint32_t peer) const { return peer % (uint32_t)streams.size(); }
  uint32_t completion_index() const { return comp_stream ? (uint32_t)streams.size() : 0u; }
  cudaStream_t completion_stream() const { return comp_stream ? comp_stream : streams[0]; }
  cudaStream_t stream_at(uint32_t si) const { return si < streams.size() ? streams[si] : comp_stream; }
  void flush_memops(uint32_t si) {
    auto& m = memops[si];
    if (m.empty()) return;
    GIN_CU(cuapi().cuStreamBatchMemOp((CUstream)stream_at(si), (unsigned)m.size(), m.data(), 0));
    m.clear();
  }
  void write64(uint32_t si, uint64_t* dev_addr, uint64_t v) {
    CUstreamBatchMemOpParams op{};
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
    op.writeValue.address = (CUdeviceptr)dev_addr;
    op.writeValue.value64 = v;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    memops[si].push_back(op);
    touched[si] = 1;
    if (memops[si].size() >= kMaxBatch) flush_memops(si);
  }
  void write32(uint32_t si, void* dev_addr, uint32_t v) {
    CUstreamBatchMemOpParams op{};
    op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_32;
    op.writeValue.address = (CUdeviceptr)dev_addr;
    op.writeValue.value = v;
    op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
    memops[si].push_back(op);
    touched[si] = 1;
    if (memops[si].size() >= kMaxBatch) flush_memops(si);
  }

  // Team-relative peer -> world rank (proxy_backend.cpp:72 hooks_.resolve_peer,
  // runtime.cpp:571 / types.cpp:14-20 team_translate).
  uint32_t resolve_peer(uint32_t team, uint32_t peer) const {
    const GinDevCommView& v = c->host_view;
    for (uint32_t i = 0; i < GIN_MAX_TEAMS; ++i) {
      const GinTeamView& t = v.teams[i];
      if (t.n == 0 || t.id != team) continue;
      if (peer >= t.n)
        fail(GINSIM_E_RANK_OUT_OF_RANGE, "proxy: team rank " + std::to_string(peer) + " out of range for team of " +
                                             std::to_string(t.n));
      return t.members[peer];
    }
    fail(GINSIM_E_USAGE, "proxy: team " + std::to_string(team) + " not registered");
  }

  // iput / iput_signal (plugin.hpp:86-90) for one decoded descriptor.
  // The socket transport's post: the same checks, then the bytes go through
  // net.cu (staging copy on the peer's stream + a GIN1 frame); the signal is
  // a frame behind them, applied by the peer's receiver; counters complete
  // with the peer's acks (the pass's completion stream waits for them).
  void post_net(uint32_t ctx, const ginsim_cuda_descriptor& d, uint32_t peer, Pass& pass) {
    const GinDevCommView& v = c->host_view;
    const uint32_t si = stream_index(peer);
    if (d.opcode != GIN_OP_SIGNAL_ONLY && d.bytes > 0) {
      if (d.dst_window >= GIN_MAX_WINDOWS || !((v.win_live >> d.dst_window) & 1ull)) fail(GINSIM_E_UNKNOWN_WINDOW, "proxy: unknown destination window");
      const GinWindowView& dw = v.win[d.dst_window];
      if (d.dst_offset > dw.size[peer] || d.bytes > dw.size[peer] - d.dst_offset)
        fail(GINSIM_E_OUT_OF_BOUNDS, "proxy: destination range exceeds capacity");
      if (d.opcode == GIN_OP_PUT) {
        if (d.src_window >= GIN_MAX_WINDOWS || !((v.win_live >> d.src_window) & 1ull)) fail(GINSIM_E_UNKNOWN_WINDOW, "proxy: unknown source window");
        const GinWindowView& sw = v.win[d.src_window];
        if (d.src_offset_or_value > sw.size[v.rank] || d.bytes > sw.size[v.rank] - d.src_offset_or_value)
          fail(GINSIM_E_OUT_OF_BOUNDS, "proxy: source range exceeds capacity");
        flush_memops(si);
        touched[si] = 1;
        net_put(net.get(), peer, ctx, d.dst_window, d.dst_offset, sw.base[v.rank] + d.src_offset_or_value, d.bytes,
                streams[si]);
      } else {
        net_put_inline(net.get(), peer, ctx, d.dst_window, d.dst_offset, d.src_offset_or_value, (uint32_t)d.bytes);
      }
      net_touched[peer] = 1;
      n_copies.fetch_add(1, std::memory_order_relaxed);
    }
    if (d.flags & GIN_FLAG_HAS_SIGNAL) {
      if (d.signal_id >= v.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "proxy: signal out of range");
      net_signal(net.get(), peer, ctx, d.signal_id, (d.flags & GIN_FLAG_SIGNAL_IS_ADD) != 0,
                 (d.flags & GIN_FLAG_SIGNAL_IS_ADD) ? d.signal_operand : 1ull);
    }
    if (d.flags & GIN_FLAG_HAS_COUNTER) {
      ctr_value[d.counter_id] += 1;
      ctr_touched[d.counter_id] = 1;
      pass.counters.push_back(d.counter_id);
    }
  }

  void post(uint32_t ctx, const ginsim_cuda_descriptor& d, Pass& pass) {
    const GinDevCommView& v = c->host_view;
    const uint32_t peer = resolve_peer(d.team, d.peer);
    if (peer >= v.world) fail(GINSIM_E_INVALID_PEER, "proxy: descriptor peer out of range");
    if (net && peer != v.rank) {
      post_net(ctx, d, peer, pass);
      return;
    }
    const uint32_t si = stream_index(peer);
    cudaStream_t stream = streams[si];
    touched[si] = 1;
    if (d.opcode != GIN_OP_SIGNAL_ONLY && d.bytes > 0) {
      if (d.dst_window >= GIN_MAX_WINDOWS || !((v.win_live >> d.dst_window) & 1ull)) fail(GINSIM_E_UNKNOWN_WINDOW, "proxy: unknown destination window");
      const GinWindowView& dw = v.win[d.dst_window];
      if (d.dst_offset > dw.size[peer] || d.bytes > dw.size[peer] - d.dst_offset)
        fail(GINSIM_E_OUT_OF_BOUNDS, "proxy: destination range exceeds capacity");
      char* dst = dw.base[peer] + d.dst_offset;
      if (d.opcode == GIN_OP_PUT) {
        if (d.src_window >= GIN_MAX_WINDOWS || !((v.win_live >> d.src_window) & 1ull)) fail(GINSIM_E_UNKNOWN_WINDOW, "proxy: unknown source window");
        const GinWindowView& sw = v.win[d.src_window];
        if (d.src_offset_or_value > sw.size[v.rank] || d.bytes > sw.size[v.rank] - d.src_offset_or_value)
          fail(GINSIM_E_OUT_OF_BOUNDS, "proxy: source range exceeds capacity");
        flush_memops(si);
        CopyTrace tr{};
        if (trace) {
          tr = CopyTrace{d.bytes, now_ns(), ctx, nullptr, nullptr};
          GIN_CUDA(cudaEventCreate(&tr.e0));
          GIN_CUDA(cudaEventCreate(&tr.e1));
          GIN_CUDA(cudaEventRecord(tr.e0, stream));
        }
        GIN_CUDA(cudaMemcpyAsync(dst, sw.base[v.rank] + d.src_offset_or_value, d.bytes, cudaMemcpyDefault, stream));
        if (trace) {
          GIN_CUDA(cudaEventRecord(tr.e1, stream));
          std::lock_guard<std::mutex> lk(trace_mu);
          if (traces.size() < 65536) traces.push_back(tr);
        }
        n_copies.fetch_add(1, std::memory_order_relaxed);
      } else if (d.bytes == 4 && ((uintptr_t)dst & 3) == 0) {  // aligned inline values: a memop, no copy
        write32(si, dst, (uint32_t)d.src_offset_or_value);
      } else if (d.bytes == 8 && ((uintptr_t)dst & 7) == 0) {
        write64(si, reinterpret_cast<uint64_t*>(dst), d.src_offset_or_value);
      } else {
        uint64_t* s = stage + (stage_next++ % kStage);
        *s = d.src_offset_or_value;
        flush_memops(si);
        GIN_CUDA(cudaMemcpyAsync(dst, s, d.bytes, cudaMemcpyHostToDevice, stream));
        n_copies.fetch_add(1, std::memory_order_relaxed);
      }
    }
    if (d.flags & GIN_FLAG_HAS_SIGNAL) {
      if (d.signal_id >= v.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "proxy: signal out of range");
      uint64_t val;
      {
        std::lock_guard<std::mutex> lk(sig_mu);
        uint64_t& cell = sig_value[(size_t)peer * v.signal_cells + d.signal_id];
        cell += (d.flags & GIN_FLAG_SIGNAL_IS_ADD) ? d.signal_operand : 1ull;
        val = cell;
      }
      write64(si, v.signals[peer] + (uint64_t)v.rank * v.signal_cells + d.signal_id, val);
    }
    if (d.flags & GIN_FLAG_HAS_COUNTER) {
      // (range-checked before counter_pending was touched)
      ctr_value[d.counter_id] += 1;
      ctr_touched[d.counter_id] = 1;
      pass.counters.push_back(d.counter_id);
    }
  }

  void retire_completed(bool block) {
    while (!inflight.empty()) {
      Pass& p = inflight.front();
      while (!p.evs.empty()) {
        cudaError_t q = block ? cudaEventSynchronize(p.evs.back()) : cudaEventQuery(p.evs.back());
        if (q == cudaErrorNotReady) return;
        GIN_CUDA(q);
        free_events.push_back(p.evs.back());
        p.evs.pop_back();
      }
      for (uint32_t i = 0; i < n_ctx; ++i) {
        if (p.host_done[i] > host_completed[i].load(std::memory_order_relaxed))
          host_completed[i].store(p.host_done[i], std::memory_order_release);
      }
      for (uint32_t id : p.counters) counter_pending[id].fetch_sub(1, std::memory_order_acq_rel);
      inflight.pop_front();
    }
  }

  // Staging entries one pass can take: 64 per device ring + 256 host ops.
  uint32_t max_stage_per_pass() const { return 64u * n_ctx + 256u; }

  size_t progress_once() {
    // Never let the inline staging ring lap an unfinished copy: the oldest
    // pass in flight holds the oldest entry whose H2D copy may not have run
    // yet, and this pass may take up to max_stage_per_pass() more.
    while (!inflight.empty() && stage_next - inflight.front().stage_begin + max_stage_per_pass() > kStage)
      retire_completed(true);
    size_t work = 0;
    bool ranged = false;  // an NVTX range only around passes that found work: the idle spin stays silent
    auto range = [&] {
      if (!ranged) nvtxRangePushA("ginsim.proxy_pass");
      ranged = true;
    };
    Pass pass;
    pass.stage_begin = stage_next;
    pass.host_done.assign(n_ctx, 0);
    std::vector<uint64_t> consumed(n_ctx, 0);
    bool any_dev = false;
    for (uint32_t ctx = 0; ctx < n_ctx; ++ctx) {
      for (uint32_t i = 0; i < 64; ++i) {
        const uint64_t t = tail[ctx];
        GinRingSlot* slot = slots[ctx] + (t & (cap - 1));
        if (__atomic_load_n(&slot->seq, __ATOMIC_ACQUIRE) != t + 1) break;
        uint8_t raw[64];
        std::memcpy(raw, slot->bytes, 64);
        __atomic_store_n(&slot->seq, t + cap, __ATOMIC_RELEASE);
        tail[ctx] = t + 1;
        ginsim_cuda_descriptor d;
        descriptor_decode(raw, &d);  // a malformed descriptor is a protocol bug: fail the run
        if (d.flags & GIN_FLAG_HAS_COUNTER) {
          if (d.counter_id >= c->cfg.counter_cells) fail(GINSIM_E_INVALID_COUNTER, "proxy: counter out of range");
          counter_pending[d.counter_id].fetch_add(1, std::memory_order_acq_rel);
        }
        range();
        post(ctx, d, pass);
        ++work;
        any_dev = true;
        consumed[ctx] = t + 1;
      }
      // free the drained slots for the GPU producers once per ring batch
      if (consumed[ctx]) __atomic_store_n(consumed_host + ctx, consumed[ctx], __ATOMIC_RELEASE);
    }
    {
      std::unique_lock<std::mutex> lk(hq_mu);
      for (uint32_t i = 0; i < 256 && !host_queue.empty(); ++i) {
        auto item = host_queue.front();
        host_queue.pop_front();
        lk.unlock();
        ginsim_cuda_descriptor d;
        descriptor_decode(item.second.data(), &d);
        range();
        post(item.first, d, pass);
        host_taken[item.first] += 1;
        pass.host_done[item.first] = host_taken[item.first];
        ++work;
        lk.lock();
      }
    }
    if (work) {
      // Completion of the pass on the completion stream: it waits for every
      // copy stream this pass used, then writes the local counters completed
      // by the pass and the device-visible flush words (every ticket consumed
      // so far is complete once the copies above are, proxy_backend.cpp:95-128).
      // One stream writes them all, so they only ever move forward; the copy
      // streams never wait on each other.
      const uint32_t S = (uint32_t)streams.size(), comp = completion_index();
      for (uint32_t si = 0; si < S; ++si) {
        if (!touched[si] || si == comp) continue;
        flush_memops(si);
        cudaEvent_t ev = get_event();
        GIN_CUDA(cudaEventRecord(ev, streams[si]));
        GIN_CUDA(cudaStreamWaitEvent(completion_stream(), ev, 0));
        pass.evs.push_back(ev);
        touched[si] = 0;
      }
      if (net) {  // socket peers: local completion = the peer acked every put posted so far
        for (uint32_t p = 0; p < c->world; ++p) {
          if (!net_touched[p]) continue;
          net_touched[p] = 0;
          CUstreamBatchMemOpParams w{};
          w.waitValue.operation = CU_STREAM_MEM_OP_WAIT_VALUE_64;
          w.waitValue.address = (CUdeviceptr)net_acked_device(net.get(), p);
          w.waitValue.value64 = net_last_seq(net.get(), p);
          w.waitValue.flags = CU_STREAM_WAIT_VALUE_GEQ;
          flush_memops(comp);
          GIN_CU(cuapi().cuStreamBatchMemOp((CUstream)completion_stream(), 1, &w, 0));
        }
      }
      for (uint32_t id : pass.counters) {
        if (!ctr_touched[id]) continue;
        ctr_touched[id] = 0;
        write64(comp, c->host_view.counters + id, ctr_value[id]);
      }
      for (uint32_t ctx = 0; ctx < n_ctx; ++ctx) {
        if (!pass.host_done[ctx]) pass.host_done[ctx] = host_taken[ctx];
        if (any_dev && consumed[ctx]) write64(comp, c->host_view.proxy.completed + ctx, consumed[ctx]);
      }
      flush_memops(comp);
      cudaEvent_t ev = get_event();
      GIN_CUDA(cudaEventRecord(ev, completion_stream()));
      pass.evs.push_back(ev);
      touched[comp] = 0;
      inflight.push_back(std::move(pass));
      n_desc.fetch_add(work, std::memory_order_relaxed);
    }
    retire_completed(false);
    if (ranged) nvtxRangePop();
    return work;
  }

  void main() {
    DeviceGuard g(c->device);
    t_start = now_ns();
    uint32_t idle = 0;
    uint64_t stop_seen = 0;
    for (;;) {
      // Stop only once drained: descriptors already handed over (host queue,
      // device rings) are still posted, so a rank that tears down right after
      // issuing its last signal -- e.g. the closing barrier of a program --
      // still delivers it (the reference destroys comms only after every
      // agent joined, harness_launch.cpp:16-63).  Bounded by the comm timeout.
      if (stop.load(std::memory_order_acquire)) {
        if (!stop_seen) stop_seen = now_ns();
        bool queued;
        {
          std::lock_guard<std::mutex> lk(hq_mu);
          queued = !host_queue.empty();
        }
        if (!queued) {
          for (uint32_t ctx = 0; ctx < n_ctx && !queued; ++ctx) {
            const GinRingSlot* slot = slots[ctx] + (tail[ctx] & (cap - 1));
            queued = __atomic_load_n(&slot->seq, __ATOMIC_ACQUIRE) == tail[ctx] + 1;
          }
        }
        if (!queued && inflight.empty()) break;
        if (now_ns() - stop_seen > c->cfg.timeout_ms * 1000000ull) {
          if (net) net_release_waits(net.get());  // a peer that left never acks: let the streams drain
          break;
        }
      }
      const uint64_t t0 = now_ns();
      size_t w = 0;
      try {
        w = progress_once();
      } catch (const std::exception& e) {
        failure = e.what();
        failed.store(true);
        uint32_t code = GIN_DEVERR_VERIFY;
        cudaMemcpy(c->host_view.error, &code, 4, cudaMemcpyHostToDevice);
        return;
      }
      if (w || !inflight.empty()) {
        busy_ns.fetch_add(now_ns() - t0, std::memory_order_relaxed);
        idle = 0;
        continue;
      }
      if (++idle < 20000) {
        busy_ns.fetch_add(now_ns() - t0, std::memory_order_relaxed);
        __builtin_ia32_pause();
      } else if (idle < 40000) {
        sched_yield();
      } else if (!stop.load(std::memory_order_relaxed)) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
    }
    retire_completed(true);
  }
};

ProxyPtr proxy_start(Comm* c) {
  ProxyPtr p(new ProxyAgent(c));
  p->n_ctx = c->cfg.n_contexts;
  p->cap = c->cfg.queue_depth;
  DeviceGuard g(c->device);
  p->streams.assign(c->shares_device ? 1u : std::min<uint32_t>(p->n_ctx, 4u), nullptr);
  for (auto& st : p->streams) GIN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  if (p->streams.size() > 1) GIN_CUDA(cudaStreamCreateWithFlags(&p->comp_stream, cudaStreamNonBlocking));
  p->memops.assign(p->streams.size() + 1, {});
  p->touched.assign(p->streams.size() + 1, 0);
  p->ctr_touched.assign(c->cfg.counter_cells, 0);
  // events are created up front: the agent must never call into the runtime
  // for anything but issuing work once kernels that wait on it are running
  for (int i = 0; i < 256; ++i) {
    cudaEvent_t e;
    GIN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    p->free_events.push_back(e);
  }
  p->slots.resize(p->n_ctx);
  p->tail.assign(p->n_ctx, 0);
  p->host_submitted.assign(p->n_ctx, 0);
  p->host_taken.assign(p->n_ctx, 0);
  for (uint32_t i = 0; i < p->n_ctx; ++i) {
    void* mem = nullptr;
    GIN_CUDA(cudaHostAlloc(&mem, sizeof(GinRingSlot) * p->cap, cudaHostAllocMapped | cudaHostAllocPortable));
    auto* s = static_cast<GinRingSlot*>(mem);
    for (uint32_t k = 0; k < p->cap; ++k) {
      s[k].seq = k;
      std::memset(s[k].bytes, 0, 64);
    }
    p->slots[i] = s;
    void* dptr = nullptr;
    GIN_CUDA(cudaHostGetDevicePointer(&dptr, mem, 0));
    c->host_view.proxy.slots[i] = static_cast<GinRingSlot*>(dptr);
  }
  {
    void* cm = nullptr;
    GIN_CUDA(cudaHostAlloc(&cm, sizeof(uint64_t) * GIN_MAX_CONTEXTS, cudaHostAllocMapped | cudaHostAllocPortable));
    std::memset(cm, 0, sizeof(uint64_t) * GIN_MAX_CONTEXTS);
    p->consumed_host = static_cast<uint64_t*>(cm);
    void* dptr = nullptr;
    GIN_CUDA(cudaHostGetDevicePointer(&dptr, cm, 0));
    c->host_view.proxy.consumed = static_cast<const uint64_t*>(dptr);
  }
  void* st = nullptr;
  GIN_CUDA(cudaHostAlloc(&st, sizeof(uint64_t) * ProxyAgent::kStage, cudaHostAllocPortable));
  p->stage = static_cast<uint64_t*>(st);
  p->sig_value.assign((size_t)c->world * c->cfg.signal_cells, 0);
  const char* tv = std::getenv("GINSIM_PROXY_TRACE");
  p->trace = tv && tv[0] == '1';
  p->ctr_value.assign(c->cfg.counter_cells, 0);
  if (c->cfg.transport == 1) {  // collective: connects every rank's agent to every other
    p->net = net_start(c);
    p->net_touched.assign(c->world, 0);
  }
  ProxyAgent* raw = p.get();
  p->th = std::thread([raw] { raw->main(); });
  return p;
}

NetTransport* proxy_net(Comm* c) { return c->proxy ? c->proxy->net.get() : nullptr; }

void ProxyDeleter::operator()(ProxyAgent* p) const { delete p; }

void proxy_stop(ProxyPtr& p) {
  if (!p) return;
  p->stop.store(true, std::memory_order_release);
  if (p->th.joinable()) p->th.join();
  DeviceGuard g(p->c->device);
  if (p->net) net_release_waits(p->net.get());  // (no-op unless an ack never came)
  for (auto st : p->streams) cudaStreamSynchronize(st);
  if (p->comp_stream) cudaStreamSynchronize(p->comp_stream);
  for (auto& f : p->inflight)
    for (auto e : f.evs) cudaEventDestroy(e);
  for (auto e : p->free_events) cudaEventDestroy(e);
  for (auto s : p->slots) cudaFreeHost(s);
  if (p->consumed_host) cudaFreeHost(p->consumed_host);
  if (p->stage) cudaFreeHost(p->stage);
  for (auto st : p->streams) cudaStreamDestroy(st);
  if (p->comp_stream) cudaStreamDestroy(p->comp_stream);
  p->net.reset();  // joins the sender / receiver threads, closes the connections
  p.reset();
}

uint64_t proxy_host_submit(Comm* c, uint32_t ctx, const uint8_t desc[64]) {
  ProxyAgent* p = c->proxy.get();
  if (p->failed.load()) fail(GINSIM_E_GENERIC, "proxy agent failed: " + p->failure);
  std::array<uint8_t, 64> d;
  std::memcpy(d.data(), desc, 64);
  ginsim_cuda_descriptor dd;
  descriptor_decode(desc, &dd);
  if (dd.flags & GIN_FLAG_HAS_COUNTER) {
    if (dd.counter_id >= c->cfg.counter_cells) fail(GINSIM_E_INVALID_COUNTER, "counter out of range");
    p->counter_pending[dd.counter_id].fetch_add(1, std::memory_order_acq_rel);
  }
  std::lock_guard<std::mutex> lk(p->hq_mu);
  p->host_queue.emplace_back(ctx, d);
  return ++p->host_submitted[ctx];
}

void proxy_check_failed(Comm* c) {
  ProxyAgent* p = c->proxy.get();
  if (p && p->failed.load()) fail(GINSIM_E_GENERIC, "proxy agent failed: " + p->failure);
  if (p && p->net) net_check_failed(p->net.get());
}

bool proxy_host_done(Comm* c, uint32_t ctx, uint64_t ticket) {
  ProxyAgent* p = c->proxy.get();
  if (p->failed.load()) fail(GINSIM_E_GENERIC, "proxy agent failed: " + p->failure);
  return p->host_completed[ctx].load(std::memory_order_acquire) >= ticket;
}

void proxy_host_flush(Comm* c, uint32_t ctx) {
  ProxyAgent* p = c->proxy.get();
  uint64_t snap;
  {
    std::lock_guard<std::mutex> lk(p->hq_mu);
    snap = p->host_submitted[ctx];
  }
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(c->cfg.timeout_ms);
  while (p->host_completed[ctx].load(std::memory_order_acquire) < snap) {
    if (p->failed.load()) fail(GINSIM_E_GENERIC, "proxy agent failed: " + p->failure);
    if (std::chrono::steady_clock::now() > deadline) fail(GINSIM_E_TIMEOUT, "flush: exceeded timeout");
    std::this_thread::yield();
  }
}

void proxy_quiesce(Comm* c) {
  ProxyAgent* p = c->proxy.get();
  if (!p) return;
  DeviceGuard g(c->device);
  std::vector<uint64_t> tickets(p->n_ctx, 0);
  GIN_CUDA(cudaMemcpy(tickets.data(), c->host_view.proxy.tickets, sizeof(uint64_t) * p->n_ctx, cudaMemcpyDeviceToHost));
  std::vector<uint64_t> done(p->n_ctx, 0);
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(c->cfg.timeout_ms);
  for (;;) {
    GIN_CUDA(cudaMemcpy(done.data(), c->host_view.proxy.completed, sizeof(uint64_t) * p->n_ctx, cudaMemcpyDeviceToHost));
    bool all = true;
    for (uint32_t i = 0; i < p->n_ctx; ++i) all &= done[i] >= tickets[i];
    if (all) break;
    if (p->failed.load()) fail(GINSIM_E_GENERIC, "proxy agent failed: " + p->failure);
    if (std::chrono::steady_clock::now() > deadline) fail(GINSIM_E_TIMEOUT, "proxy quiesce: exceeded timeout");
    std::this_thread::sleep_for(std::chrono::microseconds(20));
  }
  for (uint32_t i = 0; i < p->n_ctx; ++i) proxy_host_flush(c, i);
}

void proxy_reset_cells(Comm* c, uint32_t first, uint32_t span) {
  ProxyAgent* p = c->proxy.get();
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(p->sig_mu);
    for (uint32_t peer = 0; peer < c->world; ++peer)
      for (uint32_t i = first; i < first + span; ++i) p->sig_value[(size_t)peer * c->cfg.signal_cells + i] = 0;
  }
  if (p->net) net_reset_cells(p->net.get(), first, span);  // socket peers: the receiver keeps the values
}

bool proxy_counter_pending(Comm* c, uint32_t id) {
  return c->proxy && c->proxy->counter_pending[id].load(std::memory_order_acquire) != 0;
}

// Copy trace (GINSIM_PROXY_TRACE=1): per copy {bytes, ctx, host issue ns,
// device start us, device duration us} relative to the first traced copy;
// returns the number of records written (the trace is then cleared).
uint32_t proxy_trace(Comm* c, double* out, uint32_t max_records) {
  ProxyAgent* p = c->proxy.get();
  std::lock_guard<std::mutex> lk(p->trace_mu);
  const uint32_t nrec = std::min<uint32_t>(max_records, (uint32_t)p->traces.size());
  for (uint32_t i = 0; i < nrec; ++i) {
    auto& t = p->traces[i];
    GIN_CUDA(cudaEventSynchronize(t.e1));
    float st = 0, du = 0;
    GIN_CUDA(cudaEventElapsedTime(&st, p->traces[0].e0, t.e0));
    GIN_CUDA(cudaEventElapsedTime(&du, t.e0, t.e1));
    out[i * 5 + 0] = (double)t.bytes;
    out[i * 5 + 1] = t.ctx;
    out[i * 5 + 2] = (double)(t.issue_ns - p->traces[0].issue_ns) / 1e3;
    out[i * 5 + 3] = st * 1e3;
    out[i * 5 + 4] = du * 1e3;
  }
  for (auto& t : p->traces) {
    cudaEventDestroy(t.e0);
    cudaEventDestroy(t.e1);
  }
  p->traces.clear();
  return nrec;
}

void proxy_stats(Comm* c, uint64_t* descs, uint64_t* copies, uint64_t* busy, uint64_t* wall) {
  ProxyAgent* p = c->proxy.get();
  if (descs) *descs = p->n_desc.load();
  if (copies) *copies = p->n_copies.load();
  if (busy) *busy = p->busy_ns.load();
  if (wall) *wall = now_ns() - p->t_start;
}

}  // namespace ginsim_b200
