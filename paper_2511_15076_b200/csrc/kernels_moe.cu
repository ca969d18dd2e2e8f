// kernels_moe.cu — DeepEP-style MoE dispatch / combine over the GIN device API.
//
// Reference program: proj/core/src/harness_moe.cpp:105-250 (moe_ll_rank_program)
// and its data functions :17-98.  What is preserved bit-exactly:
//   * slot order: slot = sent_to_expert[e]++ in (t ascending, k ascending)
//     order (:143-150);
//   * dispatch message = hidden u16 payload + 16-byte LE meta {src, token, k,
//     tag = k+1} (:82-98), placed at ((e_loc*n+src)*T+slot)*dmsg in the
//     owner's dispatch window (:135-137) [layout 0], or at the compact
//     per-source position (src*T*K + prefix(e_loc) + slot)*dmsg [layout 1];
//   * per-expert release SignalAdd((1<<32)+count) on cell e_loc (:163-167);
//   * expert transform y = u16(3x+17e+1) (:36-38) fused into the combine put
//     to the source at (token*K+k)*cmsg (:203-205);
//   * per-(src, ctx) SignalAdd(count) on the combine flag e_local (:217-223);
//   * weighted reduction out = sum_k u16(w_k*y_k) in u16 wraparound (:227-242).
// bf16 mode (not in the reference) moves the same bytes and computes the
// transform/reduction in fp32 with single rounding per op.
//
// Data path (B200): one warp owns a (token, part) work item: it streams the
// part of the token row from HBM once with 128-bit non-allocating loads and
// issues K 128-bit stores per vector, straight into the K destination
// windows (local HBM or a peer's HBM over NVLink 5).  Per-expert slot numbers
// come from a per-CTA histogram prefix (no atomics on the data path), the
// release is issued by the last CTA to finish (device-scope arrival counter,
// fence.acq_rel.sys on both sides), so one red.release.sys per expert covers
// every warp's stores.
#include <cuda_bf16.h>
#include <cuda_fp8.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "gin_device.cuh"
#include "runtime_internal.h"
#include "tma.cuh"

#include "moe_common.cuh"
#include "moe_lsu.cuh"
#include "moe_tma.cuh"
#include "moe_dedup.cuh"
#include "moe_pipe.cuh"
#include "moe_gen.cuh"


// ------------------------------------------------------------------ C ABI
using namespace ginsim_b200;

struct ginsim_cuda_moe_s {
  Comm* comm = nullptr;
  ginsim_cuda_comm_t comm_handle = nullptr;
  ginsim_cuda_moe_config cfg{};
  uint32_t e_local = 0, parts = 4, G = 0, Gc = 0, Gr = 0, chunk = 0, cparts = 1, cchunk = 0;
  uint32_t win_dispatch = 0, win_counts = 0, win_combine = 0, win_stage = 0, win_cstage = 0, win_mirror = 0;
  bool proxy = false;
  bool pipe = false;              // Proxy pipeline (moe_pipe.cuh): chunked copy-engine puts, layout 1
  uint32_t* pipe_buf = nullptr;   // R.pipe
  void* buf_mirror = nullptr;
  uint32_t* midx = nullptr;
  uint32_t win_rows = 0;
  void* buf_rows = nullptr;
  // windows this handle registered, bit i = entry i of moe_destroy's owned[]
  // list (dispatch, counts, combine, rows, stage, cstage, mirror): a create
  // that failed half way releases exactly what it had
  uint32_t registered = 0;
  uint64_t* aux_g = nullptr;
  void* buf_stage = nullptr;
  void* buf_cstage = nullptr;
  void* buf_dispatch = nullptr;
  void* buf_counts = nullptr;
  void* buf_combine = nullptr;
  unsigned int* ws = nullptr;
  uint32_t* route = nullptr;
  char** dst_g = nullptr;
  bool coop = false;  // TMA dispatch route-table mode, fixed per handle (grid-barrier counters)
  uint64_t* prof = nullptr;  // GINSIM_PROFILE_PHASES=1: [3][1024][8] %globaltimer stamps
  uint64_t iteration_dispatch = 0, iteration_combine = 0;
  uint32_t last_ctas = 0;
  uint32_t fanout = 0;  // layout 2: fan-out CTAs (fixed with the grid at the first launch)
  uint32_t cell0 = 0;   // this handle's signal cells: [cell0, cell0 + e_local + 3 + kDedupChunks + kCombineChunks)
  uint32_t cchunks = 0;  // pipelined combine: source-token chunks (fixed with the grid at the first launch)
  uint32_t cell_span = 0;
  uint64_t* cell_acc = nullptr;  // [e_local] counts consumed so far per local expert cell (wait targets)
};

extern "C" {

static void check_moe(ginsim_cuda_moe_t moe) {
  if (!moe) fail(GINSIM_E_USAGE, "null moe handle");
}

int ginsim_cuda_moe_create(ginsim_cuda_comm_t comm, const ginsim_cuda_moe_config* cfg, ginsim_cuda_moe_t* out) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!cfg || !out) fail(GINSIM_E_USAGE, "moe_create: null argument");
  if (cfg->experts == 0 || cfg->experts % c->world) fail(GINSIM_E_USAGE, "experts must be divisible by ranks");
  if (cfg->experts > kMaxExperts) fail(GINSIM_E_USAGE, "at most 1024 experts");
  if (cfg->tokens == 0 || cfg->top_k == 0 || cfg->top_k > cfg->experts || cfg->top_k > 32)
    fail(GINSIM_E_USAGE, "need 1..min(experts,32) routed experts per token and at least one token");
  if (cfg->hidden == 0) fail(GINSIM_E_USAGE, "hidden must be positive");
  if (cfg->mode > 3 || cfg->layout > 2) fail(GINSIM_E_USAGE, "mode must be 0..3, layout 0, 1 or 2");
  if (cfg->mode >= 2) {
    if (cfg->hidden % 512) fail(GINSIM_E_USAGE, "fp8 mode needs hidden % 512 == 0 (128-element scale blocks)");
    if (cfg->layout == 2 || c->cfg.backend != GIN_BACKEND_DIRECT || cfg->engine == 1)
      fail(GINSIM_E_USAGE, "fp8 mode runs on the direct TMA path with layout 0 or 1");
  }
  if (cfg->layout == 2) {
    if (c->cfg.backend != GIN_BACKEND_DIRECT) fail(GINSIM_E_USAGE, "layout 2 (dedup transport) needs the direct backend");
    if (cfg->top_k > 15) fail(GINSIM_E_USAGE, "layout 2 carries at most 15 messages per row header");
    if (cfg->experts + c->world > kMaxExperts) fail(GINSIM_E_USAGE, "layout 2: experts + ranks must be <= 1024");
    if ((2u * cfg->hidden) % 16u) fail(GINSIM_E_USAGE, "layout 2 needs 16-byte aligned rows");
    if (cfg->engine == 1) fail(GINSIM_E_USAGE, "layout 2 runs on the TMA engine");
  }
  const uint32_t e_local = cfg->experts / c->world;
  // Every handle owns its signal cells (expert cells, combine flag, rows,
  // chunk and bounds cells): the waits count per-handle iterations, so two
  // handles on one comm must never share a cell.  Handles take consecutive
  // ranges in creation order (identical on every rank: creation is
  // collective); the first handle of a comm starts at cell 0, as the
  // reference's state has it.
  // A range released by moe_destroy is reused (first fit, in the same order
  // on every rank); its cells are reset to zero first -- every rank zeroes
  // the sub-cells of its own table and its proxy agent's running values,
  // between two barriers, so no stale release of the previous handle can
  // satisfy a wait of the new one.
  const uint32_t span = e_local + 3 + kDedupChunks + kCombineChunks;
  uint32_t cell0 = UINT32_MAX;
  {
    std::lock_guard<std::mutex> lk(c->mu);
    for (size_t i = 0; i < c->moe_cells_free.size(); ++i) {
      auto& fr = c->moe_cells_free[i];
      if (fr.second < span) continue;
      cell0 = fr.first;
      fr.first += span;
      fr.second -= span;
      if (fr.second == 0) c->moe_cells_free.erase(c->moe_cells_free.begin() + (long)i);
      break;
    }
    if (cell0 == UINT32_MAX) {
      cell0 = c->moe_cells_next;
      if ((uint64_t)cell0 + span > c->cfg.signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS)
        fail(GINSIM_E_USAGE, "signal table has no room for this MoE handle's " + std::to_string(span) +
                                 " cells (raise Config.signal_cells or destroy unused handles)");
      c->moe_cells_next = cell0 + span;
    }
  }
  {
    c->barrier();  // every rank has destroyed (and synchronised) the previous owner of the range
    if (c->proxy) proxy_reset_cells(c, cell0, span);
    DeviceGuard g(c->device);
    for (uint32_t src = 0; src < c->world; ++src)
      GIN_CUDA(cudaMemset(c->host_view.signals[c->rank] + (uint64_t)src * c->cfg.signal_cells + cell0, 0, span * 8ull));
    GIN_CUDA(cudaMemset(c->host_view.signal_base + cell0, 0, span * 8ull));
    GIN_CUDA(cudaDeviceSynchronize());
    // (the window registrations below are collective: no rank signals into
    //  the range before every rank has reset it)
  }
  auto m = std::make_unique<ginsim_cuda_moe_s>();
  m->comm = c;
  m->comm_handle = comm;
  m->cell0 = cell0;
  m->cell_span = span;
  try {
    m->cfg = *cfg;
    m->e_local = e_local;
    m->parts = cfg->hidden >= 1024 ? 4 : 1;
    const uint64_t dmsg = (cfg->mode >= 2 ? (uint64_t)cfg->hidden + cfg->hidden / 32 : 2ull * cfg->hidden) + 16;
    const uint64_t cmsg = cfg->mode == 3 ? (uint64_t)cfg->hidden + cfg->hidden / 32 : 2ull * cfg->hidden;
    const uint64_t n = c->world, T = cfg->tokens, K = cfg->top_k;
    const uint64_t dbytes = cfg->layout == 0 ? (uint64_t)e_local * n * T * dmsg : n * T * K * dmsg;
    // counts [src][e_loc] + row counts [src] + row bounds [src][chunks + 1] (layout 2)
    // + pipelined-combine slot bounds [src][kCombineChunks - 1][e_loc]
    const uint64_t nbytes = ((uint64_t)e_local * n + n + n * (kDedupChunks + 1) + n * (kCombineChunks - 1) * e_local) * 4;
    const uint64_t cbytes = T * K * cmsg;
    if (ginsim_cuda_mem_alloc(comm, dbytes, &m->buf_dispatch)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if (ginsim_cuda_mem_alloc(comm, nbytes, &m->buf_counts)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if (ginsim_cuda_mem_alloc(comm, cbytes, &m->buf_combine)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    auto reg = [&](void* buf, uint64_t bytes, uint32_t* win, uint32_t bit) {
      const int rc = ginsim_cuda_window_register(comm, buf, bytes, win);
      if (rc) fail(rc, ginsim_cuda_last_error());
      m->registered |= 1u << bit;
    };
    reg(m->buf_dispatch, dbytes, &m->win_dispatch, 0);
    reg(m->buf_counts, nbytes, &m->win_counts, 1);
    reg(m->buf_combine, cbytes, &m->win_combine, 2);
    m->proxy = c->cfg.backend == GIN_BACKEND_PROXY;
    {
      // Proxy backend, compact layout, 16-byte rows, one put per run: the
      // pipelined transport (GINSIM_PROXY_PIPE=0 keeps the one-shot LSU staging
      // kernels; GINSIM_PROXY_COALESCE=0 the reference's one put per message)
      const char* pv = std::getenv("GINSIM_PROXY_PIPE");
      const char* cv = std::getenv("GINSIM_PROXY_COALESCE");
      m->pipe = m->proxy && cfg->layout == 1 && cfg->mode <= 1 && (2u * cfg->hidden) % 16u == 0 &&
                !(pv && pv[0] == '0') && !(cv && cv[0] == '0');
    }
    if (cfg->layout == 2) {
      // row staging: [src][j] rows of 2H bytes, then [src][j] 128-byte headers
      const uint64_t rbytes = n * T * (2ull * cfg->hidden + 128);
      if (ginsim_cuda_mem_alloc(comm, rbytes, &m->buf_rows)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
      reg(m->buf_rows, rbytes, &m->win_rows, 3);
      DeviceGuard dgr(c->device);
      GIN_CUDA(cudaMalloc(&m->aux_g, 2 * (size_t)T * ((K + 1) & ~1ull) * sizeof(uint64_t)));
    }
    if (m->proxy) {
      // Proxy backend: dispatch rows and combine results are staged in local
      // registered windows the host agent copies from (the reference's staging
      // windows, harness_moe.cpp:122-130).  Separate windows, so a combine never
      // overwrites rows the agent may still be copying out for the dispatch.
      // (pipeline: the counts staged for the count puts follow the rows)
      const uint64_t sbytes = T * K * dmsg + (m->pipe ? ((uint64_t)cfg->experts * 4 + 15) / 16 * 16 : 0);
      const uint64_t cbytes2 = n * T * K * cmsg;
      if (ginsim_cuda_mem_alloc(comm, sbytes, &m->buf_stage)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
      reg(m->buf_stage, sbytes, &m->win_stage, 4);
      if (ginsim_cuda_mem_alloc(comm, cbytes2, &m->buf_cstage)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
      reg(m->buf_cstage, cbytes2, &m->win_cstage, 5);
      // combine results in send order ([dst][expert prefix][slot]): one put per run
      if (ginsim_cuda_mem_alloc(comm, cbytes2, &m->buf_mirror)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
      reg(m->buf_mirror, cbytes2, &m->win_mirror, 6);
      DeviceGuard dgm(c->device);
      GIN_CUDA(cudaMalloc(&m->midx, (size_t)T * K * 4));
      if (m->pipe) GIN_CUDA(cudaMalloc(&m->pipe_buf, ((size_t)T * K + kPipeCtrWords) * 4));
    }
    DeviceGuard g(c->device);
    GIN_CUDA(cudaMalloc(&m->ws, kWsBytes));
    GIN_CUDA(cudaMalloc(&m->cell_acc, (size_t)e_local * 8));
    GIN_CUDA(cudaMemset(m->cell_acc, 0, (size_t)e_local * 8));
    GIN_CUDA(cudaMalloc(&m->route, (2 * (size_t)kMaxGrid + 1) * kMaxExperts * 4));
    GIN_CUDA(cudaMalloc(&m->dst_g, (size_t)cfg->tokens * ((cfg->top_k + 1) & ~1u) * sizeof(char*)));
    GIN_CUDA(cudaMemset(m->ws, 0, kWsBytes));
    // Cooperative route tables from this many (token, k) pairs per rank on
    // (GINSIM_DISPATCH_COOP_MIN_PAIRS; the LL shape, 1024 pairs, stays local).
    const char* cm = std::getenv("GINSIM_DISPATCH_COOP_MIN_PAIRS");
    const uint64_t coop_min = cm ? std::strtoull(cm, nullptr, 10) : 8192ull;
    m->coop = (uint64_t)cfg->tokens * cfg->top_k >= coop_min;
    const char* pp = std::getenv("GINSIM_PROFILE_PHASES");
    if (pp && pp[0] == '1') {
      GIN_CUDA(cudaMalloc(&m->prof, 3 * 1024 * 8 * sizeof(uint64_t)));
      GIN_CUDA(cudaMemset(m->prof, 0, 3 * 1024 * 8 * sizeof(uint64_t)));
    }
  } catch (...) {
    // release what this rank allocated and registered, and its cell range
    // (moe_destroy is local); the rethrown error is the one reported
    ginsim_cuda_moe_destroy(m.release());
    throw;
  }
  *out = m.release();
  GIN_API_END
}

int ginsim_cuda_moe_destroy(ginsim_cuda_moe_t moe) {
  GIN_API_BEGIN
  if (!moe) return GINSIM_OK;
  Comm* c = moe->comm;
  ginsim_cuda_comm_t ch = moe->comm_handle;
  {
    DeviceGuard g(c->device);
    GIN_CUDA(cudaDeviceSynchronize());
    if (c->proxy) proxy_quiesce(c);  // no descriptor of this handle left in a ring
    if (moe->ws) cudaFree(moe->ws);
    if (moe->cell_acc) cudaFree(moe->cell_acc);
    if (moe->route) cudaFree(moe->route);
    if (moe->midx) cudaFree(moe->midx);
    if (moe->pipe_buf) cudaFree(moe->pipe_buf);
    if (moe->aux_g) cudaFree(moe->aux_g);
    if (moe->dst_g) cudaFree(moe->dst_g);
    if (moe->prof) cudaFree(moe->prof);
  }
  // Windows and their VMM memory go back (local deregistration: peers'
  // imports of this rank's memory keep it alive until they deregister too).
  const std::pair<uint32_t, void*> owned[] = {
      {moe->win_dispatch, moe->buf_dispatch}, {moe->win_counts, moe->buf_counts}, {moe->win_combine, moe->buf_combine},
      {moe->win_rows, moe->buf_rows},         {moe->win_stage, moe->buf_stage},   {moe->win_cstage, moe->buf_cstage},
      {moe->win_mirror, moe->buf_mirror}};
  for (uint32_t i = 0; i < sizeof(owned) / sizeof(owned[0]); ++i) {
    const auto& o = owned[i];
    if ((moe->registered >> i) & 1u) {
      const int rc = ginsim_cuda_window_deregister(ch, o.first);
      if (rc) fail(rc, ginsim_cuda_last_error());
    }
    if (o.second) {
      const int rc = ginsim_cuda_mem_free(ch, o.second);
      if (rc) fail(rc, ginsim_cuda_last_error());
    }
  }
  {
    std::lock_guard<std::mutex> lk(c->mu);
    c->moe_cells_free.emplace_back(moe->cell0, moe->cell_span);
  }
  delete moe;
  GIN_API_END
}

int ginsim_cuda_moe_cells(ginsim_cuda_moe_t moe, uint32_t* first, uint32_t* span) {
  GIN_API_BEGIN
  check_moe(moe);
  if (first) *first = moe->cell0;
  if (span) *span = moe->cell_span;
  GIN_API_END
}

int ginsim_cuda_moe_windows(ginsim_cuda_moe_t moe, uint32_t* d, uint32_t* c, uint32_t* cb) {
  GIN_API_BEGIN
  check_moe(moe);
  if (d) *d = moe->win_dispatch;
  if (c) *c = moe->win_counts;
  if (cb) *cb = moe->win_combine;
  GIN_API_END
}

int ginsim_cuda_moe_generate(ginsim_cuda_moe_t moe, uint64_t seed, uint32_t src, void* x, int32_t* idx, void* w,
                             void* stream) {
  GIN_API_BEGIN
  check_moe(moe);
  const auto& cfg = moe->cfg;
  DeviceGuard g(moe->comm->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (idx) {
    moe_route_kernel<<<(cfg.tokens + 63) / 64, 64, 0, s>>>(idx, seed, src, cfg.tokens, cfg.experts, cfg.top_k);
    GIN_CUDA(cudaGetLastError());
  }
  if (x) {
    moe_tokens_kernel<<<1184, 256, 0, s>>>(static_cast<uint16_t*>(x), seed, src, cfg.tokens, cfg.hidden, cfg.mode);
    GIN_CUDA(cudaGetLastError());
  }
  if (w) {
    moe_weights_kernel<<<(cfg.tokens * cfg.top_k + 255) / 256, 256, 0, s>>>(w, src, cfg.tokens, cfg.top_k, cfg.mode);
    GIN_CUDA(cudaGetLastError());
  }
  GIN_API_END
}

static MoeLaunch make_launch(const ginsim_cuda_moe_t* moes, uint32_t n) {
  MoeLaunch L{};
  const auto& cfg = moes[0]->cfg;
  L.E = cfg.experts;
  L.K = cfg.top_k;
  L.T = cfg.tokens;
  L.H = cfg.hidden;
  L.mode = cfg.mode;
  L.layout = cfg.layout;
  L.e_local = moes[0]->e_local;
  L.parts = moes[0]->parts;
  L.win_dispatch = moes[0]->win_dispatch;
  L.win_counts = moes[0]->win_counts;
  L.win_combine = moes[0]->win_combine;
  L.win_stage = moes[0]->win_stage;
  L.win_cstage = moes[0]->win_cstage;
  L.win_mirror = moes[0]->win_mirror;
  L.win_rows = moes[0]->win_rows;
  L.cell0 = moes[0]->cell0;
  // Proxy backend: one put descriptor per expert run (default) or per message
  // (GINSIM_PROXY_COALESCE=0, the reference's one-put-per-(t,k) pattern).
  const char* cv = std::getenv("GINSIM_PROXY_COALESCE");
  const bool coalesce = !(cv && cv[0] == '0');
  L.coalesce = coalesce ? 1u : 0u;
  // GINSIM_PROFILE_NO_WAIT=1 lets a profiler replay one rank's dispatch alone
  // (ncu serialises kernels, so a cross-GPU acquire would never complete).
  const char* nw = std::getenv("GINSIM_PROFILE_NO_WAIT");
  L.no_wait = (nw && nw[0] == '1') ? 1u : 0u;
  const char* dy = std::getenv("GINSIM_MOE_SCHED");
  L.dyn = (dy && std::strcmp(dy, "static") == 0) ? 0u : 1u;
  L.coop = moes[0]->coop ? 1u : 0u;
  // cross-lane work sharing: only when the launch carries every rank of the
  // comm (emulated ranks, stepped together, so every lane is at the same
  // iteration); GINSIM_MOE_SHARE=0 turns it off
  const char* sh = std::getenv("GINSIM_MOE_SHARE");
  L.share = (n > 1 && n == moes[0]->comm->world && L.coop && L.dyn && !(sh && sh[0] == '0')) ? 1u : 0u;
  const char* sc = std::getenv("GINSIM_PIPE_STAGE_CTAS");
  // own-expert rows are a plain HBM copy; on 48 CTAs it keeps pace with the
  // copy engines without starving them of HBM (tools/proxy_phases.py, N=2:
  // dispatch 412 us vs 439 us on every CTA)
  L.stage_ctas = sc ? (uint32_t)std::strtoul(sc, nullptr, 10) : 48u;
  L.fanout_ctas = moes[0]->fanout;
  L.fuse_reduce = (moes[0]->coop || moes[0]->pipe) ? 0u : 1u;
  L.mpay = cfg.mode >= 2 ? cfg.hidden + cfg.hidden / 32 : 2u * cfg.hidden;
  L.dmsg = (uint64_t)L.mpay + 16;
  L.cmsg = cfg.mode == 3 ? (uint64_t)cfg.hidden + cfg.hidden / 32 : 2ull * cfg.hidden;
  for (uint32_t i = 0; i < n; ++i) {
    if (std::memcmp(&moes[i]->cfg, &cfg, sizeof(cfg)) != 0 || moes[i]->win_dispatch != L.win_dispatch ||
        moes[i]->cell0 != L.cell0)
      fail(GINSIM_E_USAGE, "moe handles in one launch must share a config");
    L.r[i].view = moes[i]->comm->dev_view;
    L.r[i].ws = moes[i]->ws;
    L.r[i].cell_acc = moes[i]->cell_acc;
    L.r[i].route = moes[i]->route;
    L.r[i].dst_g = moes[i]->dst_g;
    L.r[i].midx = moes[i]->midx;
    L.r[i].aux_g = moes[i]->aux_g;
    L.r[i].pipe = moes[i]->pipe_buf;
    L.r[i].prof = moes[i]->prof;
  }
  return L;
}

// Grid and work split, fixed at the first launch of a handle (the arrival
// counters count CTAs per iteration, so G never changes afterwards).  Every
// CTA must be co-resident: CTAs spin on signals other CTAs release.
// Engines: 1 = LSU everywhere; 2 = TMA dispatch + TMA combine-send + reduce
// kernel; 3 = TMA dispatch + LSU combine; 0 = auto (2 when aligned).
struct MoeKernels {
  const void* dispatch;
  const void* combine;   // cooperative: expert side (+ fused reduce when reduce == nullptr)
  const void* reduce;    // optional separate source-side reduction
  int threads;           // of dispatch
  int cthreads;          // of combine
  bool tma_dispatch, tma_combine;
};

static uint32_t engine_of(const ginsim_cuda_moe_t m) {
  const bool aligned = (2u * m->cfg.hidden) % 16u == 0;
  if (!aligned || m->proxy) return 1;  // the proxy path stages with LSU stores
  return m->cfg.engine == 0 ? 2 : m->cfg.engine;
}
static bool use_tma(const ginsim_cuda_moe_t m) { return engine_of(m) != 1; }

static MoeKernels kernels_of(const ginsim_cuda_moe_t m) {
  const bool k8 = m->cfg.top_k <= 8;
  const uint32_t e = engine_of(m);
  MoeKernels k{};
  if (m->pipe) {
    k.dispatch = (const void*)moe_dispatch_pipe_kernel;
    k.combine = (const void*)moe_combine_pipe_kernel;
    k.reduce = k8 ? (const void*)moe_combine_reduce_kernel<8, false, true>
                  : (const void*)moe_combine_reduce_kernel<32, false, true>;
    k.threads = k.cthreads = kPipeThreads;
    return k;
  }
  if (e == 1 && m->proxy) {
    k.dispatch = k8 ? (const void*)moe_dispatch_kernel<8, true> : (const void*)moe_dispatch_kernel<32, true>;
    k.combine = (const void*)moe_combine_kernel<true>;
    k.threads = k.cthreads = kMoeThreads;
    return k;
  }
  if (e == 1) {
    k.dispatch = k8 ? (const void*)moe_dispatch_kernel<8, false> : (const void*)moe_dispatch_kernel<32, false>;
    k.combine = (const void*)moe_combine_kernel<false>;
    k.threads = k.cthreads = kMoeThreads;
    return k;
  }
  if (m->cfg.layout == 2)
    k.dispatch = k8 ? (const void*)moe_dispatch_dedup_kernel<8> : (const void*)moe_dispatch_dedup_kernel<32>;
  else
    k.dispatch = k8 ? (const void*)moe_dispatch_tma_kernel<8> : (const void*)moe_dispatch_tma_kernel<32>;
  k.threads = kTmaThreads;
  k.tma_dispatch = true;
  if (e == 3) {
    k.combine = (const void*)moe_combine_kernel<false>;
    k.cthreads = kMoeThreads;
  } else {
    k.cthreads = kCmbThreads;
    k.combine = k8 ? (const void*)moe_combine_tma_kernel<8> : (const void*)moe_combine_tma_kernel<32>;
    if (m->cfg.mode == 3)
      k.reduce = k8 ? (const void*)moe_combine_reduce_kernel<8, true, false>
                    : (const void*)moe_combine_reduce_kernel<32, true, false>;
    else
      k.reduce = k8 ? (const void*)moe_combine_reduce_kernel<8, false, false>
                    : (const void*)moe_combine_reduce_kernel<32, false, false>;
    k.tma_combine = true;
  }
  return k;
}

static size_t dispatch_smem(const ginsim_cuda_moe_t m, uint32_t G) {
  const size_t pairs = (size_t)((m->cfg.tokens + G - 1) / G + 1) * m->cfg.top_k;
  if (!kernels_of(m).tma_dispatch) return pairs * 4;
  // control blocks | stages of [destination row (padded to 128 B) | chunk] | own route indices
  const size_t kp = (m->cfg.top_k + 1) & ~1u;
  const size_t dhead = (kp * 8 + 127) & ~(size_t)127;
  // moe_dispatch_tma_kernel: + per-warp expert counters [kTmaWarps][E] for the
  // parallel slot assignment (after the own-route table, 16-byte aligned)
  const size_t whist = m->cfg.layout == 2 ? 0 : (size_t)kTmaWarps * m->cfg.experts * 4 + 16;
  if (m->cfg.mode >= 2) {  // + e4m3 chunk + scales per stage
    const size_t sst = (dhead + m->chunk + m->chunk / 2 + m->chunk / 64 + 15) & ~(size_t)15;
    return ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)kTmaWarps * kDispStages * sst + pairs * 4 +
           whist;
  }
  const size_t tokens = (size_t)((m->cfg.tokens + G - 1) / G + 1);
  const size_t rowj = m->cfg.layout == 2 ? tokens * m->comm->world * 4 : 0;  // dedup: (t, dst) row indices
  return ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)kTmaWarps * kDispStages * (dhead + m->chunk) +
         pairs * 4 + rowj + whist;
}
static size_t combine_smem(const ginsim_cuda_moe_t m) {
  if (!kernels_of(m).tma_combine) return 0;
  // per stage (moe_combine_tma_kernel): mode 3 [hdr][e4m3][scales in][scales out],
  // mode 2 [hdr][scales][bf16 out (codes loaded into its back half)], else [hdr][chunk]
  const size_t c = m->cchunk, scb = (c / 64 + 15) / 16 * 16;
  const size_t sst = m->cfg.mode == 3 ? 128 + c / 2 + 2 * scb : (m->cfg.mode == 2 ? 128 + scb + c : 128 + c);
  // + pipelined combine: the chunk slot bounds [(C-1)][pairs]
  const size_t btab = m->cchunks > 1 ? (size_t)(m->cchunks - 1) * m->cfg.experts * 4 : 0;
  return ((sizeof(TmaSmem) * kCmbWarps + 127) & ~(size_t)127) + (size_t)kCmbWarps * kTmaStages * sst + btab;
}
static int combine_threads(const MoeKernels& k) { return k.cthreads; }

static void plan(const ginsim_cuda_moe_t* moes, uint32_t n) {
  ginsim_cuda_moe_t m = moes[0];
  if (m->G) return;
  const MoeKernels k = kernels_of(m);
  const uint32_t payload = 2u * m->cfg.hidden;
  uint32_t parts = 1, chunk = 0, cparts = 1, cchunk = 0;
  if (use_tma(m)) {
    const char* dc = std::getenv("GINSIM_DISPATCH_CHUNK");  // tuning knob (bytes, multiple of 16)
    const uint32_t dchunk = dc ? std::max(16u, (uint32_t)std::strtoul(dc, nullptr, 10)) : 8192u;
    parts = (payload + dchunk - 1) / dchunk;
    if (!m->coop) {
      // small (latency-bound) launches: split rows further so every warp of a
      // CTA has an item (LL: one token per CTA -> 8 chunks of 1.75 KiB)
      int sms0 = 0;
      GIN_CUDA(cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, m->comm->device));
      const uint32_t G0 = std::max<uint32_t>(1, std::min<uint32_t>((uint32_t)sms0 / n, m->cfg.tokens));
      const uint32_t tpc = (m->cfg.tokens + G0 - 1) / G0;
      const uint32_t want = ((uint32_t)kTmaWarps + tpc - 1) / tpc;
      parts = std::max(parts, std::min(want, std::max(1u, payload / 1024u)));
    }
    chunk = ((payload + parts - 1) / parts + 15) / 16 * 16;
    cparts = (payload + 4095) / 4096;
    cchunk = ((payload + cparts - 1) / cparts + 15) / 16 * 16;
    if (m->cfg.mode >= 2) {
      // fp8: chunks of whole 512-element groups, so every chunk's scale slice
      // (chunk/64 bytes) is a 16-byte multiple at a 16-byte aligned offset
      chunk = (chunk + 1023) / 1024 * 1024;
      parts = (payload + chunk - 1) / chunk;
      // combine: mode 2 expands 4 KiB of bf16 output per stage (its codes
      // load into the buffer's back half); mode 3 re-quantizes 6 KiB in place
      cchunk = m->cfg.mode == 3 ? 6144 : 4096;
      cparts = (payload + cchunk - 1) / cchunk;
    }
    m->chunk = chunk;
    m->cchunk = cchunk;
  }
  // Pipelined combine (moe_common.cuh): one rank per GPU over a real fabric,
  // cooperative route tables, direct TMA kernels with a separate reduce.
  // C * E <= kMaxExperts (the send kernel's prefix table).
  // GINSIM_COMBINE_CHUNKS overrides (0 or 1 = one combine flag at the end).
  uint32_t cchunks = 0;
  if (n == 1 && m->comm->world > 1 && m->coop && !m->proxy && !m->pipe && k.tma_dispatch && k.tma_combine && k.reduce) {
    const char* cc = std::getenv("GINSIM_COMBINE_CHUNKS");
    cchunks = cc ? (uint32_t)std::strtoul(cc, nullptr, 10) : 4u;
    cchunks = std::min(cchunks, std::min(kCombineChunks, kMaxExperts / m->cfg.experts));
    if (cchunks < 2) cchunks = 0;
  }
  m->cchunks = cchunks;
  int sms = 0;
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->comm->device));
  const uint32_t G0 = std::max<uint32_t>(1, (uint32_t)sms / n);
  const size_t ds = dispatch_smem(m, G0), cs = combine_smem(m);
  // Opt every kernel into the full shared-memory budget once; the per-launch
  // dynamic size (which differs between handles) stays below it.
  for (const void* f : {k.dispatch, k.combine}) {
    cudaFuncAttributes fa{};
    GIN_CUDA(cudaFuncGetAttributes(&fa, f));
    int optin = 0;
    GIN_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, m->comm->device));
    GIN_CUDA(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
  }
  const int cap_d = max_coresident_ctas(k.dispatch, k.threads, ds, m->comm->device) / (int)n;
  const int cap_c = max_coresident_ctas(k.combine, combine_threads(k), cs, m->comm->device) / (int)n;
  auto pick = [&](int cap) {
    uint32_t G = m->cfg.ctas ? std::min<uint32_t>(m->cfg.ctas, (uint32_t)cap) : (uint32_t)cap;
    if (G > m->cfg.tokens) G = m->cfg.tokens;
    if (G < 1) fail(GINSIM_E_USAGE, "kernel does not fit on the device");
    return G;
  };
  // Proxy backend: leave half the CTA slots free.  When ranks are emulated on
  // one GPU every agent copy is a same-device copy, which the CUDA runtime
  // runs as a kernel; it must find room next to the waiting MoE kernel.
  const int div = m->proxy ? 2 : 1;
  const uint32_t Gd = pick(std::max(1, cap_d / div)), Gc = pick(std::max(1, cap_c / div));
  uint32_t Gr = 0;
  // (the reduce waits on the combine flag, which on the Proxy backend follows
  // agent copies: emulated ranks' same-device copies need free SMs)
  if (k.reduce)
    Gr = std::max<uint32_t>(1, (uint32_t)max_coresident_ctas(k.reduce, kMoeThreads, 0, m->comm->device) / n / div);
  if (!use_tma(m) || !k.tma_combine) {
    // LSU combine: (message, part) work items sized to the warp count
    const uint32_t nvec = payload % 16u == 0 ? payload / 16u : 0u;
    if (nvec >= 32 && !k.tma_dispatch) {
      const uint32_t want = (2u * Gd * kMoeWarps + m->cfg.tokens - 1) / m->cfg.tokens;
      parts = std::max(1u, std::min(want, nvec / 32u));
    }
  }
  // layout 2: two thirds of the CTAs fan received rows out while the rest
  // put (48 of 148 CTAs keep NVLink busy; N=4 HT dispatch 318 us vs 373 us
  // sequential, tools/phase_timeline.py TL_LAYOUT=2); at N=2 half and half
  // (dispatch 194-197 us vs 213-222 sequential, 220 with 98 fan-out CTAs).
  // GINSIM_DEDUP_FANOUT_CTAS overrides; 0 = every CTA puts, then fans out.
  uint32_t fanout = 0;
  if (m->cfg.layout == 2) {
    const char* fo = std::getenv("GINSIM_DEDUP_FANOUT_CTAS");
    fanout = fo ? (uint32_t)std::strtoul(fo, nullptr, 10)
                : (Gd < 4 || m->comm->world < 2 ? 0u : (m->comm->world == 2 ? Gd / 2 : 2 * Gd / 3));
    if (fanout >= Gd) fanout = Gd - 1;
  }
  for (uint32_t i = 0; i < n; ++i) {
    moes[i]->fanout = fanout;
    moes[i]->cchunks = cchunks;
    moes[i]->G = Gd;
    moes[i]->Gc = Gc;
    moes[i]->Gr = Gr;
    moes[i]->parts = parts;
    moes[i]->chunk = chunk;
    moes[i]->cparts = cparts;
    moes[i]->cchunk = cchunk;
  }
}

static void launch_coop(const void* kernel, uint32_t G, uint32_t n, int threads, size_t smem, void** args,
                        cudaStream_t s) {
  GIN_CUDA(cudaLaunchCooperativeKernel(kernel, dim3(G, n), dim3(threads), args, smem, s));
}

static void check_launch_set(const ginsim_cuda_moe_t* moes, uint32_t n) {
  if (n == 0 || n > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "launch needs 1..8 ranks");
  if (!moes) fail(GINSIM_E_USAGE, "null moe handle list");
  for (uint32_t i = 0; i < n; ++i) check_moe(moes[i]);
  for (uint32_t i = 1; i < n; ++i)
    if (moes[i]->comm->device != moes[0]->comm->device) fail(GINSIM_E_USAGE, "emulated ranks must share a device");
}

int ginsim_cuda_moe_dispatch(const ginsim_cuda_moe_t* moes, uint32_t n, const void* const* x,
                             const int32_t* const* idx, void* stream) {
  GIN_API_BEGIN
  NvtxRange nv("ginsim.moe_dispatch");
  check_launch_set(moes, n);
  MoeLaunch L = make_launch(moes, n);
  DeviceGuard g(moes[0]->comm->device);
  plan(moes, n);
  const MoeKernels k = kernels_of(moes[0]);
  L.parts = moes[0]->parts;
  L.fanout_ctas = moes[0]->fanout;
  L.cchunks = moes[0]->cchunks;
  L.dgrid = moes[0]->G;
  const uint32_t G = moes[0]->G;
  uint32_t chunk = moes[0]->chunk;
  const size_t smem = dispatch_smem(moes[0], G);
  if (smem > 227 * 1024) fail(GINSIM_E_USAGE, "too many tokens per CTA for the slot table");
  for (uint32_t i = 0; i < n; ++i) {
    moes[i]->iteration_dispatch += 1;
    L.r[i].x = static_cast<const uint16_t*>(x[i]);
    L.r[i].idx = idx[i];
    L.r[i].iteration = moes[i]->iteration_dispatch;
  }
  void* args[] = {&L, &chunk};
  launch_coop(k.dispatch, G, n, k.threads, smem, args, (cudaStream_t)stream);
  moes[0]->last_ctas = G * n;
  GIN_API_END
}

int ginsim_cuda_moe_combine(const ginsim_cuda_moe_t* moes, uint32_t n, const void* const* weights, void* const* out,
                            void* stream) {
  GIN_API_BEGIN
  NvtxRange nv("ginsim.moe_combine");
  check_launch_set(moes, n);
  MoeLaunch L = make_launch(moes, n);
  DeviceGuard g(moes[0]->comm->device);
  plan(moes, n);
  const MoeKernels k = kernels_of(moes[0]);
  L.parts = moes[0]->parts;
  L.cparts = k.tma_combine ? moes[0]->cparts : moes[0]->parts;
  uint32_t chunk = k.tma_combine ? moes[0]->cchunk : moes[0]->chunk;
  for (uint32_t i = 0; i < n; ++i) {
    moes[i]->iteration_combine += 1;
    if (moes[i]->iteration_combine != moes[i]->iteration_dispatch)
      fail(GINSIM_E_USAGE, "combine must follow exactly one dispatch");
    L.r[i].weights = weights[i];
    L.r[i].out = static_cast<uint16_t*>(out[i]);
    L.r[i].iteration = moes[i]->iteration_combine;
  }
  L.cchunks = moes[0]->cchunks;
  L.dgrid = moes[0]->G;
  void* args[] = {&L, &chunk};
  const uint32_t Gc = moes[0]->Gc;
  // Pipelined combine: the send kernel leaves `rs` SMs to the early reducer
  // (2 full CTAs per SM; nothing fits beside a send CTA -- its registers fill
  // every SM sub-partition), which is launched as a programmatic dependent of
  // the send kernel so it runs while that does and reduces chunks 0..C-2 as
  // they complete; the last chunk at full occupancy once both have finished.
  // GINSIM_EARLY_RED_SMS overrides the SM split.
  uint32_t Gs = Gc, rs = 0;
  if (L.cchunks > 1) {
    const char* es = std::getenv("GINSIM_EARLY_RED_SMS");
    rs = es ? (uint32_t)std::strtoul(es, nullptr, 10) : kEarlyRedSms;
    rs = std::min(rs, Gc / 2);
    Gs = Gc - rs;
    // no grid barrier in the send kernel: a plain launch (every CTA resident)
    GIN_CUDA(cudaLaunchKernel(k.combine, dim3(Gs, n), dim3(combine_threads(k)), args, combine_smem(moes[0]),
                              (cudaStream_t)stream));
  } else {
    launch_coop(k.combine, Gc, n, combine_threads(k), combine_smem(moes[0]), args, (cudaStream_t)stream);
  }
  if (k.reduce && !L.no_wait && !L.fuse_reduce) {  // profiling harness: the reduce would wait on every source's flag
    if (L.cchunks > 1 && rs == 0) {  // no SMs for an early reducer: every chunk after the send kernel
      L.red_first = 0;
      L.red_last = L.cchunks;
    } else if (L.cchunks > 1) {
      MoeLaunch Le = L;
      Le.red_first = 0;
      Le.red_last = L.cchunks - 1;
      void* eargs[] = {&Le, &chunk};
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(2 * rs, n);
      lc.blockDim = dim3(kMoeThreads);
      lc.dynamicSmemBytes = 0;
      lc.stream = (cudaStream_t)stream;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      GIN_CUDA(cudaLaunchKernelExC(&lc, k.reduce, eargs));
      L.red_first = L.cchunks - 1;
      L.red_last = L.cchunks;
    }
    GIN_CUDA(cudaLaunchKernel(k.reduce, dim3(moes[0]->Gr, n), dim3(kMoeThreads), args, 0, (cudaStream_t)stream));
  }
  moes[0]->last_ctas = Gc * n;
  GIN_API_END
}

int ginsim_cuda_moe_phase_times(ginsim_cuda_moe_t moe, uint32_t kernel, uint64_t* out, uint32_t* ctas) {
  GIN_API_BEGIN
  check_moe(moe);
  if (!moe->prof) fail(GINSIM_E_USAGE, "phase stamps need GINSIM_PROFILE_PHASES=1 at moe_create");
  if (kernel > 2) fail(GINSIM_E_USAGE, "kernel: 0 dispatch, 1 combine send, 2 combine reduce");
  DeviceGuard g(moe->comm->device);
  GIN_CUDA(cudaDeviceSynchronize());
  GIN_CUDA(cudaMemcpy(out, moe->prof + (uint64_t)kernel * 1024 * 8, 1024 * 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (ctas) *ctas = kernel == 0 ? moe->G : (kernel == 1 ? moe->Gc : moe->Gr);
  GIN_API_END
}

int ginsim_cuda_moe_transport(ginsim_cuda_moe_t moe, uint32_t* kind) {
  GIN_API_BEGIN
  check_moe(moe);
  if (kind) *kind = moe->pipe ? 2u : (moe->proxy ? 1u : 0u);
  GIN_API_END
}

int ginsim_cuda_moe_last_launch(ginsim_cuda_moe_t moe, uint32_t* ctas, uint32_t* threads) {
  GIN_API_BEGIN
  check_moe(moe);
  if (ctas) *ctas = moe->last_ctas;
  if (threads) *threads = (uint32_t)kernels_of(moe).threads;
  GIN_API_END
}

}  // extern "C"

extern "C" int ginsim_cuda_moe_create_all(const ginsim_cuda_comm_t* comms, uint32_t n,
                                          const ginsim_cuda_moe_config* cfg, ginsim_cuda_moe_t* out) {
  GIN_API_BEGIN
  if (n == 0 || n > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "need 1..8 comms");
  if (!comms || !cfg || !out) fail(GINSIM_E_USAGE, "moe_create_all: null argument");
  for (uint32_t r = 0; r < n; ++r) comm_impl(comms[r]);  // before any rank enters the collective
  std::vector<int> rcs(n, 0);
  std::vector<std::string> msgs(n);
  std::vector<std::thread> ts;
  for (uint32_t r = 0; r < n; ++r) {
    ts.emplace_back([&, r] {
      out[r] = nullptr;
      rcs[r] = ginsim_cuda_moe_create(comms[r], cfg, &out[r]);
      if (rcs[r]) msgs[r] = ginsim_cuda_last_error();
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < n; ++r) {
    if (!rcs[r]) continue;
    // one rank failed: the handles the others made are released (no half-built set)
    for (uint32_t q = 0; q < n; ++q) {
      if (out[q]) ginsim_cuda_moe_destroy(out[q]);
      out[q] = nullptr;
    }
    fail(rcs[r], "rank " + std::to_string(r) + ": " + msgs[r]);
  }
  GIN_API_END
}
