// moe_pipe.cuh -- the Proxy backend's pipelined MoE transport (layout 1).
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
//
// The Proxy backend moves payload with the copy engines (the host agent's
// cudaMemcpyAsync over the peer mapping), which on B200
// reach 770 GB/s per GPU toward a peer where SM-issued stores stop at 705
// (DESIGN.md §3.2).  The copy engines need contiguous runs, so the SMs stage
// every message of a destination at its final position in a local mirror of
// that destination's receive region -- staging runs at HBM speed, ~5x the
// link -- in position order, and hand each finished chunk (<= 4 per peer,
// >= 2 MiB) to the agent the moment its last message lands, so the copies
// start microseconds after the launch and overlap the rest of the staging.
//
// Wire protocol per (source, destination) and step, all on the destination's
// context ring (ordered onto one stream by the agent, fabric.cpp:63-79):
//   one put of the source's e_local counts (the count window is
//   source-major; issued right after the route tables, so the copy engine
//   moves it while the first chunk stages)  ->  k chunk puts  ->
//   SignalAdd(1) on the destination's rows cell (e_local + 1).
// The destination acquires the rows cell (>= n: its combine kernel resets the
// cell, so the signal table ends as the reference's) and then releases every
// (local expert, source) cell on the source's behalf by (1<<32)+count --
// the reference's per-expert release values (harness_moe.cpp:163-167), so
// cells, counts and windows end bit-identical to the direct path, with 2 +
// k ring descriptors per peer instead of 2*e_local stream memops (a memop
// costs ~1.3 us of stream time, tools/host_op_probe.py).
//
// Peers are visited in the rotated order rank+1, rank+2, ... (own experts
// last, written in place), so at any moment the ranks' first chunks target
// distinct destinations.  The combine send mirrors this: results of source s
// are staged in s's receive order and land in s's mirror window with one
// SignalAdd(total) per source; the reduce gathers through the dispatch's
// (t, k) -> mirror index.
#pragma once

namespace ginsim_b200 {

constexpr int kPipeThreads = 512;
constexpr int kPipeWarps = kPipeThreads / 32;
constexpr uint32_t kPipeChunksPerPeer = 4;
// R.pipe: [T*K] staging position -> (t*K + k) of the dispatch, then the
// counters: dispatch [n][kPipeChunksPerPeer] chunk fill + [n] chunks issued,
// combine the same at +kPipeCombineCtr
constexpr uint32_t kPipeCombineCtr = 128;
constexpr uint32_t kPipeCtrWords = 2 * kPipeCombineCtr;

__device__ __forceinline__ uint32_t pipe_chunk_msgs(uint32_t tot, uint64_t msg_bytes) {
  const uint32_t min_msgs = (uint32_t)max(1ull, ((2ull << 20) + msg_bytes - 1) / msg_bytes);
  return max(min_msgs, (tot + kPipeChunksPerPeer - 1) / kPipeChunksPerPeer);
}

// Flush (runtime.cpp:460-470): a staging window is rewritten only once the
// agent has completed every put this rank submitted before.
__device__ __forceinline__ void pipe_flush_all(const GinDevCommView* v) {
  for (uint32_t ctx = 0; ctx < v->n_ctx; ++ctx) {
    const uint64_t snap = atomicAdd(&v->proxy.tickets[ctx], 0ull);
    gin::Gin(v, ctx).wait_ge(&v->proxy.completed[ctx], snap);
  }
}

// One warp copies a message payload (16-byte vectors, 8 per lane in flight),
// optionally through the combine transform of expert e.
template <bool TRANSFORM>
__device__ __forceinline__ void pipe_copy_row(char* dst, const char* src, uint32_t payload, uint32_t lane,
                                              uint32_t mode, uint32_t e) {
  const uint32_t nv = payload / 16;
  for (uint32_t i0 = 0; i0 < nv; i0 += 256) {
    uint4 r[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t i = i0 + u * 32 + lane;
      if (i < nv) r[u] = gin::ld_nc_v4(src + 16ull * i);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const uint32_t i = i0 + u * 32 + lane;
      if (i < nv) gin::st_v4(dst + 16ull * i, TRANSFORM ? transform_vec(r[u], mode, e) : r[u]);
    }
  }
}

// Chunk bookkeeping after a warp's message at position q of rotated peer j
// landed: every lane orders its stores before the count (GPU scope; the agent
// reads the descriptor after a .sys release, so the copy engine sees them);
// the lane completing a chunk submits its put, the one completing a peer's
// last chunk runs `finish` (same context ring, later tickets).
template <class Finish>
__device__ __forceinline__ void pipe_chunk_done(uint32_t* ctr, uint32_t n, uint32_t j, uint32_t q, uint32_t tot,
                                                uint32_t ch, uint32_t lane, const Finish& finish,
                                                const gin::Gin& g, uint32_t peer, uint32_t dst_win,
                                                uint64_t dst_off0, uint32_t src_win, uint64_t src_off0,
                                                uint64_t msg) {
  gin::fence_acq_rel_gpu();
  __syncwarp();
  if (lane != 0) return;
  const uint32_t c = q / ch, len = min(ch, tot - c * ch);
  if (atomicAdd(&ctr[j * kPipeChunksPerPeer + c], 1u) + 1 != len) return;
  gin::fence_acq_rel_gpu();
  gin::CoopThread me;
  g.put(me, gin::WorldTeam(n), peer, dst_win, dst_off0 + (uint64_t)c * ch * msg, src_win,
        src_off0 + (uint64_t)c * ch * msg, (uint64_t)len * msg);
  gin::fence_acq_rel_gpu();  // this put's ticket before the issued-count increment
  if (atomicAdd(&ctr[n * kPipeChunksPerPeer + j], 1u) + 1 == (tot + ch - 1) / ch) {
    gin::fence_acq_rel_gpu();  // every chunk's ticket before the finishing ops
    finish();
  }
}

__global__ void __launch_bounds__(kPipeThreads, 1) moe_dispatch_pipe_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 0, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t E = L.E, K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = L.dmsg, TK = (uint64_t)T * K;
  const uint32_t payload = 2u * H;
  const uint32_t t0 = (uint32_t)((uint64_t)b * T / G), t1 = (uint32_t)((uint64_t)(b + 1) * T / G);
  const unsigned int bar_target = (unsigned int)(iteration * G);
  MOE_STAMP(R, 0, 0);

  __shared__ uint32_t hist_all[kMaxExperts], run[kMaxExperts], prefix_e[kMaxExperts];
  __shared__ uint32_t pbase[GIN_MAX_RANKS + 1], pch[GIN_MAX_RANKS];
  __shared__ int is_last;
  extern __shared__ uint32_t own[];  // [(t1-t0)*K] experts of this CTA's pairs
  uint32_t* inv = R.pipe;
  uint32_t* ctr = R.pipe + TK;
  unsigned long long* grab = reinterpret_cast<unsigned long long*>(R.ws + 32);  // [2]
  char* stg = v->win[L.win_stage].base[rank];
  const uint64_t cnt_off = TK * dmsg;  // staged counts [E] after the rows

  if (tid == 0) pipe_flush_all(v);
  if (b == 0) {  // published to the grid by the route-table barriers
    for (uint32_t i = tid; i < kPipeCombineCtr; i += kPipeThreads) ctr[i] = 0;
    if (tid == 0) grab[0] = grab[1] = 0;
  }
  for (uint32_t e = tid; e < E; e += kPipeThreads) {
    hist_all[e] = 0;
    run[e] = 0;
  }
  __syncthreads();
  const uint32_t nq = (t1 - t0) * K;
  coop_route_tables<kPipeThreads>(R, E, K, t0, nq, own, hist_all, run, R.ws + 20, R.ws + 21, bar_target);
  for (uint32_t d = warp; d < n; d += kPipeWarps) {  // per-destination exclusive prefix of the expert totals
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < e_local; c0 += 32) {
      const uint32_t e = d * e_local + c0 + lane;
      const uint32_t xv = c0 + lane < e_local ? hist_all[e] : 0u;
      uint32_t incl = xv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (c0 + lane < e_local) prefix_e[e] = carry + incl - xv;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  if (tid == 0) {  // rotated peer order; own experts last
    uint32_t acc = 0;
    for (uint32_t j = 0; j < n; ++j) {
      const uint32_t d = (rank + 1 + j) % n, last = (d + 1) * e_local - 1;
      const uint32_t tot = prefix_e[last] + hist_all[last];
      pbase[j] = acc;
      pch[j] = pipe_chunk_msgs(tot, dmsg);
      acc += tot;
    }
    pbase[n] = acc;
  }
  if (b == 0) {  // counts: staged for the peers' count puts, own ones in place
    uint32_t* cst = reinterpret_cast<uint32_t*>(stg + cnt_off);
    uint32_t* cown = reinterpret_cast<uint32_t*>(v->win[L.win_counts].base[rank]);
    for (uint32_t e = tid; e < E; e += kPipeThreads) {
      cst[e] = hist_all[e];
      if (e / e_local == rank) cown[rank * e_local + e % e_local] = hist_all[e];
    }
  }
  __syncthreads();
  if (warp == 0) {
    // reference slot order (t, k ascending, harness_moe.cpp:143-150), as the
    // TMA dispatch: staging position of every own pair + its mirror index
    for (uint32_t c0 = 0; c0 < nq; c0 += 32) {
      const uint32_t q = c0 + lane;
      const bool valid = q < nq;
      const uint32_t e = valid ? own[q] : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, e);
      const uint32_t before = __popc(peers & ((1u << lane) - 1u));
      const uint32_t base = valid ? run[e] : 0u;
      __syncwarp();
      if (valid) {
        if (before == 0) run[e] = base + __popc(peers);
        const uint32_t d = e / e_local, j = (d + n - rank - 1) % n;
        const uint32_t pos = prefix_e[e] + base + before;
        const uint32_t pair = t0 * K + q;
        inv[pbase[j] + pos] = pair;
        R.midx[pair] = d * (uint32_t)TK + pos;
      }
      __syncwarp();
    }
  }
  MOE_STAMP(R, 0, 3);
  rank_grid_barrier(R.ws + 22, bar_target);
  MOE_STAMP(R, 0, 4);

  // rows release of rotated peer j (one thread), after every chunk put and
  // the counts put on the same ring
  auto finish_peer = [&](uint32_t j) {
    const uint32_t d = (rank + 1 + j) % n;
    gin::CoopThread me;
    gin::Gin(v, d % n_ctx).signal(me, gin::WorldTeam(n), d, L.cell0 + e_local + 1, gin::SignalAdd(1));
  };
  if (b == 0 && tid + 1 < n) {
    // counts first: the copy engine moves them while the first chunk stages
    const uint32_t d = (rank + 1 + tid) % n;
    gin::CoopThread me;
    gin::Gin(v, d % n_ctx).put(me, gin::WorldTeam(n), d, L.win_counts, (uint64_t)rank * e_local * 4, L.win_stage,
                               cnt_off + (uint64_t)d * e_local * 4, (uint64_t)e_local * 4);
    if (pbase[tid + 1] == pbase[tid]) {  // no messages for that peer
      gin::fence_acq_rel_gpu();
      finish_peer(tid);
    }
  }

  // Phase B: messages in staging order, one warp each, from a grab counter
  const char* x = reinterpret_cast<const char*>(R.x);
  char* own_win = v->win[L.win_dispatch].base[rank] + (uint64_t)rank * TK * dmsg;
  // remote messages on every CTA; own ones (a plain HBM copy that would only
  // compete with the copy engines for HBM) on the first L.stage_ctas
  const uint32_t remote_end = pbase[n - 1];
  for (bool own_phase = false;;) {
    uint32_t m = 0;
    if (lane == 0) m = (uint32_t)atomicAdd(grab + (own_phase ? 1 : 0), 1ull) + (own_phase ? remote_end : 0u);
    m = __shfl_sync(0xffffffffu, m, 0);
    if (!own_phase && m >= remote_end) {
      if (b >= L.stage_ctas) break;
      own_phase = true;
      continue;
    }
    if (m >= (uint32_t)TK) break;
    uint32_t j = 0;
    while (m >= pbase[j + 1]) ++j;
    const uint32_t q = m - pbase[j], d = (rank + 1 + j) % n;
    const uint32_t pair = __ldcg(inv + m);
    const uint32_t t = pair / K, k = pair % K;
    char* dst = d == rank ? own_win + (uint64_t)q * dmsg : stg + (uint64_t)m * dmsg;
    pipe_copy_row<false>(dst, x + (uint64_t)t * payload, payload, lane, 0, 0);
    if (lane == 0) gin::st_v4(dst + payload, make_uint4(rank, t, k, k + 1));  // meta {src, token, k, tag}
    if (d != rank)
      pipe_chunk_done(ctr, n, j, q, pbase[j + 1] - pbase[j], pch[j], lane, [&] { finish_peer(j); },
                      gin::Gin(v, d % n_ctx), d, L.win_dispatch, (uint64_t)rank * TK * dmsg, L.win_stage,
                      (uint64_t)pbase[j] * dmsg, dmsg);
  }
  MOE_STAMP(R, 0, 5);

  // Phase C: own experts' rows are in place -> own rows cell (GPU scope)
  arrive_last(R.ws + 0, bar_target, &is_last);
  if (is_last && tid == 0) *moe_iter_ptr(R, 0) = iteration;  // every CTA has read it (arrival)
  if (is_last && tid == 0) {
    gin::fence_acq_rel_gpu();
    gin::red_relaxed_sys_add(gin.sub_cell(rank, rank, L.cell0 + e_local + 1), 1ull);
  }
  MOE_STAMP(R, 0, 6);
  if (L.no_wait) return;
  // Phase D: once every source's rows cell arrived (its chunks, then its
  // counts, precede it on one stream), release each (expert, source) cell on
  // the source's behalf; this GPU is the only reader of these cells
  const uint32_t P = e_local * n;
  if ((uint64_t)b * kPipeThreads < P) {
    if (tid == 0) gin.wait_ge_signal(L.cell0 + e_local + 1, (uint64_t)n);
    __syncthreads();
    const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
    for (uint32_t i = b * kPipeThreads + tid; i < P; i += G * kPipeThreads) {
      const uint32_t src = i / e_local, e_loc = i % e_local;
      gin::red_relaxed_sys_add(gin.sub_cell(rank, src, L.cell0 + e_loc), (1ull << 32) + gin::ld_acquire_sys32(counts + i));
    }
  }
  MOE_STAMP(R, 0, 7);
}

__global__ void __launch_bounds__(kPipeThreads, 1) moe_combine_pipe_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 1, true);
  const GinDevCommView* v = R.view;
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const uint64_t dmsg = L.dmsg, cmsg = L.cmsg, TK = (uint64_t)T * K;
  const uint32_t payload = 2u * H;
  const unsigned int bar_target = (unsigned int)(iteration * G);
  MOE_STAMP(R, 1, 0);

  __shared__ uint32_t cnt[kMaxExperts], src_prefix[kMaxExperts];
  __shared__ uint32_t pbase[GIN_MAX_RANKS + 1], pch[GIN_MAX_RANKS];
  __shared__ int is_last;
  uint32_t* ctr = R.pipe + TK + kPipeCombineCtr;
  unsigned long long* grab = reinterpret_cast<unsigned long long*>(R.ws + 36);  // [2]

  if (tid == 0) pipe_flush_all(v);
  if (b == 0) {
    for (uint32_t i = tid; i < kPipeCombineCtr; i += kPipeThreads) ctr[i] = 0;
    // the dispatch's rows cell back to 0 (runtime.cpp:414-418): every source
    // signalled it once this step, and none signals it again before this
    // rank's combine results reach it
    if (tid == 0) {
      grab[0] = grab[1] = 0;
      if (!L.no_wait) gin::Gin(v, 0).reset_signal(L.cell0 + e_local + 1);
    }
  }
  const uint32_t P = e_local * n;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
  for (uint32_t i = tid; i < P; i += kPipeThreads) cnt[i] = gin::ld_acquire_sys32(counts + count_index(i, n, e_local));
  __syncthreads();
  source_prefix<kPipeWarps>(cnt, src_prefix, n, e_local);
  __syncthreads();
  if (tid == 0) {
    uint32_t acc = 0;
    for (uint32_t j = 0; j < n; ++j) {
      const uint32_t s = (rank + 1 + j) % n, last = (e_local - 1) * n + s;
      const uint32_t tot = src_prefix[last] + cnt[last];
      pbase[j] = acc;
      pch[j] = pipe_chunk_msgs(tot, cmsg);
      acc += tot;
    }
    pbase[n] = acc;
  }
  rank_grid_barrier(R.ws + 26, bar_target);  // counters zeroed
  MOE_STAMP(R, 1, 1);

  const char* recv = v->win[L.win_dispatch].base[rank];
  char* cst = v->win[L.win_cstage].base[rank];
  char* own_mirror = v->win[L.win_mirror].base[rank] + (uint64_t)rank * TK * cmsg;
  const uint32_t total = pbase[n], remote_end = pbase[n - 1];
  for (bool own_phase = false;;) {
    uint32_t m = 0;
    if (lane == 0) m = (uint32_t)atomicAdd(grab + (own_phase ? 1 : 0), 1ull) + (own_phase ? remote_end : 0u);
    m = __shfl_sync(0xffffffffu, m, 0);
    if (!own_phase && m >= remote_end) {
      if (b >= L.stage_ctas) break;
      own_phase = true;
      continue;
    }
    if (m >= total) break;
    uint32_t j = 0;
    while (m >= pbase[j + 1]) ++j;
    const uint32_t q = m - pbase[j], s = (rank + 1 + j) % n;
    // expert of receive position q: the last e_loc whose prefix is <= q
    uint32_t lo = 0, hi = e_local;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (src_prefix[mid * n + s] <= q) lo = mid; else hi = mid;
    }
    const char* msg = recv + ((uint64_t)s * TK + q) * dmsg;
    char* dst = s == rank ? own_mirror + (uint64_t)q * cmsg : cst + (uint64_t)m * cmsg;
    pipe_copy_row<true>(dst, msg, payload, lane, L.mode, rank * e_local + lo);
    if (s != rank) {
      const uint32_t tot = pbase[j + 1] - pbase[j];
      pipe_chunk_done(ctr, n, j, q, tot, pch[j], lane,
                      [&] {
                        gin::CoopThread me;
                        gin::Gin(v, s % n_ctx).signal(me, gin::WorldTeam(n), s, L.cell0 + e_local, gin::SignalAdd(tot));
                      },
                      gin::Gin(v, s % n_ctx), s, L.win_mirror, (uint64_t)rank * TK * cmsg, L.win_cstage,
                      (uint64_t)pbase[j] * cmsg, cmsg);
    }
  }
  MOE_STAMP(R, 1, 2);
  // own results are in place: this rank's share of its own combine flag,
  // through the agent like every other source's (one writer per sub-cell)
  arrive_last(R.ws + 1, bar_target, &is_last);
  if (is_last && tid == 0) *moe_iter_ptr(R, 1) = iteration;  // every CTA has read it (arrival)
  if (is_last && tid == 0) {
    const uint32_t own_tot = pbase[n] - pbase[n - 1];
    gin::fence_acq_rel_gpu();
    gin::CoopThread me;
    if (own_tot) gin::Gin(v, rank % n_ctx).signal(me, gin::WorldTeam(n), rank, L.cell0 + e_local, gin::SignalAdd(own_tot));
  }
  MOE_STAMP(R, 1, 3);
}

}  // namespace ginsim_b200
