// moe_dedup.cuh -- layout 2: dispatch with a per-rank dedup transport.
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
#pragma once

namespace ginsim_b200 {

// ------------------------------------------------------------------ dedup transport (layout 2)
// Layout 2 = the compact receive layout of layout 1 with a per-rank dedup
// transport: a token whose top-k experts include several on one destination
// rank crosses NVLink ONCE for that rank (into the destination's row staging
// window, with a 128-byte header listing (k, local expert, slot) of each of
// its messages there); the destination fans the row out into every expert
// slot locally (HBM) and writes the metas.  The dispatch window, count window
// and expert cells end bit-identical to layout 1 / the reference
// (harness_moe.cpp:135-167): only the wire traffic changes -- at 8 ranks and
// top-8 of 256 a token has 4.63 distinct remote ranks instead of 7.0 remote
// messages, at 2 ranks one row instead of ~4 messages.
//
// Phases (cooperative route tables as moe_dispatch_tma_kernel with the n
// destination "row" bins appended to the E expert bins):
//   A': CTA 0 publishes, per remote destination, the row boundaries of the
//      kDedupChunks token chunks (chunk c = the tokens of CTAs [c*G/C,
//      (c+1)*G/C), so its first row is that CTA's exclusive row prefix) into
//      the destination's count window, then releases its J-ready cell.
//   B: sender CTAs (b < G - Gf) put one row per (token, destination rank);
//      a sender warp that leaves a token chunk drains its bulk stores and
//      counts itself out of the chunk; the last one releases that chunk's
//      cell (e_local + 2 + c) at every destination.
//   C: per remote destination: counts + row count + one release of its rows
//      cell; own experts released as usual.
//   F: fan-out CTAs (b >= G - Gf; all CTAs after C when Gf = 0) walk the
//      (source, chunk) segments in order, acquire each segment's chunk cell
//      and fan its rows out (bulk load header + row chunk, bulk store to each
//      listed message position) while the senders are still putting -- the
//      HBM-bound fan-out overlaps the NVLink-bound row puts.  The last
//      fan-out CTA acquires the rows cells (counts) and releases the
//      experts' (1<<32)+count on behalf of each source (GPU scope).
//   D: acquire every local expert as before.
constexpr uint32_t kRowHdr = 128;

template <int KMAX>
__global__ void __launch_bounds__(kTmaThreads, 1) moe_dispatch_dedup_kernel(MoeLaunch L, uint32_t chunk) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 0, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank;
  const uint32_t E = L.E, K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t EB = E + n;  // expert bins + destination-row bins
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = 2ull * H + 16;
  const uint32_t payload = 2u * H, parts = L.parts;
  const uint32_t Kp = (K + 1) & ~1u;
  const uint32_t t0 = (uint32_t)((uint64_t)b * T / G), t1 = (uint32_t)((uint64_t)(b + 1) * T / G);
  const unsigned int bar_target = (unsigned int)(iteration * G);
  MOE_STAMP(R, 0, 0);

  __shared__ uint32_t hist_all[kMaxExperts + GIN_MAX_RANKS], run[kMaxExperts + GIN_MAX_RANKS];
  __shared__ uint32_t prefix_e[kMaxExperts];
  __shared__ uint32_t seg[GIN_MAX_RANKS * kDedupChunks + 1];  // fan-out: first row item of each (source, chunk)
  __shared__ uint32_t segj[GIN_MAX_RANKS * kDedupChunks];     // first row index (j) of the segment
  __shared__ char* sbase[GIN_MAX_RANKS];
  __shared__ char* rbase[GIN_MAX_RANKS];
  __shared__ int is_last;
  extern __shared__ __align__(128) char dsm[];
  TmaSmem* ctl = reinterpret_cast<TmaSmem*>(dsm) + warp;
  const uint32_t dhead = (Kp * 8 + 127) & ~127u;  // >= kRowHdr for K <= 15
  const uint32_t sstride = dhead + chunk;
  char* stage = dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)warp * kDispStages * sstride;
  uint32_t* own = reinterpret_cast<uint32_t*>(dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) +
                                              (size_t)kTmaWarps * kDispStages * sstride);
  uint32_t* rowj = own + (t1 - t0) * K;  // [t - t0][d]: row index of (t, d) (written by its first pair)
  uint32_t* g_hist = R.route;
  uint32_t* g_pre = R.route + (size_t)kMaxGrid * kMaxExperts;
  uint32_t* g_tot = R.route + 2 * (size_t)kMaxGrid * kMaxExperts;
  char** dst_g = R.dst_g;                 // [T][Kp] payload destination (null: row already sent)
  uint64_t* hdr_g = R.aux_g;              // [T][Kp] header address of the (t, dst) row (remote pairs)
  uint64_t* ent_g = R.aux_g + (size_t)T * Kp;  // [T][Kp] slot | e_loc << 32
  const uint64_t rows_bytes = (uint64_t)n * T * payload;  // row region of the row window, headers follow
  // sender / fan-out split (L.fanout_ctas = Gf; 0 = every CTA does both, in turn)
  const uint32_t Gf = L.fanout_ctas, Gs = G - Gf;
  const bool sender = Gf == 0 || b < Gs, fanner = Gf == 0 || b >= Gs;
  const uint32_t C = kDedupChunks;
  auto chunk_t0 = [&](uint32_t c) { return (uint32_t)((uint64_t)(c * G / C) * T / G); };
  const uint32_t P = e_local * n;
  uint32_t* jwin = reinterpret_cast<uint32_t*>(v->win[L.win_counts].base[rank]) + P + n;  // [src][C+1] row bounds

  for (uint32_t e = tid; e < EB; e += kTmaThreads) {
    hist_all[e] = 0;
    run[e] = 0;
  }
  if (lane == 0) {
    for (int s = 0; s < kDispStages; ++s) gin::tma::mbar_init(&ctl->bar[s], 1);
    gin::tma::fence_mbar_init();
  }
  if (tid < n) {
    sbase[tid] = v->win[L.win_dispatch].base[tid];
    rbase[tid] = v->win[L.win_rows].base[tid];
  }
  __syncthreads();
  // ---- Phase A: route tables over E expert bins + n row bins
  const uint32_t nq = (t1 - t0) * K;
  for (uint32_t q = tid; q < nq; q += kTmaThreads) own[q] = (uint32_t)__ldg(R.idx + (uint64_t)t0 * K + q);
  __syncthreads();
  for (uint32_t q = tid; q < nq; q += kTmaThreads) {
    const uint32_t e = own[q], d = e / e_local, k = q % K, qt = q - k;
    atomicAdd(&hist_all[e], 1u);
    bool first = true;  // first pair of this token on destination d
    for (uint32_t k2 = 0; k2 < k; ++k2) first = first && (own[qt + k2] / e_local != d);
    if (first) atomicAdd(&hist_all[E + d], 1u);
  }
  __syncthreads();
  for (uint32_t e = tid; e < EB; e += kTmaThreads) g_hist[(size_t)b * EB + e] = hist_all[e];
  MOE_STAMP(R, 0, 1);
  rank_grid_barrier(R.ws + 3, bar_target);
  for (uint32_t e = b + warp * G; e < EB; e += kTmaWarps * G) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < G; c0 += 32) {
      const uint32_t bb = c0 + lane;
      const uint32_t xv = bb < G ? __ldcg(g_hist + (size_t)bb * EB + e) : 0u;
      uint32_t incl = xv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (bb < G) g_pre[(size_t)bb * EB + e] = carry + incl - xv;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) g_tot[e] = carry;
  }
  MOE_STAMP(R, 0, 2);
  rank_grid_barrier(R.ws + 4, bar_target);
  for (uint32_t e = tid; e < EB; e += kTmaThreads) {
    run[e] = __ldcg(g_pre + (size_t)b * EB + e);
    hist_all[e] = __ldcg(g_tot + e);
  }
  __syncthreads();
  for (uint32_t d = warp; d < n; d += kTmaWarps) {  // compact-layout prefix per destination
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
  if (b == 0) {
    // A': row boundaries of every token chunk, per remote destination, then
    // its J-ready cell (fence: the bounds before the release)
    for (uint32_t i = tid; i < n * (C + 1); i += kTmaThreads) {
      const uint32_t d = i / (C + 1), c = i % (C + 1);
      if (d == rank) continue;
      const uint32_t j = c == C ? hist_all[E + d] : __ldcg(g_pre + (size_t)(c * G / C) * EB + E + d);
      gin::st_relaxed_sys32(reinterpret_cast<uint32_t*>(v->win[L.win_counts].base[d]) + P + n + rank * (C + 1) + c, j);
    }
    __syncthreads();
    if (tid < n && tid != rank) {
      gin::fence_acq_rel_sys();
      gin::red_relaxed_sys_add(gin.sub_cell(tid, rank, L.cell0 + e_local + 2 + C), 1ull);
    }
  }
  if (nq <= (uint32_t)kTmaWarps * 32) {
    // Every warp ranks one 32-pair segment (warp w: pairs [32w, 32w+32)).
    // Cross-warp offsets: an expert's pairs in earlier segments are counted
    // by scanning own[] (at most 224 broadcast reads); a destination's first
    // pairs in earlier segments come from per-warp row counts.
    __shared__ uint32_t rowcnt[kTmaWarps][GIN_MAX_RANKS];
    if (tid < kTmaWarps * GIN_MAX_RANKS) (&rowcnt[0][0])[tid] = 0;
    __syncthreads();
    const uint32_t q = warp * 32 + lane;
    const bool valid = q < nq;
    const uint32_t e = valid ? own[q] : 0xFFFFFFFFu;
    const uint32_t d = valid ? e / e_local : 0xFFFFFFFFu;
    const uint32_t k = valid ? q % K : 0, qt = q - k;
    bool first = valid;
    for (uint32_t k2 = 0; valid && k2 < k; ++k2) first = first && (own[qt + k2] / e_local != d);
    const uint32_t peers = __match_any_sync(0xffffffffu, e);
    const uint32_t before = __popc(peers & ((1u << lane) - 1u));
    const uint32_t fkey = first ? d : 0xFFFFFFFEu;
    const uint32_t fpeers = __match_any_sync(0xffffffffu, fkey);
    const uint32_t fbefore = __popc(fpeers & ((1u << lane) - 1u));
    uint32_t eprior = 0;
    const uint32_t qlo = min(warp * 32, nq);
    for (uint32_t q2 = 0; q2 < qlo; ++q2) eprior += own[q2] == e ? 1u : 0u;
    if (first && fbefore == 0) rowcnt[warp][d] = __popc(fpeers);
    __syncthreads();
    uint32_t rprior = 0;
    for (uint32_t w2 = 0; first && w2 < warp; ++w2) rprior += rowcnt[w2][d];
    if (valid) {
      const uint32_t t = t0 + q / K, slot = run[e] + eprior + before, e_loc = e % e_local;
      const uint64_t pi = (uint64_t)t * Kp + k;
      ent_g[pi] = (uint64_t)(prefix_e[e] + slot) | ((uint64_t)e_loc << 32);  // position in src's region
      if (d == rank) {
        dst_g[pi] = sbase[d] + ((uint64_t)rank * T * K + prefix_e[e] + slot) * dmsg;
        hdr_g[pi] = 0;
      } else if (first) {
        rowj[(t - t0) * n + d] = run[E + d] + rprior + fbefore;  // the j-th row this rank sends to d
      }
    }
    __syncthreads();  // a token's first pair on d may sit in the previous warp's segment
    if (valid && d != rank) {
      const uint32_t t = t0 + q / K;
      const uint64_t pi = (uint64_t)t * Kp + k;
      const uint32_t j = rowj[(t - t0) * n + d];
      dst_g[pi] = first ? rbase[d] + ((uint64_t)rank * T + j) * payload : nullptr;
      hdr_g[pi] = (uint64_t)(rbase[d] + rows_bytes + ((uint64_t)rank * T + j) * kRowHdr);
    }
    gin::tma::fence_proxy_async_global();
  } else if (warp == 0) {  // larger segments: one warp ranks them in order
    for (uint32_t c0 = 0; c0 < nq; c0 += 32) {
      const uint32_t q = c0 + lane;
      const bool valid = q < nq;
      const uint32_t e = valid ? own[q] : 0xFFFFFFFFu;
      const uint32_t d = valid ? e / e_local : 0xFFFFFFFFu;
      const uint32_t k = valid ? q % K : 0, qt = q - k;
      bool first = valid;
      for (uint32_t k2 = 0; valid && k2 < k; ++k2) first = first && (own[qt + k2] / e_local != d);
      // expert slot: rank among this chunk's pairs with the same expert
      const uint32_t peers = __match_any_sync(0xffffffffu, e);
      const uint32_t before = __popc(peers & ((1u << lane) - 1u));
      const uint32_t base = valid ? run[e] : 0u;
      // row index: rank among this chunk's FIRST pairs with the same destination
      const uint32_t fkey = first ? d : 0xFFFFFFFEu;
      const uint32_t fpeers = __match_any_sync(0xffffffffu, fkey);
      const uint32_t fbefore = __popc(fpeers & ((1u << lane) - 1u));
      const uint32_t fbase = first ? run[E + d] : 0u;
      __syncwarp();
      if (valid) {
        if (before == 0) run[e] = base + __popc(peers);
        if (first && fbefore == 0) run[E + d] = fbase + __popc(fpeers);
      }
      __syncwarp();
      if (valid) {
        const uint32_t t = t0 + q / K, slot = base + before, e_loc = e % e_local;
        const uint64_t pi = (uint64_t)t * Kp + k;
        ent_g[pi] = (uint64_t)(prefix_e[e] + slot) | ((uint64_t)e_loc << 32);  // position in src's region
        if (d == rank) {
          dst_g[pi] = sbase[d] + ((uint64_t)rank * T * K + prefix_e[e] + slot) * dmsg;
          hdr_g[pi] = 0;
        } else if (first) {
          rowj[(t - t0) * n + d] = fbase + fbefore;  // the j-th row this rank sends to d
        }
      }
      __syncwarp();
      // every remote pair of row (t, d) -- its first pair carries the payload,
      // all of them fill their header entry (the first pair has the lowest k,
      // so it sits in this chunk or an earlier one)
      if (valid && d != rank) {
        const uint32_t t = t0 + q / K;
        const uint64_t pi = (uint64_t)t * Kp + k;
        const uint32_t j = rowj[(t - t0) * n + d];
        dst_g[pi] = first ? rbase[d] + ((uint64_t)rank * T + j) * payload : nullptr;
        hdr_g[pi] = (uint64_t)(rbase[d] + rows_bytes + ((uint64_t)rank * T + j) * kRowHdr);
      }
      __syncwarp();
    }
    gin::tma::fence_proxy_async_global();
  }
  MOE_STAMP(R, 0, 3);
  rank_grid_barrier(R.ws + 5, bar_target);
  MOE_STAMP(R, 0, 4);

  // ---- Phase B: one bulk store per (token, destination rank) for remote
  // rows, one per message for own experts
  const char* x = reinterpret_cast<const char*>(R.x);
  const uint64_t items = sender ? (uint64_t)T * parts : 0;
  const uint64_t gw = (uint64_t)b * kTmaWarps + warp, wstride = (uint64_t)Gs * kTmaWarps;
  // a token chunk is done once every sender warp holding one of its items has
  // drained its bulk stores; monotone per-chunk arrival counters (ws[48+c])
  auto chunk_of = [&](uint32_t t) {
    uint32_t c = 0;
    while (c + 1 < C && chunk_t0(c + 1) <= t) ++c;
    return c;
  };
  auto chunk_done = [&](uint32_t c) {  // lane 0, once this warp's items of chunk c completed
    gin::fence_acq_rel_sys();
    const uint64_t len = (uint64_t)(chunk_t0(c + 1 < C ? c + 1 : C) - chunk_t0(c)) * parts;
    const unsigned warps_c = (unsigned)(len < wstride ? len : wstride);
    const unsigned prev = atomicAdd(R.ws + 48 + c, 1u);
    if (prev + 1 == (unsigned)iteration * warps_c) {
      gin::fence_acq_rel_sys();  // every sender warp's rows of the chunk, then the releases
      for (uint32_t d = 0; d < n; ++d)
        if (d != rank) gin::red_relaxed_sys_add(gin.sub_cell(d, rank, L.cell0 + e_local + 2 + c), 1ull);
    }
  };
  uint32_t cur_chunk = 0xFFFFFFFFu;
  auto issue = [&](int s, uint64_t it) {
    const uint32_t t = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + Kp * 8);
    gin::tma::load(sb, dst_g + (uint64_t)t * Kp, Kp * 8, &ctl->bar[s]);
    gin::tma::load(sb + dhead, x + (uint64_t)t * payload + (uint64_t)p * chunk, len, &ctl->bar[s]);
  };
  if (lane == 0) {
    for (int s = 0; s < kDispStages; ++s) {
      const uint64_t it = gw + s * wstride;
      if (it < items) issue(s, it);
    }
  }
  for (uint32_t j = 0;; ++j) {
    const uint64_t it = gw + (uint64_t)j * wstride;
    if (it >= items) break;
    const int s = (int)(j % kDispStages);
    const uint32_t t = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    char* sb = stage + (size_t)s * sstride;
    char* const* dp = reinterpret_cast<char* const*>(sb);
    uint64_t hdr = 0, ent = 0;
    if (p == 0 && lane < K) {
      hdr = hdr_g[(uint64_t)t * Kp + lane];
      ent = ent_g[(uint64_t)t * Kp + lane];
    }
    gin::tma::mbar_wait(&ctl->bar[s], (j / kDispStages) & 1);
    if (p == 0 && lane < K) {
      if (hdr == 0) {
        gin::st_v4(dp[lane] + payload, make_uint4(rank, t, lane, lane + 1));  // own expert: meta in place
      } else {
        // header entry k: {slot, e_loc | k << 16}; the row's first pair also
        // writes {token, mask of this row's k}
        const uint32_t mask = __match_any_sync(__activemask(), (uint32_t)(hdr >> 7));
        *reinterpret_cast<uint2*>(reinterpret_cast<char*>(hdr) + 8 + 8 * lane) =
            make_uint2((uint32_t)ent, (uint32_t)(ent >> 32) | (lane << 16));
        if (dp[lane] != nullptr) *reinterpret_cast<uint2*>(reinterpret_cast<char*>(hdr)) = make_uint2(t, mask);
      }
    }
    if (lane == 0) {
      const uint32_t len = tma_chunk_len(payload, chunk, p);
      for (uint32_t k = 0; k < K; ++k)
        if (dp[k]) gin::tma::store(dp[k] + (uint64_t)p * chunk, sb + dhead, len);
      gin::tma::commit();
      // first item of a new token chunk: once every older group completed
      // (this item's stores stay in flight), count this warp out of the old one
      const uint32_t c = chunk_of(t);
      if (cur_chunk != 0xFFFFFFFFu && c != cur_chunk) {
        gin::tma::wait_done<1>();
        chunk_done(cur_chunk);
      }
      cur_chunk = c;
      if (j >= 1) {
        gin::tma::wait_read<1>();
        const uint64_t nxt = it - wstride + kDispStages * wstride;
        if (nxt < items) issue((int)((j - 1) % kDispStages), nxt);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    gin::tma::wait_all();
    if (cur_chunk != 0xFFFFFFFFu) chunk_done(cur_chunk);
    gin::tma::fence_proxy_async_global();
  }
  MOE_STAMP(R, 0, 5);

  // ---- Phase C (senders): per remote destination: counts + row count, one
  // fence, one release of its rows cell; own experts as usual (GPU scope)
  if (sender) arrive_last(R.ws + 0, (unsigned)(iteration * Gs), &is_last);
  if (sender && is_last && tid == 0) *moe_iter_ptr(R, 0) = iteration;  // all CTAs read it before Phase A's barriers
  if (sender && is_last) {
    for (uint32_t d = warp; d < n; d += kTmaWarps) {
      uint32_t* cb = reinterpret_cast<uint32_t*>(v->win[L.win_counts].base[d]);
      for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
        gin::st_relaxed_sys32(cb + (uint64_t)rank * e_local + e_loc, hist_all[d * e_local + e_loc]);
      if (lane == 0) gin::st_relaxed_sys32(cb + (uint64_t)e_local * n + rank, hist_all[E + d]);
      for (uint32_t c = 1; c < L.cchunks; ++c)  // pipelined combine: chunk slot bounds (moe_common.cuh)
        for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
          gin::st_relaxed_sys32(cb + combine_bounds_index(n, e_local, rank, c, L.cchunks) + e_loc,
                                __ldcg(g_pre + (size_t)combine_chunk_cta(c, L.cchunks, G) * EB + d * e_local + e_loc));
      if (d == rank) {
        gin::fence_acq_rel_gpu();
        for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
          gin::red_relaxed_sys_add(gin.sub_cell(d, rank, L.cell0 + e_loc), (1ull << 32) + hist_all[d * e_local + e_loc]);
      } else {
        gin::fence_acq_rel_sys();
        if (lane == 0) gin::red_relaxed_sys_add(gin.sub_cell(d, rank, L.cell0 + e_local + 1), 1ull);
      }
    }
  }
  MOE_STAMP(R, 0, 6);

  // ---- Phase F: receive side -- fan the rows of every source out into the
  // expert slots of this rank's dispatch window, chunk by chunk as they land
  if (L.no_wait) return;  // profiling harness: the sender's part only
  const uint32_t GF = Gf ? Gf : G, fb = Gf ? b - Gs : b;  // fan-out CTA count / index
  if (fanner) {
    if (tid == 0) {  // every source's row bounds
      for (uint32_t s2 = 0; s2 < n; ++s2)
        if (s2 != rank) gin.wait_ge(gin.sub_cell(rank, s2, L.cell0 + e_local + 2 + C), iteration);
    }
    __syncthreads();
    if (tid == 0) {  // segments chunk-major (the order they land in), sources rotated
      uint32_t acc = 0, i = 0;
      for (uint32_t c = 0; c < C; ++c) {
        for (uint32_t jj = 1; jj < n; ++jj, ++i) {
          const uint32_t s2 = (rank + jj) % n;
          const uint32_t j0 = gin::ld_acquire_sys32(jwin + s2 * (C + 1) + c);
          const uint32_t j1 = gin::ld_acquire_sys32(jwin + s2 * (C + 1) + c + 1);
          seg[i] = acc;
          segj[i] = j0;
          acc += (j1 - j0) * parts;
        }
      }
      seg[i] = acc;
    }
    __syncthreads();
  }
  const uint32_t nseg = (n - 1) * C;
  const char* rows = v->win[L.win_rows].base[rank];
  char* mywin = v->win[L.win_dispatch].base[rank];
  const uint64_t fitems = fanner ? seg[nseg] : 0;
  const uint64_t gwf = (uint64_t)fb * kTmaWarps + warp, fstride = (uint64_t)GF * kTmaWarps;
  auto locate_row = [&](uint64_t it, uint32_t& si, uint32_t& src, uint32_t& jr) {
    uint32_t lo = 0, hi = nseg;  // last segment whose first item <= it
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (seg[mid] <= it) lo = mid; else hi = mid;
    }
    while (lo + 1 < nseg && seg[lo + 1] == seg[lo]) ++lo;  // skip empty segments
    si = lo;
    src = (rank + 1 + lo % (n - 1)) % n;
    jr = segj[lo] + (uint32_t)((it - seg[lo]) / parts);
  };
  uint32_t ready_seg = 0xFFFFFFFFu;  // lane 0: highest segment acquired so far (items ascend)
  auto fissue = [&](int s, uint64_t it) {
    uint32_t si, src, jr;
    locate_row(it, si, src, jr);
    if (ready_seg == 0xFFFFFFFFu || si > ready_seg) {
      gin.wait_ge(gin.sub_cell(rank, src, L.cell0 + e_local + 2 + si / (n - 1)), iteration);
      gin::tma::fence_proxy_async_global();  // rows written by the peer -> this warp's bulk loads
      ready_seg = si;
    }
    const uint32_t p = (uint32_t)(it % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + kRowHdr);
    gin::tma::load(sb, rows + rows_bytes + ((uint64_t)src * T + jr) * kRowHdr, kRowHdr, &ctl->bar[s]);
    gin::tma::load(sb + dhead, rows + ((uint64_t)src * T + jr) * payload + (uint64_t)p * chunk, len, &ctl->bar[s]);
  };
  const uint32_t phase0 = items > gw ? (uint32_t)((items - gw + wstride - 1) / wstride) : 0u;  // items run in B
  if (lane == 0) {
    for (int s = 0; s < kDispStages; ++s) {
      const uint64_t it = gwf + s * fstride;
      if (it < fitems) fissue((int)((phase0 + s) % kDispStages), it);
    }
  }
  for (uint32_t j = 0;; ++j) {
    const uint64_t it = gwf + (uint64_t)j * fstride;
    if (it >= fitems) break;
    const uint32_t jj = phase0 + j;  // continue the stage/parity sequence of Phase B
    const int s = (int)(jj % kDispStages);
    uint32_t si, src, jr;
    locate_row(it, si, src, jr);
    const uint32_t p = (uint32_t)(it % parts);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_wait(&ctl->bar[s], (jj / kDispStages) & 1);
    const uint32_t* h = reinterpret_cast<const uint32_t*>(sb);
    const uint32_t tok = h[0], mask = h[1];
    if (p == 0 && lane < K && ((mask >> lane) & 1)) {
      char* m = mywin + ((uint64_t)src * T * K + h[2 + 2 * lane]) * dmsg;
      gin::st_v4(m + payload, make_uint4(src, tok, lane, lane + 1));
    }
    if (lane == 0) {
      const uint32_t len = tma_chunk_len(payload, chunk, p);
      for (uint32_t k = 0; k < K; ++k) {
        if (!((mask >> k) & 1)) continue;
        char* m = mywin + ((uint64_t)src * T * K + h[2 + 2 * k]) * dmsg;
        gin::tma::store(m + (uint64_t)p * chunk, sb + dhead, len);
      }
      gin::tma::commit();
      if (j >= 1) {
        gin::tma::wait_read<1>();
        const uint64_t nxt = it - fstride + kDispStages * fstride;
        if (nxt < fitems) fissue((int)((jj - 1) % kDispStages), nxt);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    gin::tma::wait_all();
    gin::tma::fence_proxy_async_global();
  }
  // the last fan-out CTA releases every (local expert, remote source) pair on
  // the source's behalf once its counts are in: this GPU is the only reader
  if (fanner) arrive_last(R.ws + 12, (unsigned)(iteration * GF), &is_last);
  if (fanner && is_last) {
    if (tid == 0) gin.wait_ge_signal(L.cell0 + e_local + 1, iteration * (uint64_t)(n - 1));
    __syncthreads();
    const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
    gin::fence_acq_rel_gpu();
    for (uint32_t i = tid; i < P; i += kTmaThreads) {
      const uint32_t e_loc = i / n, src = i % n;
      if (src != rank)
        gin::red_relaxed_sys_add(gin.sub_cell(rank, src, L.cell0 + e_loc),
                                 (1ull << 32) + gin::ld_acquire_sys32(counts + count_index(i, n, e_local)));
    }
  }
  MOE_STAMP(R, 0, 7);
  if (tid == 0 && !L.no_wait)
    for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) acquire_expert_cell(gin, R, L.cell0 + e_loc, e_loc, iteration, n);
}

}  // namespace ginsim_b200
