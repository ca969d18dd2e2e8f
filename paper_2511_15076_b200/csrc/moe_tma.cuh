// moe_tma.cuh -- TMA-engine dispatch, combine send and reduce kernels.
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
#pragma once

namespace ginsim_b200 {

// Grid-wide barrier among the G CTAs of one rank's cooperative launch: a
// monotone arrival counter (target = iteration * G), so it needs no reset.
__device__ __forceinline__ void rank_grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gin::fence_acq_rel_gpu();
    atomicAdd(ctr, 1u);
    const uint64_t t0 = gin::globaltimer();
    while (true) {
      unsigned cur;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      if (gin::globaltimer() - t0 > 60000000000ull) break;  // 60 s: a broken launch must not hang the GPU
      __nanosleep(20);
    }
  }
  __syncthreads();
}

// Cooperative route tables (Phase A of the TMA dispatch kernels): CTA b
// histograms its own pairs [t0*K, t0*K + nq) into smem (own[] keeps their
// experts) and a global row hist[b][E]; after a grid barrier warp w of CTA b
// scans expert e = b + w*G down the G rows (exclusive prefix = the slots
// taken by earlier CTAs, total = the expert's count); after a second barrier
// the CTA loads its prefix row into run[] and the totals into hist_all[].
template <int THREADS>
__device__ __forceinline__ void coop_route_tables(const MoeRankArgs& R, uint32_t E, uint32_t K, uint32_t t0,
                                                  uint32_t nq, uint32_t* own, uint32_t* hist_all, uint32_t* run,
                                                  unsigned int* bar0, unsigned int* bar1, unsigned int bar_target) {
  constexpr int WARPS = THREADS / 32;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t* g_hist = R.route;                                  // [G][E]
  uint32_t* g_pre = R.route + (size_t)kMaxGrid * kMaxExperts;  // [G][E]
  uint32_t* g_tot = R.route + 2 * (size_t)kMaxGrid * kMaxExperts;  // [E]
  // A0: own routes -> smem + own histogram -> global row
  for (uint32_t q = tid; q < nq; q += THREADS) {
    const uint32_t e = (uint32_t)__ldg(R.idx + (uint64_t)t0 * K + q);
    own[q] = e;
    atomicAdd(&hist_all[e], 1u);
  }
  __syncthreads();
  for (uint32_t e = tid; e < E; e += THREADS) g_hist[(size_t)b * E + e] = hist_all[e];
  MOE_STAMP(R, 0, 1);
  rank_grid_barrier(bar0, bar_target);
  // A1: column scans, one warp per expert e = b + w*G
  for (uint32_t e = b + warp * G; e < E; e += WARPS * G) {
    uint32_t carry = 0;
    auto scan_chunk = [&](uint32_t c0, uint32_t x) {
      uint32_t incl = x;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (c0 + lane < G) g_pre[(size_t)(c0 + lane) * E + e] = carry + incl - x;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    };
    uint32_t pre[8];  // the first 256 rows' loads in flight together
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const uint32_t bb = c * 32 + lane;
      pre[c] = bb < G ? __ldcg(g_hist + (size_t)bb * E + e) : 0u;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c)
      if ((uint32_t)c * 32 < G) scan_chunk(c * 32, pre[c]);
    for (uint32_t c0 = 256; c0 < G; c0 += 32)
      scan_chunk(c0, c0 + lane < G ? __ldcg(g_hist + (size_t)(c0 + lane) * E + e) : 0u);
    if (lane == 0) g_tot[e] = carry;
  }
  MOE_STAMP(R, 0, 2);
  rank_grid_barrier(bar1, bar_target);
  // A2: this CTA's prefix row and the totals; reference slot numbers
  for (uint32_t e = tid; e < E; e += THREADS) {
    run[e] = __ldcg(g_pre + (size_t)b * E + e);
    hist_all[e] = __ldcg(g_tot + e);
  }
  __syncthreads();
}

// Dispatch over the TMA engine.
//  Phase A (route tables, cooperative): CTA b histograms only its own token
//    range into a global row hist[b][E]; after a grid barrier, warp w of CTA
//    b scans expert e = b + w*G down the G rows (exclusive prefix = the slots
//    already taken by earlier CTAs, total = the expert's count); after a
//    second barrier every CTA reads its prefix row and assigns the reference
//    slot numbers to its own (t, k) pairs in (t, k) order
//    (harness_moe.cpp:143-150), writing each pair's destination pointer to a
//    global table dst_g[t][Kp]; a third barrier publishes the table.  Every
//    CTA touches O(E + own pairs) entries instead of scanning all T*K routes
//    with shared-memory atomics (which cost ~20 us per launch at T=4096).
//  Phase B (puts): per-warp 3-stage TMA pipeline over (token, chunk) items;
//    a stage's mbarrier covers both the row chunk and the token's K
//    destination pointers (one 64-byte bulk load from dst_g), so no lane ever
//    waits on a global load; lane 0 bulk-stores the chunk to the K
//    destinations (local HBM or NVLink peer mappings).  Items come from a
//    device counter in one-token batches (L.dyn), so warps whose messages go
//    to slower destinations take fewer tokens and the grid ends together.
//  Phase C/D: last-CTA release per expert, then acquire of local experts.
template <int KMAX>
__global__ void __launch_bounds__(kTmaThreads, 1) moe_dispatch_tma_kernel(MoeLaunch L, uint32_t chunk) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 0, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank;
  const uint32_t E = L.E, K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = L.dmsg;
  const bool fp8 = L.mode >= 2;
  const uint32_t payload = 2u * H, parts = L.parts;
  const uint32_t Kp = (K + 1) & ~1u;  // dst_g row stride: 16-byte rows for the bulk load
  const uint32_t t0 = (uint32_t)((uint64_t)b * T / G), t1 = (uint32_t)((uint64_t)(b + 1) * T / G);
  const unsigned int bar_target = (unsigned int)(iteration * G);
  // coop: route tables built cooperatively + work over all tokens (large T*K);
  // local: every CTA histograms the whole (small) route table and moves only
  // its own tokens -- no grid barrier on the latency-bound LL path
  const bool coop = L.coop != 0;
  MOE_STAMP(R, 0, 0);

  __shared__ uint32_t hist_all[kMaxExperts], run[kMaxExperts], prefix_e[kMaxExperts];
  __shared__ char* sbase[GIN_MAX_RANKS];
  __shared__ uint32_t lane_rank[GIN_MAX_RANKS];
  __shared__ int is_last;
  extern __shared__ __align__(128) char dsm[];
  TmaSmem* ctl = reinterpret_cast<TmaSmem*>(dsm) + warp;
  // Cross-lane sharing (emulated ranks in one launch, L.share): items carry
  // their lane in bits 48+; after the static first round warps take tokens of
  // every lane, round robin, from one launch-wide counter (lane 0's
  // workspace, one counter per iteration parity), so the lanes' puts end
  // together.  Each lane's release then waits until every CTA of the launch
  // has drained its bulk stores (launch-wide arrival counter).
  const uint32_t nl = gridDim.y, my_lane = blockIdx.y;
  const bool share = L.share != 0;
  unsigned long long* sgrab = reinterpret_cast<unsigned long long*>(L.r[0].ws + 40);  // [2] by iteration parity
  unsigned int* sarrive = L.r[0].ws + 44;
  if (tid < nl) lane_rank[tid] = L.r[tid].view->rank;
  // per stage: [dst pointers: Kp * 8 bytes, padded to 128][row chunk]
  const uint32_t dhead = (Kp * 8 + 127) & ~127u;
  // fp8: [dst row][bf16 chunk][e4m3 chunk/2][scales chunk/64, padded]
  const uint32_t qoff = dhead + chunk, soff = qoff + chunk / 2;
  const uint32_t sstride = fp8 ? ((soff + chunk / 64 + 15) & ~15u) : dhead + chunk;
  char* stage = dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)warp * kDispStages * sstride;
  uint32_t* own = reinterpret_cast<uint32_t*>(dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) +
                                              (size_t)kTmaWarps * kDispStages * sstride);  // [(t1-t0)*K]
  char** dst_g = R.dst_g;                                      // [T][Kp]

  for (uint32_t e = tid; e < E; e += kTmaThreads) {
    hist_all[e] = 0;
    run[e] = 0;
  }
  if (lane == 0) {
    for (int s = 0; s < kDispStages; ++s) gin::tma::mbar_init(&ctl->bar[s], 1);
    gin::tma::fence_mbar_init();
  }
  if (tid < n) sbase[tid] = v->win[L.win_dispatch].base[tid];
  __syncthreads();
  // Work source for Phase B.
  const char* x = reinterpret_cast<const char*>(R.x);
  const uint64_t items = coop ? (uint64_t)T * parts : (uint64_t)t1 * parts;
  const uint64_t gw = (uint64_t)b * kTmaWarps + warp, wstride = (uint64_t)G * kTmaWarps;
  const uint64_t lbase = (uint64_t)t0 * parts + warp;  // local mode: warp takes lbase + j*kTmaWarps
  unsigned long long* grab_ctr = reinterpret_cast<unsigned long long*>(R.ws + 10);
  constexpr uint64_t kLaneShift = 48, kItemMask = (1ull << kLaneShift) - 1;
  const uint64_t own_lane_bits = (uint64_t)my_lane << kLaneShift;
  auto next_item = [&]() -> uint64_t {  // lane 0 only
    uint64_t it;
    if (!coop) {
      it = lbase + (ctl->cur++) * kTmaWarps;
    } else if (share && ctl->cur >= kDispStages) {
      if (ctl->end == 0 || ctl->itc >= ctl->end) {
        const uint64_t u = atomicAdd(sgrab + (iteration & 1), 1ull);
        const uint64_t li = (uint64_t)kDispStages * wstride + (u / nl) * parts;
        if (li >= items) return kNoItem;  // every lane holds as many items: all done
        ctl->itc = ((u % nl) << kLaneShift) | li;
        ctl->end = ctl->itc + parts;
      }
      return ctl->itc++;
    } else if (L.dyn && ctl->cur >= kDispStages) {
      // after a static, interleaved first round (items gw + s*wstride, so
      // 1000+ warps do not all hit the counter at once and a small launch
      // still spreads over every CTA): one token per grab
      if (ctl->end == 0 || ctl->itc >= ctl->end) {
        ctl->itc = (uint64_t)kDispStages * wstride + atomicAdd(grab_ctr, (unsigned long long)parts);
        ctl->end = ctl->itc + parts;
      }
      it = ctl->itc++;
    } else {
      it = gw + (ctl->cur++) * wstride;
    }
    return it < items ? (it | own_lane_bits) : kNoItem;
  };
  // A stage's mbarrier expects the row chunk AND the token's destination row;
  // the row chunk does not depend on routing, so it can be requested first.
  auto issue_row = [&](int s, uint64_t it) {  // lane 0
    const uint32_t ln = (uint32_t)(it >> kLaneShift);
    const uint64_t li = it & kItemMask;
    const uint32_t t = (uint32_t)(li / parts), p = (uint32_t)(li % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    const char* xl = ln == my_lane ? x : reinterpret_cast<const char*>(L.r[ln].x);
    gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + Kp * 8);
    gin::tma::load(sb + dhead, xl + (uint64_t)t * payload + (uint64_t)p * chunk, len, &ctl->bar[s]);
  };
  uint32_t lanes_ready = 1u << my_lane;  // lane 0 of each warp: lanes whose dst_g table is published
  auto issue_dst = [&](int s, uint64_t it) {  // lane 0, once dst_g is published
    const uint32_t ln = (uint32_t)(it >> kLaneShift);
    const uint32_t t = (uint32_t)((it & kItemMask) / parts);
    if (!((lanes_ready >> ln) & 1u)) {  // another lane's table: wait for its Phase A barrier
      const unsigned int* b3 = L.r[ln].ws + 5;
      const uint64_t tw = gin::globaltimer();
      for (;;) {
        unsigned cur;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(b3) : "memory");
        if (cur >= bar_target) break;
        if (gin::globaltimer() - tw > v->timeout_ns) {
          gin::raise_error(v, GIN_DEVERR_TIMEOUT);
          break;
        }
        __nanosleep(64);
      }
      gin::tma::fence_proxy_async_global();
      lanes_ready |= 1u << ln;
    }
    char** dg = ln == my_lane ? dst_g : L.r[ln].dst_g;
    gin::tma::load(stage + (size_t)s * sstride, dg + (uint64_t)t * Kp, Kp * 8, &ctl->bar[s]);
  };
  if (lane == 0) {
    // first round static (warp gw: items [gw*S, gw*S+S)), so 1000+ warps do
    // not all hit the grab counter at once when the kernel starts
    ctl->cur = 0;
    ctl->end = 0;
    for (int s = 0; s < kDispStages; ++s) {
      const uint64_t it = next_item();
      ctl->itm[s] = it;
      if (it != kNoItem) issue_row(s, it);
    }
  }
  const uint32_t nq = (t1 - t0) * K;
  if (!coop) {
    // local: the whole route table is small; totals, this CTA's prefix and
    // its own pairs in one vectorised pass (no grid barrier)
    histogram_pass<kTmaThreads>(R.idx, T * K, t0 * K, nq, hist_all, run, own);
    __syncthreads();
  } else {
    coop_route_tables<kTmaThreads>(R, E, K, t0, nq, own, hist_all, run, R.ws + 3, R.ws + 4, bar_target);
  }
  if (L.layout != 0) {  // per-destination exclusive prefix of the expert totals, one warp per destination
    for (uint32_t d = warp; d < n; d += kTmaWarps) {
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
  }
  // Reference slot order (t, k ascending, harness_moe.cpp:143-150), assigned
  // by all warps at once: warp w owns the w-th contiguous segment of this
  // CTA's pairs; per-warp expert counts, scanned across warps in segment
  // order, give each warp its starting slot per expert (whist[w][e]).
  // Within a segment, 32 pairs at a time: lanes with the same expert rank
  // themselves by lane (match_any) and the group's lowest lane advances the
  // warp's running count.
  // (few pairs, e.g. the LL shape's 8 per CTA: warp 0 alone, no scan)
  const bool one_warp = nq <= 256;
  uint32_t* whist = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(own) + (((size_t)nq * 4 + 15) & ~(size_t)15));
  const uint32_t seg = one_warp ? nq : (((nq + kTmaWarps - 1) / kTmaWarps) + 31) & ~31u;
  const uint32_t q0 = one_warp ? (warp == 0 ? 0u : nq) : min(nq, warp * seg);
  const uint32_t q1 = one_warp ? nq : min(nq, q0 + seg);
  if (!one_warp) {
    for (uint32_t i = tid; i < (uint32_t)kTmaWarps * E; i += kTmaThreads) whist[i] = 0;
    __syncthreads();
    for (uint32_t q = q0 + lane; q < q1; q += 32) atomicAdd(&whist[warp * E + own[q]], 1u);
    __syncthreads();
    for (uint32_t e = tid; e < E; e += kTmaThreads) {
      uint32_t base = run[e];
#pragma unroll
      for (int w = 0; w < kTmaWarps; ++w) {
        const uint32_t c = whist[w * E + e];
        whist[w * E + e] = base;
        base += c;
      }
    }
    __syncthreads();
  }
  if (q0 < q1) {
    uint32_t* wrun = one_warp ? run : whist + warp * E;
    for (uint32_t c0 = q0; c0 < q1; c0 += 32) {
      const uint32_t q = c0 + lane;
      const bool valid = q < q1;
      const uint32_t e = valid ? own[q] : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, e);
      const uint32_t before = __popc(peers & ((1u << lane) - 1u));
      const uint32_t base = valid ? wrun[e] : 0u;
      __syncwarp();
      if (valid) {
        if (before == 0) wrun[e] = base + __popc(peers);
        const uint32_t slot = base + before;
        const uint32_t t = t0 + q / K, k = q % K;
        const uint32_t dst = e / e_local, e_loc = e % e_local;
        const uint64_t off = L.layout == 0 ? (((uint64_t)e_loc * n + rank) * T + slot) * dmsg
                                           : ((uint64_t)rank * T * K + prefix_e[e] + slot) * dmsg;
        dst_g[(uint64_t)t * Kp + k] = sbase[dst] + off;
      }
      __syncwarp();
    }
    gin::tma::fence_proxy_async_global();  // generic writes of dst_g -> read by other CTAs' bulk loads
  }
  MOE_STAMP(R, 0, 3);
  if (coop) rank_grid_barrier(R.ws + 5, bar_target);
  else __syncthreads();  // this CTA's own dst rows, read back by its own bulk loads
  MOE_STAMP(R, 0, 4);

  // Phase B (the first stages' row chunks were requested before Phase A)
  if (lane == 0) {
    gin::tma::fence_proxy_async_global();
    for (int s = 0; s < kDispStages; ++s)
      if (ctl->itm[s] != kNoItem) issue_dst(s, ctl->itm[s]);
  }
  __syncwarp();
  for (uint32_t j = 0;; ++j) {
    const int s = (int)(j % kDispStages);
    const uint64_t it = ctl->itm[s];
    if (it == kNoItem) break;
    const uint32_t ln = (uint32_t)(it >> kLaneShift);
    const uint64_t li = it & kItemMask;
    const uint32_t t = (uint32_t)(li / parts), p = (uint32_t)(li % parts);
    char* sb = stage + (size_t)s * sstride;
    char* const* dp = reinterpret_cast<char* const*>(sb);
    gin::tma::mbar_wait(&ctl->bar[s], (j / kDispStages) & 1);
    if (p == 0 && lane < K) gin::st_v4(dp[lane] + L.mpay, make_uint4(lane_rank[ln], t, lane, lane + 1));  // meta
    if (fp8) {  // quantize the chunk in shared memory, 128 elements per warp step
      const uint32_t len = tma_chunk_len(payload, chunk, p);
      for (uint32_t blk = 0; blk < len / 256; ++blk)
        fp8_quant_block(reinterpret_cast<const uint16_t*>(sb + dhead + blk * 256), reinterpret_cast<uint8_t*>(sb + qoff + blk * 128),
                        reinterpret_cast<float*>(sb + soff) + blk, lane);
      gin::tma::fence_proxy_async_shared();
      __syncwarp();
    }
    if (lane == 0) {
      const uint32_t len = tma_chunk_len(payload, chunk, p);
      if (fp8) {  // e4m3 codes at [p*chunk/2], scales at [H + p*chunk/64]
        for (uint32_t k = 0; k < K; ++k) {
          gin::tma::store(dp[k] + (uint64_t)p * (chunk / 2), sb + qoff, len / 2);
          gin::tma::store(dp[k] + H + (uint64_t)p * (chunk / 64), sb + soff, len / 64);
        }
      } else {
        for (uint32_t k = 0; k < K; ++k) gin::tma::store(dp[k] + (uint64_t)p * chunk, sb + dhead, len);
      }
      gin::tma::commit();
      // Refill the stage of the PREVIOUS item: its stores were committed one
      // iteration ago, so their shared-memory reads overlapped this wait.
      if (j >= 1) {
        gin::tma::wait_read<1>();
        const int ps = (int)((j - 1) % kDispStages);
        const uint64_t nxt = next_item();
        ctl->itm[ps] = nxt;
        if (nxt != kNoItem) {
          issue_row(ps, nxt);
          issue_dst(ps, nxt);
        }
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    gin::tma::wait_all();
    gin::tma::fence_proxy_async_global();
  }

  // Phase C/D as the LSU kernel.
  if (R.prof) {  // puts end = the CTA's LAST warp to drain its bulk stores
    __shared__ unsigned long long warp_end;
    if (tid == 0) warp_end = 0;
    __syncthreads();
    if (lane == 0) atomicMax(&warp_end, (unsigned long long)gin::globaltimer());
    __syncthreads();
    if (tid == 0) R.prof[((uint64_t)0 * 1024 + blockIdx.x) * 8 + 5] = warp_end;
  }
  if (share) {  // launch-wide: this CTA's stores (of any lane) are drained
    __syncthreads();
    if (tid == 0) {
      gin::fence_acq_rel_gpu();
      atomicAdd(sarrive, 1u);
    }
  }
  arrive_last(R.ws + 0, (unsigned)(iteration * G), &is_last);
  if (is_last) {
    if (tid == 0) *grab_ctr = 0;  // every CTA is past Phase B
    if (tid == 0) *moe_iter_ptr(R, 0) = iteration;  // every CTA has read it (arrival)
    if (share) {
      // every lane's items may sit in any CTA: wait for the whole launch
      if (tid == 0) {
        const unsigned target = (unsigned)(iteration * (uint64_t)G * nl);
        const uint64_t tw = gin::globaltimer();
        for (;;) {
          unsigned cur;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(sarrive) : "memory");
          if (cur >= target) break;
          if (gin::globaltimer() - tw > v->timeout_ns) {
            gin::raise_error(v, GIN_DEVERR_TIMEOUT);
            break;
          }
          __nanosleep(32);
        }
        if (my_lane == 0) sgrab[(iteration + 1) & 1] = 0;  // the next iteration's counter (untouched now)
      }
      __syncthreads();
    }
    release_experts(gin, v, L.win_counts, hist_all, n, rank, e_local, L.cell0, L.cchunks > 1 ? L.cchunks : 0u,
                    R.route + (size_t)kMaxGrid * kMaxExperts, E, G);
  }
  MOE_STAMP(R, 0, 6);
  if (tid == 0 && !L.no_wait)
    for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) acquire_expert_cell(gin, R, L.cell0 + e_loc, e_loc, iteration, n);
  MOE_STAMP(R, 0, 7);
}

template <int KMAX>
__global__ void __launch_bounds__(kCmbThreads, 1) moe_combine_tma_kernel(MoeLaunch L, uint32_t chunk) {
  // The transform pass keeps the SM busy between TMA waits, so this kernel
  // runs 16 warps with smaller (<= 4 KiB) chunks instead of the dispatch's 8.
  constexpr int kTmaThreads = kCmbThreads;
  constexpr int kTmaWarps = kCmbThreads / 32;
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 1, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = L.dmsg, cmsg = L.cmsg;
  const bool fp8 = L.mode >= 2, fp8c = L.mode == 3;
  const uint32_t payload = 2u * H, parts = L.cparts;
  // pipelined combine (moe_common.cuh): C source-token chunks; the reducer
  // launched behind this kernel may start as soon as every CTA is resident
  const uint32_t C = L.cchunks > 1 ? L.cchunks : 1u;
  const bool chunked = C > 1;
  if (chunked) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  MOE_STAMP(R, 1, 0);

  // pair_start: exclusive message prefix over pairs (e_loc, src) -- chunked,
  // over (chunk, pair) in chunk-major order (C * P <= kMaxExperts)
  __shared__ uint32_t cnt[kMaxExperts], pair_start[kMaxExperts + 1], src_prefix[kMaxExperts];
  __shared__ uint32_t csrc[kCombineChunks * GIN_MAX_RANKS];  // chunked: messages of (chunk, source)
  __shared__ uint32_t warp_tot[kMoeWarps];
  __shared__ uint32_t total_msgs;
  __shared__ int is_last;
  extern __shared__ __align__(128) char dsm[];
  TmaSmem* ctl = reinterpret_cast<TmaSmem*>(dsm) + warp;
  // per stage: [128-byte header: the message's 16-byte meta][chunk]
  //   mode 2: [header][scales chunk/64][bf16 output chunk], the e4m3 codes
  //     bulk-loaded into the back half of the output buffer (every lane holds
  //     its codes in registers before any output is written)
  //   mode 3: [header][e4m3 chunk/2][scales in chunk/64][scales out chunk/64],
  //     re-quantized in place in registers (no bf16 staging)
  const uint32_t sc_bytes = ((chunk / 64) + 15) & ~15u;
  const uint32_t q_off = fp8c ? 128 : 128 + sc_bytes + chunk / 2;  // e4m3 codes
  const uint32_t s_off = fp8c ? 128 + chunk / 2 : 128;             // scales in
  const uint32_t o_off = fp8c ? 0 : (fp8 ? 128 + sc_bytes : 128);  // bf16 output (modes 0-2)
  const uint32_t os_off = 128 + chunk / 2 + sc_bytes;              // scales out (mode 3)
  const uint32_t sstride = fp8c ? os_off + sc_bytes : (fp8 ? o_off + chunk : 128 + chunk);
  char* stage = dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)warp * kTmaStages * sstride;

  const uint32_t P = e_local * n;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
  // chunked: btab[(c-1)*P + pair] = first slot of chunk c (c = 1..C-1) in the
  // pair's run, from the dispatch's bounds (after the stage buffers)
  uint32_t* btab = reinterpret_cast<uint32_t*>(dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) +
                                               (size_t)kTmaWarps * kTmaStages * sstride);
  for (uint32_t i = tid; i < P; i += kTmaThreads) {
    const uint32_t c = gin::ld_acquire_sys32(counts + count_index(i, n, e_local));
    cnt[i] = c;
    pair_start[i] = c;
  }
  for (uint32_t i = tid; chunked && i < (C - 1) * P; i += kTmaThreads) {
    const uint32_t c = 1 + i / P, pr = i % P, e_loc = pr / n, src = pr % n;
    btab[i] = gin::ld_acquire_sys32(counts + combine_bounds_index(n, e_local, src, c, C) + e_loc);
  }
  if (tid < kMoeWarps) warp_tot[tid] = 0;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) gin::tma::mbar_init(&ctl->bar[s], 1);
    gin::tma::fence_mbar_init();
  }
  __syncthreads();
  if (L.layout != 0) source_prefix<kTmaWarps>(cnt, src_prefix, n, e_local);
  const uint32_t NP = chunked ? C * P : P;  // entries of the work prefix
  if (chunked) {
    for (uint32_t i = tid; i < NP; i += kTmaThreads) {
      const uint32_t c = i / P, pr = i % P;
      const uint32_t lo = c == 0 ? 0u : btab[(c - 1) * P + pr], hi = c + 1 == C ? cnt[pr] : btab[c * P + pr];
      pair_start[i] = hi - lo;
    }
    for (uint32_t i = warp; i < C * n; i += kTmaWarps) {  // one warp per (chunk, source)
      const uint32_t c = i / n, src = i % n;
      uint32_t m = 0;
      for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32) {
        const uint32_t pr = e_loc * n + src;
        m += (c + 1 == C ? cnt[pr] : btab[c * P + pr]) - (c == 0 ? 0u : btab[(c - 1) * P + pr]);
      }
      m = __reduce_add_sync(0xffffffffu, m);
      if (lane == 0) csrc[i] = m;
    }
    __syncthreads();
  }
  // exclusive scan of NP <= 1024 entries with 512 threads (2 per thread)
  {
    const uint32_t per = (NP + kTmaThreads - 1) / kTmaThreads;
    const uint32_t lo = tid * per, hi = min(lo + per, NP);
    uint32_t local = 0;
    for (uint32_t i = lo; i < hi; ++i) local += pair_start[i];
    uint32_t incl = local;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (tid == 0) {
      uint32_t acc = 0;
      for (int w = 0; w < kTmaWarps; ++w) {
        const uint32_t x = warp_tot[w];
        warp_tot[w] = acc;
        acc += x;
      }
      total_msgs = acc;
    }
    __syncthreads();
    uint32_t r = warp_tot[warp] + incl - local;
    for (uint32_t i = lo; i < hi; ++i) {
      const uint32_t d = pair_start[i];
      pair_start[i] = r;
      r += d;
    }
    __syncthreads();
    if (tid == 0) pair_start[NP] = total_msgs;
    __syncthreads();
  }

  MOE_STAMP(R, 1, 1);
  const char* recv = v->win[L.win_dispatch].base[rank];
  char* const* cbases = v->win[L.win_combine].base;
  const uint64_t items = (uint64_t)total_msgs * parts;
  const uint64_t gw = (uint64_t)b * kTmaWarps + warp, stride = (uint64_t)G * kTmaWarps;
  // message m of the work order -> its pair (| chunk << 16) and address
  auto locate = [&](uint32_t m, uint32_t& lo_pair) -> const char* {
    uint32_t lo = 0, hi = NP;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pair_start[mid] <= m) lo = mid; else hi = mid;
    }
    const uint32_t ch = lo / P, pr = lo % P;
    lo_pair = pr | (ch << 16);
    const uint32_t e_loc = pr / n, src = pr % n;
    const uint32_t slot = (ch == 0 ? 0u : btab[(ch - 1) * P + pr]) + (m - pair_start[lo]);
    const uint64_t moff = L.layout == 0 ? (((uint64_t)e_loc * n + src) * T + slot) * dmsg
                                        : ((uint64_t)src * T * K + src_prefix[pr] + slot) * dmsg;
    return recv + moff;
  };
  // lane 0: locate the message once, record (expert, source) for the stage and
  // bulk-load the chunk AND the message's 16-byte meta onto one mbarrier, so
  // no lane ever waits on a global load of its own
  auto issue_load = [&](int s, uint64_t it) {
    uint32_t pr;
    const char* msg = locate((uint32_t)(it / parts), pr);
    const uint32_t p = (uint32_t)(it % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    ctl->dptr[s] = reinterpret_cast<char*>((uint64_t)pr);  // pair index of the stage's message
    if (fp8) {  // the chunk's e4m3 codes and their block scales
      gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len / 2 + len / 64 + 16);
      gin::tma::load(sb, msg + L.mpay, 16, &ctl->bar[s]);
      gin::tma::load(sb + q_off, msg + (uint64_t)p * (chunk / 2), len / 2, &ctl->bar[s]);
      gin::tma::load(sb + s_off, msg + H + (uint64_t)p * (chunk / 64), len / 64, &ctl->bar[s]);
    } else {
      gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + 16);
      gin::tma::load(sb, msg + L.mpay, 16, &ctl->bar[s]);
      gin::tma::load(sb + 128, msg + (uint64_t)p * chunk, len, &ctl->bar[s]);
    }
  };
  // Work source.  Static: warp gw takes items gw, gw+stride, ...  Dynamic
  // (L.dyn): warps grab batches of one message's parts from a device counter,
  // so CTAs whose messages go to slower (remote) destinations take fewer
  // and the kernel has no straggler tail; the last CTA resets the counter.
  unsigned long long* grab_ctr = reinterpret_cast<unsigned long long*>(R.ws + 8);
  auto next_item = [&]() -> uint64_t {  // lane 0 only
    uint64_t it;
    if (L.dyn && ctl->cur >= kTmaStages) {  // one message per grab after the interleaved first round
      if (ctl->end == 0 || ctl->itc >= ctl->end) {
        ctl->itc = (uint64_t)kTmaStages * stride + atomicAdd(grab_ctr, (unsigned long long)parts);
        ctl->end = ctl->itc + parts;
      }
      it = ctl->itc++;
    } else {
      it = gw + (ctl->cur++) * stride;
    }
    return it < items ? it : kNoItem;
  };
  // chunked: a chunk is complete once all its items' stores completed (per
  // chunk arrival counter in items, ws[64 + c], reset by the completing warp
  // for the next launch); that warp releases the chunk at every source by the
  // messages it holds from there (GPU scope toward its own tokens)
  uint32_t cur_ch = 0xFFFFFFFFu, cur_n = 0;  // lane 0
  auto chunk_arrive = [&](uint32_t c, uint32_t nitems) {
    gin::tma::fence_proxy_async_global();
    gin::fence_acq_rel_gpu();
    const unsigned total = (pair_start[(c + 1) * P] - pair_start[c * P]) * parts;
    const unsigned prev = atomicAdd(R.ws + 64 + c, nitems);
    if (prev + nitems == total) {
      gin::fence_acq_rel_gpu();
      R.ws[64 + c] = 0;
      const uint32_t cell = combine_chunk_cell(L.cell0, e_local, c);
      for (uint32_t src = 0; src < n; ++src) {
        const uint32_t m = csrc[c * n + src];
        if (!m) continue;
        if (src == rank) gin::red_relaxed_sys_add(gin.sub_cell(src, rank, cell), m);
        else gin.release_signal_raw(src, cell, m);
      }
    }
  };
  if (lane == 0) {
    ctl->cur = 0;
    ctl->end = 0;
    for (int s = 0; s < kTmaStages; ++s) {
      const uint64_t it = next_item();
      ctl->itm[s] = it;
      if (it != kNoItem) issue_load(s, it);
    }
  }
  __syncwarp();
  for (uint64_t j = 0;; ++j) {
    const int s = (int)(j % kTmaStages);
    const uint64_t it = ctl->itm[s];
    if (it == kNoItem) break;
    const uint32_t p = (uint32_t)(it % parts);
    const uint32_t packed = (uint32_t)reinterpret_cast<uint64_t>(ctl->dptr[s]);
    const uint32_t pr = packed & 0xFFFFu, ch = packed >> 16;
    const uint32_t e = rank * e_local + pr / n, src = pr % n;
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_wait(&ctl->bar[s], (uint32_t)((j / kTmaStages) & 1));
    uint4* buf = reinterpret_cast<uint4*>(sb + o_off);
    {
      const uint32_t nv = len / 16;
      uint32_t i = lane;
      if (fp8c) {  // dequant -> transform -> bf16 -> re-quantize, 8 lanes per 128-element block
        const float sc = 1.0f + (float)(e % 7u) / 8.0f, cc = ((float)(e % 9u) - 4.0f) / 16.0f;
        const float* scl = reinterpret_cast<const float*>(sb + s_off);
        float* sco = reinterpret_cast<float*>(sb + os_off);
        const uint32_t grp = lane >> 3, sub8 = lane & 7;
        for (uint32_t blk0 = 0; blk0 < len / 256; blk0 += 4) {  // len is a multiple of 1024: 4 blocks per step
          const uint32_t blk = blk0 + grp;
          uint4* cp = reinterpret_cast<uint4*>(sb + q_off + blk * 128 + sub8 * 16);
          const uint4 codes = *cp;
          fp8_requant16(cp, codes, scl[blk], sc, cc, sco + blk, sub8);
        }
      } else if (fp8) {  // expand: 8 codes -> one 16-byte bf16 vector; scale per 128 elements
        const float sc = 1.0f + (float)(e % 7u) / 8.0f, cc = ((float)(e % 9u) - 4.0f) / 16.0f;
        const uint2* qin = reinterpret_cast<const uint2*>(sb + q_off);
        const float* scl = reinterpret_cast<const float*>(sb + s_off);
        uint2 q[kFp8MaxVec];  // the codes share the output buffer: read them all first
#pragma unroll
        for (int m = 0; m < kFp8MaxVec; ++m)
          if (i + 32 * m < nv) q[m] = qin[i + 32 * m];
        __syncwarp();
#pragma unroll
        for (int m = 0; m < kFp8MaxVec; ++m)
          if (i + 32 * m < nv) buf[i + 32 * m] = fp8x8_transform(q[m], scl[(i + 32 * m) / 16], sc, cc);
      } else if (L.mode == 0) {
        const uint32_t add = (e * 17u + 1u) & 0xFFFFu;
        for (; i < nv; i += 32) {
          uint4 a = buf[i];
          a.x = u16x2_transform(a.x, add), a.y = u16x2_transform(a.y, add);
          a.z = u16x2_transform(a.z, add), a.w = u16x2_transform(a.w, add);
          buf[i] = a;
        }
      } else {
        const float sc = 1.0f + (float)(e % 7u) / 8.0f, cc = ((float)(e % 9u) - 4.0f) / 16.0f;
        for (; i + 32 < nv; i += 64) {  // 2 independent vectors per lane in flight
          const uint4 a = buf[i], c = buf[i + 32];
          buf[i] = bf16x8_transform(a, sc, cc);
          buf[i + 32] = bf16x8_transform(c, sc, cc);
        }
        for (; i < nv; i += 32) buf[i] = bf16x8_transform(buf[i], sc, cc);
      }
    }
    gin::tma::fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) {
      const uint4 meta = *reinterpret_cast<const uint4*>(sb);  // {src, token, k, tag}
      char* cdst = cbases[src] + ((uint64_t)meta.y * K + meta.z) * cmsg;
      if (fp8c) {
        gin::tma::store(cdst + (uint64_t)p * (chunk / 2), sb + q_off, len / 2);
        gin::tma::store(cdst + H + (uint64_t)p * (chunk / 64), sb + os_off, len / 64);
      } else {
        gin::tma::store(cdst + (uint64_t)p * chunk, buf, len);
      }
      gin::tma::commit();
      if (chunked) {
        // first item of a later chunk: once every older bulk group completed
        // (this item's stores stay in flight), count the warp's items of the
        // previous chunk in (items arrive in increasing order, so chunks too)
        if (cur_ch != ch) {
          if (cur_ch != 0xFFFFFFFFu) {
            gin::tma::wait_done<1>();
            chunk_arrive(cur_ch, cur_n);
          }
          cur_ch = ch;
          cur_n = 0;
        }
        ++cur_n;
      }
      if (j >= 1) {  // refill the previous item's stage (its store has been reading meanwhile)
        gin::tma::wait_read<1>();
        const int ps = (int)((j - 1) % kTmaStages);
        const uint64_t nxt = next_item();
        ctl->itm[ps] = nxt;
        if (nxt != kNoItem) issue_load(ps, nxt);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    gin::tma::wait_all();
    gin::tma::fence_proxy_async_global();
    if (chunked && cur_ch != 0xFFFFFFFFu) chunk_arrive(cur_ch, cur_n);
  }
  MOE_STAMP(R, 1, 2);

  arrive_last(R.ws + 1, (unsigned)(iteration * G), &is_last);
  if (is_last) {
    if (tid == 0) *grab_ctr = 0;  // every CTA is past its loop: ready for the next launch
    if (tid == 0) *moe_iter_ptr(R, 1) = iteration;  // every CTA has read it (arrival)
    for (uint32_t sc = tid; sc < n * n_ctx; sc += kTmaThreads) {
      const uint32_t src = sc / n_ctx, ctx = sc % n_ctx;
      uint32_t c = 0;
      for (uint32_t e_loc = 0; e_loc < e_local; ++e_loc)
        if ((rank * e_local + e_loc) % n_ctx == ctx) c += cnt[e_loc * n + src];
      if (c) {
        if (src == rank) {  // own tokens: the reducer is on this GPU
          gin::fence_acq_rel_gpu();
          gin::red_relaxed_sys_add(gin.sub_cell(src, rank, L.cell0 + e_local), c);
        } else {
          gin.release_signal_raw(src, L.cell0 + e_local, c);
        }
      }
    }
  }
  MOE_STAMP(R, 1, 3);
  if (L.fuse_reduce) {
    // small launches: the source-side reduction right here (saves the second
    // launch); same arithmetic as moe_combine_reduce_kernel
    if (tid == 0) gin.wait_ge_signal(L.cell0 + e_local, iteration * (uint64_t)T * K);
    __syncthreads();
    const char* crecv = v->win[L.win_combine].base[rank];
    const uint32_t nvec = payload / 16;
    const uint64_t ritems = (uint64_t)T * nvec, rstride = (uint64_t)G * kTmaThreads;
    for (uint64_t q = (uint64_t)b * kTmaThreads + tid; q < ritems; q += rstride) {
      const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
      uint4 y[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < (int)K && !fp8c) y[k] = gin::ld_na_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i);
      gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
                 fp8c ? reduce_fp8_vec<KMAX>(crecv, cmsg, H, t, i, K, R.weights)
                      : reduce_vec<KMAX>(y, K, L.mode, R.weights, t));
    }
  }
}

// Source side of the combine, split off the TMA send kernel so it runs at
// full occupancy (32 warps/SM; the TMA kernel holds 1 CTA/SM for its staging
// buffers): acquire the combine flag (>= T*K per iteration, harness_moe.cpp:
// 227) then the top-k weighted reduction, two 16-byte vectors per thread with
// all 2K loads in flight before any use.  No CTA waits on another CTA of
// this launch, so it needs no co-residency.  MIRROR (Proxy pipeline): the
// results arrived in the mirror window in send order; y is gathered through
// the dispatch's (t, k) -> mirror index and also written to (t*K+k)*cmsg, so
// the combine window ends as the reference's (harness_moe.cpp:203-205).
template <int KMAX, bool FP8C, bool MIRROR>
__global__ void __launch_bounds__(kMoeThreads, 2) moe_combine_reduce_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 1, false);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t rank = v->rank;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const uint64_t cmsg = L.cmsg;
  constexpr bool fp8c = FP8C;  // mode 3 (a separate instantiation keeps the bf16 path spill-free)
  const uint32_t payload = 2u * H;
  MOE_STAMP(R, 2, 0);
  const uint32_t nvec = payload / 16;
  if (L.share && !MIRROR && !fp8c) {
    // Emulated ranks: CTAs take chunks of kRedChunk tokens of ANY lane from a
    // launch-wide counter (lane 0's workspace, one per iteration parity; the
    // next parity's is zeroed here -- nobody uses it before this kernel ends),
    // so the lanes finish together.  A CTA acquires a lane's combine flag the
    // first time it takes a chunk of that lane.
    constexpr uint32_t kRedChunk = 4;
    const uint32_t nl = gridDim.y;
    unsigned int* ctr = L.r[0].ws + 46 + (uint32_t)(iteration & 1);
    if (b == 0 && blockIdx.y == 0 && tid == 0) L.r[0].ws[46 + (uint32_t)((iteration + 1) & 1)] = 0;
    const uint32_t chunks_per_lane = (T + kRedChunk - 1) / kRedChunk, total = chunks_per_lane * nl;
    __shared__ uint32_t s_chunk, s_acquired;
    if (tid == 0) s_acquired = 0;
    for (;;) {
      __syncthreads();
      if (tid == 0) {
        s_chunk = atomicAdd(ctr, 1u);
        const uint32_t ln = s_chunk % nl;
        if (s_chunk < total && !((s_acquired >> ln) & 1u)) {
          const MoeRankArgs& Rl = L.r[ln];
          gin::Gin gl(Rl.view, 0);
          gl.wait_ge_signal(L.cell0 + e_local, iteration * (uint64_t)T * K);
          s_acquired |= 1u << ln;
        }
      }
      __syncthreads();
      const uint32_t c = s_chunk;
      if (c >= total) break;
      const uint32_t ln = c % nl, tb = (c / nl) * kRedChunk;
      const MoeRankArgs& Rl = L.r[ln];
      const GinDevCommView* vl = Rl.view;
      const char* crl = vl->win[L.win_combine].base[vl->rank];
      const uint32_t te = min(T, tb + kRedChunk);
      for (uint64_t q = (uint64_t)tb * nvec + tid; q < (uint64_t)te * nvec; q += kMoeThreads) {
        const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
        uint4 y[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < (int)K) y[k] = gin::ld_na_v4(crl + ((uint64_t)t * K + k) * cmsg + 16ull * i);
        gin::st_v4(reinterpret_cast<char*>(Rl.out) + (uint64_t)t * payload + 16ull * i,
                   reduce_vec<KMAX>(y, K, L.mode, Rl.weights, t));
      }
    }
    MOE_STAMP(R, 2, 1);
    MOE_STAMP(R, 2, 2);
    return;
  }
  const char* crecv = v->win[L.win_combine].base[rank];
  const uint32_t nthr = blockDim.x;
  const uint64_t rstride = (uint64_t)G * nthr;
  if (L.cchunks > 1 && !MIRROR) {
    // pipelined combine: chunks [red_first, red_last) in order, each once its
    // cell holds every expert rank's messages for the chunk's tokens.  The
    // iteration is the dispatch's: this grid may start before the send
    // kernel (whose combine counter it would otherwise read) has finished.
    const uint32_t C = L.cchunks;
    const uint64_t it0 = moe_iteration(R, 0, false);
    // phase stamps of the early reducer: CTA slots 512+ of the reduce table
    const bool early = L.red_first == 0 && L.red_last < C;
    auto estamp = [&](int slot) {
      if (early && R.prof && tid == 0 && b < 512) R.prof[((uint64_t)2 * 1024 + 512 + b) * 8 + slot] = gin::globaltimer();
    };
    estamp(0);
    for (uint32_t c = L.red_first; c < L.red_last; ++c) {
      const uint32_t ta = combine_chunk_t0(c, C, L.dgrid, T), tb = combine_chunk_t0(c + 1, C, L.dgrid, T);
      if (tid == 0) gin.wait_ge_signal(combine_chunk_cell(L.cell0, e_local, c), it0 * (uint64_t)(tb - ta) * K);
      __syncthreads();
      for (uint64_t q = (uint64_t)ta * nvec + (uint64_t)b * nthr + tid; q < (uint64_t)tb * nvec; q += rstride) {
        const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
        if (fp8c) {
          gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
                     reduce_fp8_vec<KMAX>(crecv, cmsg, H, t, i, K, R.weights));
          continue;
        }
        uint4 y[KMAX];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < (int)K) y[k] = gin::ld_na_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i);
        gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
                   reduce_vec<KMAX>(y, K, L.mode, R.weights, t));
      }
      estamp(1 + (int)c);
    }
    if (early) {
      estamp(6);
      asm volatile("griddepcontrol.wait;" ::: "memory");
      estamp(7);
      return;
    }
    MOE_STAMP(R, 2, 1);
    // the send grid has completed before this one does (stream order for the
    // next launch; a no-op when launched without the programmatic attribute)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    MOE_STAMP(R, 2, 2);
    return;
  }
  if (tid == 0) gin.wait_ge_signal(L.cell0 + e_local, iteration * (uint64_t)T * K);
  __syncthreads();
  MOE_STAMP(R, 2, 1);
  const uint64_t ritems = (uint64_t)T * nvec;
  for (uint64_t q = (uint64_t)b * nthr + tid; q < ritems; q += rstride) {
    const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
    if (fp8c) {
      gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
                 reduce_fp8_vec<KMAX>(crecv, cmsg, H, t, i, K, R.weights));
      continue;
    }
    uint4 y[KMAX];
    if (MIRROR) {
      const char* mirror = v->win[L.win_mirror].base[rank];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < (int)K) y[k] = gin::ld_na_v4(mirror + (uint64_t)__ldg(R.midx + (uint64_t)t * K + k) * cmsg + 16ull * i);
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < (int)K) gin::st_v4(const_cast<char*>(crecv) + ((uint64_t)t * K + k) * cmsg + 16ull * i, y[k]);
    } else {
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < (int)K) y[k] = gin::ld_na_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i);
    }
    gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
               reduce_vec<KMAX>(y, K, L.mode, R.weights, t));
  }
  MOE_STAMP(R, 2, 2);
}

}  // namespace ginsim_b200
