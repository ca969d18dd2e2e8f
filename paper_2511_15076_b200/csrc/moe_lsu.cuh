// moe_lsu.cuh -- LSU-engine dispatch/combine kernels and their Proxy-backend variants.
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
#pragma once

namespace ginsim_b200 {

// PROXY = the Proxy backend: rows are staged into a local
// registered window laid out in destination order -- (dst_base[dst] +
// prefix_e[e] + slot) -- so every expert's messages form ONE contiguous run
// at both ends, and the last CTA hands each run to the host agent as a put
// descriptor (ordered before the expert's release on ctx e % n_ctx,
// harness_moe.cpp:135-167).  No NVLink store is issued by the kernel.
template <int KMAX, bool PROXY>
__global__ void __launch_bounds__(kMoeThreads, KMAX <= 8 ? 2 : 1) moe_dispatch_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 0, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank;
  const uint32_t E = L.E, K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = 2ull * H + 16;
  const uint32_t t0 = (uint32_t)((uint64_t)b * T / G), t1 = (uint32_t)((uint64_t)(b + 1) * T / G);

  __shared__ uint32_t hist_all[kMaxExperts], run[kMaxExperts], prefix_e[kMaxExperts];
  __shared__ uint32_t dst_base[GIN_MAX_RANKS + 1];
  __shared__ int is_last;
  extern __shared__ uint32_t slots[];  // [(t1-t0)*K]

  for (uint32_t e = tid; e < E; e += kMoeThreads) {
    hist_all[e] = 0;
    run[e] = 0;
  }
  if (PROXY && tid == 0) {
    // flush (runtime.cpp:460-470): the staging window is reused only once the
    // host agent has completed every put this rank submitted earlier
    for (uint32_t ctx = 0; ctx < v->n_ctx; ++ctx) {
      const uint64_t snap = atomicAdd(&v->proxy.tickets[ctx], 0ull);
      gin::Gin(v, ctx).wait_ge(&v->proxy.completed[ctx], snap);
    }
  }
  __syncthreads();
  // Phase A: per-expert totals and the prefix of tokens before this CTA.
  const uint32_t TK = T * K, pre_end = t0 * K;
  histogram_pass<kMoeThreads>(R.idx, TK, pre_end, 0, hist_all, run, nullptr);
  __syncthreads();
  // Destination base offsets for the compact layout: exclusive prefix of this
  // source's counts within each destination's expert group.
  if (L.layout != 0 || PROXY) {
    for (uint32_t d = tid; d < n; d += kMoeThreads) {
      uint32_t acc = 0;
      for (uint32_t e = d * e_local; e < (d + 1) * e_local; ++e) {
        prefix_e[e] = acc;
        acc += hist_all[e];
      }
      dst_base[d + 1] = acc;  // messages to d (turned into a prefix below)
    }
  }
  if (PROXY) {
    __syncthreads();
    if (tid == 0) {
      dst_base[0] = 0;
      for (uint32_t d = 0; d < n; ++d) dst_base[d + 1] += dst_base[d];
    }
  }
  // Slots of this CTA's tokens, in (t, k) order (harness_moe.cpp:143-150).
  if (warp == 0) {
    for (uint32_t t = t0; t < t1; ++t) {
      if (lane < K) {
        const uint32_t e = (uint32_t)R.idx[(uint64_t)t * K + lane];
        const uint32_t s = run[e];
        run[e] = s + 1;  // experts of one token are distinct
        slots[(t - t0) * K + lane] = s;
        // proxy: where (t, k)'s combine result lands in this rank's mirror
        // window -- the send order [dst][expert prefix][slot]
        if (PROXY) R.midx[(uint64_t)t * K + lane] = (e / e_local) * T * K + prefix_e[e] + s;
      }
      __syncwarp();
    }
  }
  __syncthreads();

  // Phase B: (token, part) work items, one warp each.
  const uint32_t parts = L.parts;
  const uint32_t payload = 2u * H;
  const bool vec_ok = (payload % 16u) == 0;
  const uint32_t nvec = payload / 16u;
  const uint32_t vec_per_part = (nvec + parts - 1) / parts;
  char* const* bases = v->win[L.win_dispatch].base;
  const uint32_t items = (t1 - t0) * parts;
  for (uint32_t it = warp; it < items; it += kMoeWarps) {
    const uint32_t t = t0 + it / parts, p = it % parts;
    // lane k < K: destination of message (t, k)
    char* my_dst = nullptr;
    if (lane < K) {
      const uint32_t e = (uint32_t)R.idx[(uint64_t)t * K + lane];
      const uint32_t dst = e / e_local, e_loc = e % e_local;
      const uint32_t slot = slots[(t - t0) * K + lane];
      if (PROXY && dst != rank) {
        my_dst = v->win[L.win_stage].base[rank] + ((uint64_t)dst_base[dst] + prefix_e[e] + slot) * dmsg;
      } else {
        const uint64_t off = L.layout == 0 ? (((uint64_t)e_loc * n + rank) * T + slot) * dmsg
                                           : ((uint64_t)rank * T * K + prefix_e[e] + slot) * dmsg;
        my_dst = bases[dst] + off;
      }
    }
    char* dptr[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k) dptr[k] = (char*)__shfl_sync(0xffffffffu, (uintptr_t)my_dst, k < 32 ? k : 0);
    const char* src = reinterpret_cast<const char*>(R.x) + (uint64_t)t * payload;
    if (vec_ok) {
      const uint32_t vlo = p * vec_per_part, vhi = min(vlo + vec_per_part, nvec);
      uint32_t i = vlo + lane;
      for (; i + 96 < vhi; i += 128) {
        const uint4 a = gin::ld_nc_v4(src + 16ull * i), bb = gin::ld_nc_v4(src + 16ull * (i + 32));
        const uint4 c = gin::ld_nc_v4(src + 16ull * (i + 64)), d = gin::ld_nc_v4(src + 16ull * (i + 96));
#pragma unroll
        for (int k = 0; k < KMAX; ++k) {
          if (k < (int)K) {
            gin::st_v4(dptr[k] + 16ull * i, a);
            gin::st_v4(dptr[k] + 16ull * (i + 32), bb);
            gin::st_v4(dptr[k] + 16ull * (i + 64), c);
            gin::st_v4(dptr[k] + 16ull * (i + 96), d);
          }
        }
      }
      for (; i < vhi; i += 32) {
        const uint4 a = gin::ld_nc_v4(src + 16ull * i);
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < (int)K) gin::st_v4(dptr[k] + 16ull * i, a);
      }
    } else if (p == 0) {
      for (uint32_t j = lane; j < payload; j += 32) {
        const char byte = src[j];
#pragma unroll
        for (int k = 0; k < KMAX; ++k)
          if (k < (int)K) dptr[k][j] = byte;
      }
    }
    if (p == 0 && lane < K) {  // meta {src, token, k, tag = k+1}
      char* m = my_dst + payload;
      if ((((uintptr_t)m) & 15) == 0) {
        gin::st_v4(m, make_uint4(rank, t, lane, lane + 1));
      } else {
        const uint32_t w[4] = {rank, t, lane, lane + 1};
        for (int q = 0; q < 16; ++q) m[q] = (char)(w[q >> 2] >> (8 * (q & 3)));
      }
    }
  }

  // Phase C: the last CTA to finish releases every expert.
  arrive_last(R.ws + 0, (unsigned)(iteration * G), &is_last);
  if (is_last && tid == 0) *moe_iter_ptr(R, 0) = iteration;  // every CTA has read it (arrival)
  if (is_last && PROXY) {
    // Three phases, each fully submitted before the next (CTA barrier), so on
    // every context ring all counts precede all payload puts, which precede
    // all releases: a release lands after its expert's payload (the agent
    // drains a ring in ticket order onto one stream, fabric.cpp:63-79).
    //   coalesce: every op of destination d goes on ctx d % n_ctx, and with
    //     the compact layout all of d's experts form ONE contiguous run at
    //     both ends (staging [dst_base][prefix][slot] == d's window
    //     [src][prefix][slot]) -> one copy-engine transfer per destination;
    //     with the reference layout one run per expert.
    //   reference pattern (GINSIM_PROXY_COALESCE=0): ctx e % n_ctx and one
    //     put per (t, k) message (harness_moe.cpp:135-167).
    // Own experts' rows were written in place by the SMs (a same-device copy
    // by the agent would need SMs this kernel holds): counts and releases only.
    const gin::Team world = gin::WorldTeam(n);
    gin::CoopThread me;
    auto ctx_of = [&](uint32_t e) { return L.coalesce ? (e / e_local) % v->n_ctx : e % v->n_ctx; };
    for (uint32_t e = tid; e < E; e += kMoeThreads) {
      const uint32_t dst = e / e_local, e_loc = e % e_local;
      gin::Gin(v, ctx_of(e)).put_value(me, world, dst, L.win_counts, ((uint64_t)rank * e_local + e_loc) * 4, hist_all[e]);
    }
    __syncthreads();
    if (L.coalesce && L.layout != 0) {
      for (uint32_t d = tid; d < n; d += kMoeThreads) {
        const uint32_t tot = dst_base[d + 1] - dst_base[d];
        if (d == rank || tot == 0) continue;
        gin::Gin(v, d % v->n_ctx).put(me, world, d, L.win_dispatch, (uint64_t)rank * T * K * dmsg, L.win_stage,
                                       (uint64_t)dst_base[d] * dmsg, (uint64_t)tot * dmsg);
      }
    } else {
      for (uint32_t e = tid; e < E; e += kMoeThreads) {
        const uint32_t dst = e / e_local, e_loc = e % e_local, cnt = hist_all[e];
        if (dst == rank || cnt == 0) continue;
        const gin::Gin g(v, ctx_of(e));
        const uint64_t src0 = ((uint64_t)dst_base[dst] + prefix_e[e]) * dmsg;
        const uint64_t dst0 = L.layout == 0 ? (((uint64_t)e_loc * n + rank) * T) * dmsg
                                            : ((uint64_t)rank * T * K + prefix_e[e]) * dmsg;
        if (L.coalesce) {
          g.put(me, world, dst, L.win_dispatch, dst0, L.win_stage, src0, (uint64_t)cnt * dmsg);
        } else {
          for (uint32_t q = 0; q < cnt; ++q)
            g.put(me, world, dst, L.win_dispatch, dst0 + q * dmsg, L.win_stage, src0 + q * dmsg, dmsg);
        }
      }
    }
    __syncthreads();
    for (uint32_t e = tid; e < E; e += kMoeThreads) {
      const uint32_t dst = e / e_local, e_loc = e % e_local;
      gin::Gin(v, ctx_of(e)).signal(me, world, dst, L.cell0 + e_loc, gin::SignalAdd((1ull << 32) + hist_all[e]));
    }
  } else if (is_last) {
    release_experts(gin, v, L.win_counts, hist_all, n, rank, e_local, L.cell0);
  }
  // Phase D: return once every local expert has been released by every source.
  if (tid == 0)
    for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) acquire_expert_cell(gin, R, L.cell0 + e_loc, e_loc, iteration, n);
}

// ------------------------------------------------------------------ combine
// PROXY: the expert transform writes message m (receive order) to m*cmsg of
// the local staging window, then the last CTA submits one put descriptor per message
// to (token*K+k)*cmsg of its source and, after them on the same context, the
// per-(source, ctx) combine flag (harness_moe.cpp:169-223).
template <bool PROXY>
__global__ void __launch_bounds__(kMoeThreads, 2) moe_combine_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const uint64_t iteration = moe_iteration(R, 1, true);
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = 2ull * H + 16, cmsg = 2ull * H;
  const uint32_t payload = 2u * H;

  __shared__ uint32_t cnt[kMaxExperts], pair_start[kMaxExperts + 1], src_prefix[kMaxExperts];
  __shared__ uint32_t warp_tot[kMoeWarps];
  __shared__ uint32_t total_msgs;
  __shared__ int is_last;

  // Received counts: pair (e_loc, src) in e_loc-major order (reference scan
  // order, harness_moe.cpp:174-179).
  const uint32_t P = e_local * n;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
  for (uint32_t i = tid; i < P; i += kMoeThreads) {
    const uint32_t c = gin::ld_acquire_sys32(counts + count_index(i, n, e_local));
    cnt[i] = c;
    pair_start[i] = c;
  }
  __syncthreads();
  // (the proxy mirror needs the per-source expert prefix in both layouts)
  if (L.layout != 0 || PROXY) source_prefix<kMoeWarps>(cnt, src_prefix, n, e_local);
  // proxy + coalesce: the staging window holds results source-major
  // ([src_base[s] + src_prefix + slot]) so all of a source's results are one
  // contiguous run at both ends (its mirror region is [rank*T*K + prefix + slot])
  __shared__ uint32_t src_base[GIN_MAX_RANKS + 1];
  if (PROXY) {
    __syncthreads();
    if (tid == 0) {
      src_base[0] = 0;
      for (uint32_t sidx = 0; sidx < n; ++sidx)
        src_base[sidx + 1] = src_base[sidx] + src_prefix[(e_local - 1) * n + sidx] + cnt[(e_local - 1) * n + sidx];
    }
  }
  block_exclusive_scan(pair_start, P, warp_tot, &total_msgs);
  if (tid == 0) pair_start[P] = total_msgs;
  __syncthreads();

  // Expert side: (message, part) items over every warp of this rank.
  const uint32_t parts = L.parts;
  const bool vec_ok = (payload % 16u) == 0;
  const uint32_t nvec = payload / 16u;
  const uint32_t vec_per_part = (nvec + parts - 1) / parts;
  const uint64_t items = (uint64_t)total_msgs * parts;
  const char* recv = v->win[L.win_dispatch].base[rank];
  char* const* cbases = v->win[L.win_combine].base;
  for (uint64_t it = (uint64_t)b * kMoeWarps + warp; it < items; it += (uint64_t)G * kMoeWarps) {
    const uint32_t m = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    // pair containing m: last i with pair_start[i] <= m
    uint32_t lo = 0, hi = P;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pair_start[mid] <= m) lo = mid; else hi = mid;
    }
    const uint32_t e_loc = lo / n, src = lo % n, slot = m - pair_start[lo];
    const uint64_t moff = L.layout == 0 ? (((uint64_t)e_loc * n + src) * T + slot) * dmsg
                                        : ((uint64_t)src * T * K + src_prefix[lo] + slot) * dmsg;
    const char* msg = recv + moff;
    const unsigned char* meta = reinterpret_cast<const unsigned char*>(msg + payload);
    uint32_t token, k;
    if ((((uintptr_t)meta) & 3) == 0) {
      token = reinterpret_cast<const uint32_t*>(meta)[1];
      k = reinterpret_cast<const uint32_t*>(meta)[2];
    } else {
      token = meta[4] | (meta[5] << 8) | (meta[6] << 16) | ((uint32_t)meta[7] << 24);
      k = meta[8] | (meta[9] << 8) | (meta[10] << 16) | ((uint32_t)meta[11] << 24);
    }
    const uint32_t e = rank * e_local + e_loc;
    char* dst;
    if (!PROXY) {
      dst = cbases[src] + ((uint64_t)token * K + k) * cmsg;
    } else if (src != rank) {  // staged for the agent
      dst = v->win[L.win_cstage].base[rank] +
            (L.coalesce ? (uint64_t)src_base[src] + src_prefix[lo] + slot : (uint64_t)m) * cmsg;
    } else if (L.coalesce) {  // own tokens: straight into this rank's mirror window
      dst = v->win[L.win_mirror].base[rank] + ((uint64_t)rank * T * K + src_prefix[lo] + slot) * cmsg;
    } else {
      dst = cbases[src] + ((uint64_t)token * K + k) * cmsg;
    }
    if (vec_ok) {
      const uint32_t vlo = p * vec_per_part, vhi = min(vlo + vec_per_part, nvec);
      uint32_t i = vlo + lane;
      for (; i + 96 < vhi; i += 128) {
        uint4 a = gin::ld_nc_v4(msg + 16ull * i), bb = gin::ld_nc_v4(msg + 16ull * (i + 32));
        uint4 c = gin::ld_nc_v4(msg + 16ull * (i + 64)), d = gin::ld_nc_v4(msg + 16ull * (i + 96));
        gin::st_v4(dst + 16ull * i, transform_vec(a, L.mode, e));
        gin::st_v4(dst + 16ull * (i + 32), transform_vec(bb, L.mode, e));
        gin::st_v4(dst + 16ull * (i + 64), transform_vec(c, L.mode, e));
        gin::st_v4(dst + 16ull * (i + 96), transform_vec(d, L.mode, e));
      }
      for (; i < vhi; i += 32) gin::st_v4(dst + 16ull * i, transform_vec(gin::ld_nc_v4(msg + 16ull * i), L.mode, e));
    } else if (p == 0) {
      const uint16_t* s16 = reinterpret_cast<const uint16_t*>(msg);
      uint16_t* d16 = reinterpret_cast<uint16_t*>(dst);
      for (uint32_t j = lane; j < H; j += 32) {
        const uint32_t two = transform_vec(make_uint4(s16[j], 0, 0, 0), L.mode, e).x;
        d16[j] = (uint16_t)(two & 0xFFFFu);
      }
    }
  }

  // Release: the last CTA signals each (source, context) with its count.
  arrive_last(R.ws + 1, (unsigned)(iteration * G), &is_last);
  if (is_last && tid == 0) *moe_iter_ptr(R, 1) = iteration;  // every CTA has read it (arrival)
  if (is_last && PROXY && L.coalesce) {
    // one copy-engine transfer per source (all its results, every expert),
    // then that source's combine flag with the total, on ctx src % n_ctx
    const gin::Team world = gin::WorldTeam(n);
    gin::CoopThread me;
    for (uint32_t src = tid; src < n; src += kMoeThreads) {
      const uint32_t tot = src_base[src + 1] - src_base[src];
      const gin::Gin g(v, src % n_ctx);
      if (src != rank && tot)
        g.put(me, world, src, L.win_mirror, (uint64_t)rank * T * K * cmsg, L.win_cstage, (uint64_t)src_base[src] * cmsg,
              (uint64_t)tot * cmsg);
      if (tot) g.signal(me, world, src, L.cell0 + e_local, gin::SignalAdd(tot));
    }
  } else if (is_last && PROXY) {  // reference pattern: one put per message, per-(source, ctx) flags
    const gin::Team world = gin::WorldTeam(n);
    gin::CoopThread me;
    for (uint32_t sc = tid; sc < n * n_ctx; sc += kMoeThreads) {
      const uint32_t src = sc / n_ctx, ctx = sc % n_ctx;
      const gin::Gin g(v, ctx);
      uint32_t c = 0;
      for (uint32_t e_loc = 0; e_loc < e_local; ++e_loc) {
        if ((rank * e_local + e_loc) % n_ctx != ctx) continue;
        const uint32_t pr = e_loc * n + src;
        for (uint32_t slot = 0; src != rank && slot < cnt[pr]; ++slot) {  // own tokens were written in place
          const uint64_t moff = L.layout == 0 ? (((uint64_t)e_loc * n + src) * T + slot) * dmsg
                                              : ((uint64_t)src * T * K + src_prefix[pr] + slot) * dmsg;
          const unsigned char* meta = reinterpret_cast<const unsigned char*>(recv + moff + payload);
          const uint32_t token = meta[4] | (meta[5] << 8) | (meta[6] << 16) | ((uint32_t)meta[7] << 24);
          const uint32_t k = meta[8] | (meta[9] << 8) | (meta[10] << 16) | ((uint32_t)meta[11] << 24);
          g.put(me, world, src, L.win_combine, ((uint64_t)token * K + k) * cmsg, L.win_cstage,
                ((uint64_t)pair_start[pr] + slot) * cmsg, cmsg);
        }
        c += cnt[pr];
      }
      if (c) g.signal(me, world, src, L.cell0 + e_local, gin::SignalAdd(c));
    }
  } else if (is_last) {
    for (uint32_t sc = tid; sc < n * n_ctx; sc += kMoeThreads) {
      const uint32_t src = sc / n_ctx, ctx = sc % n_ctx;
      uint32_t c = 0;
      for (uint32_t e_loc = 0; e_loc < e_local; ++e_loc)
        if ((rank * e_local + e_loc) % n_ctx == ctx) c += cnt[e_loc * n + src];
      if (c) gin.release_signal_raw(src, L.cell0 + e_local, c);
    }
  }

  // Source side: acquire all T*K outputs, then reduce with the top-k weights.
  if (tid == 0) {
    const uint64_t want = iteration * (uint64_t)T * K;
    const uint64_t t_start = gin::globaltimer();
    uint32_t spins = 0;
    while (gin.read_signal(L.cell0 + e_local) < want) {
      if (++spins > 32) __nanosleep(64);
      if ((spins & 1023) == 0 && gin::globaltimer() - t_start > v->timeout_ns) {
        gin::raise_error(v, GIN_DEVERR_TIMEOUT);
        break;
      }
    }
  }
  __syncthreads();
  char* crecv = v->win[L.win_combine].base[rank];
  // proxy + coalesce: results arrived in the mirror window (send order); the
  // reduce gathers them through the (t, k) -> mirror index of the dispatch and
  // also writes them to (t*K+k)*cmsg, so the combine window ends identical to
  // the reference's (harness_moe.cpp:203-205)
  const bool mirrored = PROXY && L.coalesce;
  const char* mirror = mirrored ? v->win[L.win_mirror].base[rank] : nullptr;
  auto ysrc = [&](uint32_t t, uint32_t k) -> const char* {
    return mirrored ? mirror + (uint64_t)R.midx[(uint64_t)t * K + k] * cmsg : crecv + ((uint64_t)t * K + k) * cmsg;
  };
  const uint64_t ritems = (uint64_t)T * parts;
  for (uint64_t it = (uint64_t)b * kMoeWarps + warp; it < ritems; it += (uint64_t)G * kMoeWarps) {
    const uint32_t t = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    char* o = reinterpret_cast<char*>(R.out) + (uint64_t)t * payload;
    if (vec_ok) {
      const uint32_t vlo = p * vec_per_part, vhi = min(vlo + vec_per_part, nvec);
      for (uint32_t i = vlo + lane; i < vhi; i += 32) {
        if (L.mode == 0) {
          uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
          const uint16_t* w = reinterpret_cast<const uint16_t*>(R.weights) + (uint64_t)t * K;
          for (uint32_t k = 0; k < K; ++k) {
            const uint32_t wk = w[k];
            const uint4 y = gin::ld_na_v4(ysrc(t, k) + 16ull * i);
            if (mirrored) gin::st_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i, y);
            const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[2 * q] += wk * (ys[q] & 0xFFFFu);
              acc[2 * q + 1] += wk * (ys[q] >> 16);
            }
          }
          uint4 r;
          r.x = (acc[0] & 0xFFFFu) | (acc[1] << 16);
          r.y = (acc[2] & 0xFFFFu) | (acc[3] << 16);
          r.z = (acc[4] & 0xFFFFu) | (acc[5] << 16);
          r.w = (acc[6] & 0xFFFFu) | (acc[7] << 16);
          gin::st_v4(o + 16ull * i, r);
        } else {
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          const float* w = reinterpret_cast<const float*>(R.weights) + (uint64_t)t * K;
          for (uint32_t k = 0; k < K; ++k) {
            const float wk = w[k];
            const uint4 y = gin::ld_na_v4(ysrc(t, k) + 16ull * i);
            if (mirrored) gin::st_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i, y);
            const uint32_t ys[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              acc[2 * q] = __fadd_rn(acc[2 * q], __fmul_rn(wk, __uint_as_float(ys[q] << 16)));
              acc[2 * q + 1] = __fadd_rn(acc[2 * q + 1], __fmul_rn(wk, __uint_as_float(ys[q] & 0xFFFF0000u)));
            }
          }
          uint32_t pk[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            pk[q] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[2 * q])) |
                    ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[2 * q + 1])) << 16);
          }
          gin::st_v4(o + 16ull * i, make_uint4(pk[0], pk[1], pk[2], pk[3]));
        }
      }
    } else if (p == 0) {
      uint16_t* o16 = reinterpret_cast<uint16_t*>(o);
      for (uint32_t j = lane; j < H; j += 32) {
        if (L.mode == 0) {
          uint32_t acc = 0;
          const uint16_t* w = reinterpret_cast<const uint16_t*>(R.weights) + (uint64_t)t * K;
          for (uint32_t k = 0; k < K; ++k) {
            const uint16_t y = reinterpret_cast<const uint16_t*>(ysrc(t, k))[j];
            if (mirrored) reinterpret_cast<uint16_t*>(crecv + ((uint64_t)t * K + k) * cmsg)[j] = y;
            acc += (uint32_t)w[k] * y;
          }
          o16[j] = (uint16_t)acc;
        } else {
          float acc = 0.f;
          const float* w = reinterpret_cast<const float*>(R.weights) + (uint64_t)t * K;
          for (uint32_t k = 0; k < K; ++k) {
            const uint16_t y = reinterpret_cast<const uint16_t*>(ysrc(t, k))[j];
            if (mirrored) reinterpret_cast<uint16_t*>(crecv + ((uint64_t)t * K + k) * cmsg)[j] = y;
            acc = __fadd_rn(acc, __fmul_rn(w[k], __uint_as_float((uint32_t)y << 16)));
          }
          o16[j] = __bfloat16_as_ushort(__float2bfloat16_rn(acc));
        }
      }
    }
  }
}

}  // namespace ginsim_b200
