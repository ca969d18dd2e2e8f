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

namespace ginsim_b200 {

constexpr int kMoeThreads = 512;
constexpr int kMoeWarps = kMoeThreads / 32;
constexpr uint32_t kMaxExperts = 1024;
constexpr uint32_t kMaxGrid = 1024;  // CTAs per rank of one launch

struct MoeRankArgs {
  const GinDevCommView* view;
  unsigned int* ws;           // per-moe arrival counters [0] dispatch [1] combine [2] slot barrier
  uint32_t* route;            // TMA dispatch scratch: hist [kMaxGrid][E], prefix [kMaxGrid][E], totals [E]
  char** dst_g;               // TMA dispatch: [T][Kp] destination pointer of every (t, k) pair
  uint32_t* midx;             // proxy: [T][K] index of (t, k)'s result in the combine mirror window
  uint64_t* aux_g;            // layout 2: [2][T][Kp] row-header address and (slot, e_loc) per pair
  const uint16_t* x;          // [T][H]
  const int32_t* idx;         // [T][K]
  const void* weights;        // [T][K] u16 (mode 0) / f32 (mode 1)
  uint16_t* out;              // [T][H]
  uint64_t iteration;         // 1-based
  uint64_t* prof;             // optional per-CTA %globaltimer stamps [3 kernels][1024 CTAs][8]
};

// Phase timeline (GINSIM_PROFILE_PHASES=1): thread 0 of each CTA stamps
// %globaltimer at its phase boundaries; ginsim_cuda_moe_phase_times reads them.
#define MOE_STAMP(R, kern, slot)                                                                  \
  do {                                                                                            \
    if ((R).prof && threadIdx.x == 0)                                                             \
      (R).prof[((uint64_t)(kern) * 1024 + blockIdx.x) * 8 + (slot)] = gin::globaltimer();         \
  } while (0)

struct MoeLaunch {
  MoeRankArgs r[GIN_MAX_RANKS];
  uint32_t E, K, T, H, mode, layout, e_local, parts, cparts;
  uint32_t win_dispatch, win_counts, win_combine;
  uint32_t win_stage, win_cstage, coalesce;  // proxy backend: dispatch / combine staging windows
  uint32_t win_mirror;           // proxy + coalesce: combine results in the source's send order
  uint32_t win_rows;             // layout 2: per-source row staging + 128-byte row headers
  uint32_t coop;                 // TMA dispatch: cooperative route tables + all-token work (large T*K)
  uint32_t fuse_reduce;          // TMA combine: reduce inside the send kernel (small, latency-bound T)
  uint64_t dmsg;                 // dispatch message bytes: payload + 16-byte meta
  uint32_t mpay;                 // payload bytes before the meta (2H; fp8: H + H/32)
  uint64_t cmsg;                 // combine message bytes (2H; fp8 combine, mode 3: H + H/32)
  uint32_t no_wait;              // profiling only: dispatch returns without acquiring its experts
  uint32_t dyn;                  // TMA kernels: warps grab work in batches from a device counter (1) or static (0)
};

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t u16x2_transform(uint32_t two, uint32_t add) {
  // two u16 lanes: y = 3x + (17e+1), each lane mod 2^16
  const uint32_t lo = ((two & 0xFFFFu) * 3u + add) & 0xFFFFu;
  const uint32_t hi = ((two >> 16) * 3u + add) & 0xFFFFu;
  return lo | (hi << 16);
}

__device__ __forceinline__ uint32_t bf16x2_transform(uint32_t two, float s, float c) {
  const float a = __uint_as_float(two << 16), b = __uint_as_float(two & 0xFFFF0000u);
  const __nv_bfloat16 ya = __float2bfloat16_rn(__fadd_rn(__fmul_rn(a, s), c));
  const __nv_bfloat16 yb = __float2bfloat16_rn(__fadd_rn(__fmul_rn(b, s), c));
  return (uint32_t)__bfloat16_as_ushort(ya) | ((uint32_t)__bfloat16_as_ushort(yb) << 16);
}

// 8 bf16 lanes: y = bf16(fp32(x)*s + c), single-rounded mul and add, packed
// back two at a time (cvt.rn.bf16x2.f32) -- same rounding as bf16x2_transform.
__device__ __forceinline__ uint32_t bf16x2_pack_transform(uint32_t two, float s, float c) {
  const float a = __fadd_rn(__fmul_rn(__uint_as_float(two << 16), s), c);
  const float b = __fadd_rn(__fmul_rn(__uint_as_float(two & 0xFFFF0000u), s), c);
  const __nv_bfloat162 r = __floats2bfloat162_rn(a, b);  // .x = a (low half), .y = b
  return *reinterpret_cast<const uint32_t*>(&r);
}
__device__ __forceinline__ uint4 bf16x8_transform(uint4 v, float s, float c) {
  return make_uint4(bf16x2_pack_transform(v.x, s, c), bf16x2_pack_transform(v.y, s, c),
                    bf16x2_pack_transform(v.z, s, c), bf16x2_pack_transform(v.w, s, c));
}

// fp8 mode (mode 2): one 128-element block of a bf16 row per
// warp step, 4 elements per lane: amax by warp reduction (exact), scale =
// amax/448 and inv = 448/amax single-rounded, q = e4m3(x*inv) with RNE and
// saturation (cvt.rn.satfinite.e4m3x2.f32) -- the oracle's gso_fp8_quant_row.
__device__ __forceinline__ void fp8_quant_block(const uint16_t* in, uint8_t* q, float* scale_out, uint32_t lane) {
  const uint2 raw = *reinterpret_cast<const uint2*>(in + 4 * lane);
  float f[4] = {__uint_as_float(raw.x << 16), __uint_as_float(raw.x & 0xFFFF0000u), __uint_as_float(raw.y << 16),
                __uint_as_float(raw.y & 0xFFFF0000u)};
  float amax = fmaxf(fmaxf(fabsf(f[0]), fabsf(f[1])), fmaxf(fabsf(f[2]), fabsf(f[3])));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float scale = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const float inv = amax > 0.0f ? __fdiv_rn(448.0f, amax) : 1.0f;
  const __nv_fp8x2_storage_t lo =
      __nv_cvt_float2_to_fp8x2(make_float2(__fmul_rn(f[0], inv), __fmul_rn(f[1], inv)), __NV_SATFINITE, __NV_E4M3);
  const __nv_fp8x2_storage_t hi =
      __nv_cvt_float2_to_fp8x2(make_float2(__fmul_rn(f[2], inv), __fmul_rn(f[3], inv)), __NV_SATFINITE, __NV_E4M3);
  *reinterpret_cast<uint32_t*>(q + 4 * lane) = (uint32_t)lo | ((uint32_t)hi << 16);
  if (lane == 0) *scale_out = scale;
}
// 8 e4m3 codes (one 16-byte bf16 output vector): deq = fp32(q)*scale, then the
// bf16 expert transform y = bf16(deq*s + c), single-rounded ops.  Codes are
// widened two at a time (cvt.rn.f16x2.e4m3x2: exact, e4m3 is a subset of f16).
__device__ __forceinline__ uint4 fp8x8_transform(uint2 codes, float scale, float s, float c) {
  uint32_t out[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const uint32_t w = h < 2 ? codes.x : codes.y;
    const __nv_fp8x2_storage_t pair = (__nv_fp8x2_storage_t)((w >> ((h & 1) * 16)) & 0xFFFF);
    const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2(pair, __NV_E4M3);
    const float2 f = __half22float2(__half2(hr));
    const float a = __fmul_rn(f.x, scale), b = __fmul_rn(f.y, scale);
    const __nv_bfloat162 r = __floats2bfloat162_rn(__fadd_rn(__fmul_rn(a, s), c), __fadd_rn(__fmul_rn(b, s), c));
    out[h] = *reinterpret_cast<const uint32_t*>(&r);
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

__device__ __forceinline__ uint4 transform_vec(uint4 v, uint32_t mode, uint32_t e) {
  if (mode == 0) {
    const uint32_t add = (e * 17u + 1u) & 0xFFFFu;
    v.x = u16x2_transform(v.x, add);
    v.y = u16x2_transform(v.y, add);
    v.z = u16x2_transform(v.z, add);
    v.w = u16x2_transform(v.w, add);
  } else {
    const float s = 1.0f + (float)(e % 7u) / 8.0f;
    const float c = ((float)(e % 9u) - 4.0f) / 16.0f;
    v.x = bf16x2_transform(v.x, s, c);
    v.y = bf16x2_transform(v.y, s, c);
    v.z = bf16x2_transform(v.z, s, c);
    v.w = bf16x2_transform(v.w, s, c);
  }
  return v;
}

// Per-source exclusive prefix over the experts of this rank (compact layout):
// src_prefix[e*n+s] = sum_{e'<e} cnt[e'*n+s]; one warp per source.
template <int WARPS>
__device__ __forceinline__ void source_prefix(const uint32_t* cnt, uint32_t* src_prefix, uint32_t n, uint32_t e_local) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t sidx = warp; sidx < n; sidx += WARPS) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < e_local; c0 += 32) {
      const uint32_t e = c0 + lane;
      const uint32_t xv = e < e_local ? cnt[e * n + sidx] : 0u;
      uint32_t incl = xv;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      if (e < e_local) src_prefix[e * n + sidx] = carry + incl - xv;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
}

// Grid arrival at the end of a phase: the last CTA of this rank's launch to
// arrive returns true (in every thread).  CTAs order their own traffic
// before the arrival at GPU scope (fence.acq_rel.gpu, much cheaper than a
// .sys fence per CTA); the last CTA then holds, by cumulativity, every CTA's
// puts, and its .sys release (one fence per releasing warp) publishes them to
// the peers (the paper's ordering rule, fabric.cpp:63-79).
__device__ __forceinline__ bool arrive_last(unsigned int* ctr, unsigned int target, int* flag_smem) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gin::fence_acq_rel_gpu();
    const unsigned prev = atomicAdd(ctr, 1u);
    const bool last = prev + 1 == target;
    if (last) gin::fence_acq_rel_gpu();
    *flag_smem = last ? 1 : 0;
  }
  __syncthreads();
  return *flag_smem != 0;
}

// Per-expert release of one dispatch (harness_moe.cpp:163-167) by the last
// CTA: warp d takes destination rank d; each lane writes its experts' counts,
// fences (one MEMBAR per warp instruction) and adds (1<<32)+count to their
// cells with relaxed reductions -- a release pattern per lane, one .sys fence
// per destination instead of one per expert.
__device__ __forceinline__ void release_experts(const gin::Gin& gin, const GinDevCommView* v, uint32_t win_counts,
                                                const uint32_t* hist, uint32_t n, uint32_t rank, uint32_t e_local) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t d = warp; d < n; d += nw) {
    uint32_t* cb = reinterpret_cast<uint32_t*>(v->win[win_counts].base[d]);
    // the counts need no ordering against the puts, only before the cells:
    // one fence between them releases both the puts (by cumulativity) and
    // the counts; for own experts the acquirer is on this GPU (GPU scope)
    for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
      gin::st_relaxed_sys32(cb + (uint64_t)e_loc * n + rank, hist[d * e_local + e_loc]);
    if (d == rank) gin::fence_acq_rel_gpu(); else gin::fence_acq_rel_sys();
    for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
      gin::red_relaxed_sys_add(gin.sub_cell(d, rank, e_loc), (1ull << 32) + hist[d * e_local + e_loc]);
  }
}

// Block-wide exclusive scan of n <= 4*kMoeThreads u32 values in smem.
__device__ void block_exclusive_scan(uint32_t* data, uint32_t n, uint32_t* warp_tot, uint32_t* total_out) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t per = (n + kMoeThreads - 1) / kMoeThreads;
  const uint32_t lo = tid * per, hi = min(lo + per, n);
  uint32_t local = 0;
  for (uint32_t i = lo; i < hi; ++i) local += data[i];
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kMoeWarps ? warp_tot[lane] : 0;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (uint32_t)o) wi += y;
    }
    if (lane < kMoeWarps) warp_tot[lane] = wi - w;
    if (lane == kMoeWarps - 1 && total_out) *total_out = wi;
  }
  __syncthreads();
  uint32_t run = warp_tot[warp] + incl - local;
  for (uint32_t i = lo; i < hi; ++i) {
    const uint32_t d = data[i];
    data[i] = run;
    run += d;
  }
  __syncthreads();
}

// ------------------------------------------------------------------ dispatch
// Phase A of every dispatch kernel: per-expert totals over the whole route
// table (hist), the counts of the pairs before this CTA's first token (run)
// and, optionally, a copy of this CTA's own pairs [pre_end, pre_end+nq).
// Every CTA reads all T*K indices from L2, so the loads are issued 16 bytes
// and 8 entries per thread at a time -- a scalar loop with a data-dependent
// store in its body is not unrolled by the compiler and serialises T*K/threads
// L2 round trips (~40 us at T=4096, measured).
template <int THREADS>
__device__ __forceinline__ void histogram_pass(const int32_t* idx, uint32_t TK, uint32_t pre_end, uint32_t nq,
                                               uint32_t* hist, uint32_t* run, uint32_t* own) {
  const uint32_t tid = threadIdx.x;
  auto take = [&](uint32_t j, uint32_t e) {
    atomicAdd(&hist[e], 1u);
    if (j < pre_end) atomicAdd(&run[e], 1u);
    else if (own && j - pre_end < nq) own[j - pre_end] = e;
  };
  uint32_t done = 0;
  if ((reinterpret_cast<uintptr_t>(idx) & 15) == 0) {
    const int4* v = reinterpret_cast<const int4*>(idx);
    const uint32_t n4 = TK / 4;
    uint32_t q = tid;
    for (; q + THREADS < n4; q += 2 * THREADS) {
      const int4 a = __ldg(v + q), b = __ldg(v + q + THREADS);
      take(4 * q, a.x), take(4 * q + 1, a.y), take(4 * q + 2, a.z), take(4 * q + 3, a.w);
      const uint32_t jb = 4 * (q + THREADS);
      take(jb, b.x), take(jb + 1, b.y), take(jb + 2, b.z), take(jb + 3, b.w);
    }
    for (; q < n4; q += THREADS) {
      const int4 a = __ldg(v + q);
      take(4 * q, a.x), take(4 * q + 1, a.y), take(4 * q + 2, a.z), take(4 * q + 3, a.w);
    }
    done = n4 * 4;
  }
  for (uint32_t j = done + tid; j < TK; j += THREADS) take(j, (uint32_t)__ldg(idx + j));
}

// PROXY = the Proxy backend: rows are staged into a local
// registered window laid out in destination order -- (dst_base[dst] +
// prefix_e[e] + slot) -- so every expert's messages form ONE contiguous run
// at both ends, and the last CTA hands each run to the host agent as a put
// descriptor (ordered before the expert's release on ctx e % n_ctx,
// harness_moe.cpp:135-167).  No NVLink store is issued by the kernel.
template <int KMAX, bool PROXY>
__global__ void __launch_bounds__(kMoeThreads, KMAX <= 8 ? 2 : 1) moe_dispatch_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
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
  arrive_last(R.ws + 0, (unsigned)(R.iteration * G), &is_last);
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
      gin::Gin(v, ctx_of(e)).put_value(me, world, dst, L.win_counts, ((uint64_t)e_loc * n + rank) * 4, hist_all[e]);
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
      gin::Gin(v, ctx_of(e)).signal(me, world, dst, e_loc, gin::SignalAdd((1ull << 32) + hist_all[e]));
    }
  } else if (is_last) {
    release_experts(gin, v, L.win_counts, hist_all, n, rank, e_local);
  }
  // Phase D: return once every local expert has been released by every source.
  if (tid == 0) {
    const uint64_t want = R.iteration * ((uint64_t)n << 32);
    for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) {
      const uint64_t t_start = gin::globaltimer();
      uint32_t spins = 0;
      while (gin.read_signal(e_loc) < want) {
        if (++spins > 32) __nanosleep(64);
        if ((spins & 1023) == 0 && gin::globaltimer() - t_start > v->timeout_ns) {
          gin::raise_error(v, GIN_DEVERR_TIMEOUT);
          break;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ combine
// PROXY: the expert transform writes message m (receive order) to m*cmsg of
// the local staging window, then the last CTA submits one put descriptor per message
// to (token*K+k)*cmsg of its source and, after them on the same context, the
// per-(source, ctx) combine flag (harness_moe.cpp:169-223).
template <bool PROXY>
__global__ void __launch_bounds__(kMoeThreads, 2) moe_combine_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t E = L.E, K = L.K, T = L.T, H = L.H, e_local = L.e_local;
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
    const uint32_t c = gin::ld_acquire_sys32(counts + i);
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
  arrive_last(R.ws + 1, (unsigned)(R.iteration * G), &is_last);
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
      if (tot) g.signal(me, world, src, e_local, gin::SignalAdd(tot));
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
      if (c) g.signal(me, world, src, e_local, gin::SignalAdd(c));
    }
  } else if (is_last) {
    for (uint32_t sc = tid; sc < n * n_ctx; sc += kMoeThreads) {
      const uint32_t src = sc / n_ctx, ctx = sc % n_ctx;
      uint32_t c = 0;
      for (uint32_t e_loc = 0; e_loc < e_local; ++e_loc)
        if ((rank * e_local + e_loc) % n_ctx == ctx) c += cnt[e_loc * n + src];
      if (c) gin.release_signal_raw(src, e_local, c);
    }
  }

  // Source side: acquire all T*K outputs, then reduce with the top-k weights.
  if (tid == 0) {
    const uint64_t want = R.iteration * (uint64_t)T * K;
    const uint64_t t_start = gin::globaltimer();
    uint32_t spins = 0;
    while (gin.read_signal(e_local) < want) {
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
            const uint4 y = gin::ld_nc_v4(ysrc(t, k) + 16ull * i);
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
            const uint4 y = gin::ld_nc_v4(ysrc(t, k) + 16ull * i);
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

// ------------------------------------------------------------------ TMA engine
// Same protocol as the LSU kernels above, with the data path moved onto the
// TMA engine: each warp runs its own kTmaStages-deep pipeline in which lane 0
// bulk-loads a message chunk (<= 8 KiB) from HBM into shared memory on an
// mbarrier and bulk-stores it to the K destinations (local HBM or NVLink
// peer mappings).  No registers or scoreboard slots are held by in-flight
// data, so one CTA of 8 warps per SM keeps ~170 KiB of loads and K times
// that of stores in flight.  Used whenever messages are 16-byte aligned.
constexpr int kTmaThreads = 256;
constexpr int kTmaWarps = kTmaThreads / 32;
constexpr int kCmbThreads = 512;
constexpr int kCmbWarps = kCmbThreads / 32;
// Pipeline depth per warp.  Dispatch uses 2 stages (a shallower per-SM TMA
// store queue drains faster at the end of the launch: -4 us at N=1, -6 us at
// N=2, measured); the combine send keeps 3 (its transform needs the slack).
constexpr int kTmaStages = 3;   // TmaSmem capacity, combine send
constexpr int kDispStages = 2;  // dispatch kernels

struct TmaSmem {  // per-warp control block, followed by the staging buffers
  uint64_t bar[kTmaStages];
  char* dptr[32];
  uint64_t itm[kTmaStages];  // item held by each stage (~0 = none)
  uint64_t cur;              // static sequence number (first round / static schedule)
  uint64_t itc, end;         // dynamic schedule: the grabbed batch [itc, end)
};
constexpr uint64_t kNoItem = ~0ull;

__device__ __forceinline__ uint32_t tma_chunk_len(uint32_t payload, uint32_t chunk, uint32_t p) {
  return min(chunk, payload - p * chunk);
}

// fp8 combine (mode 3): out = bf16(sum_k w_k * fp32(q_k)*scale_k) for one
// 16-byte output vector (8 elements) of token t, fp32 in k order.
template <int KMAX>
__device__ __forceinline__ uint4 reduce_fp8_vec(const char* crecv, uint64_t cmsg, uint32_t H, uint32_t t, uint32_t i,
                                                uint32_t K, const void* weights) {
  uint2 q[KMAX];
  float sc[KMAX];
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < (int)K) {
      const char* m = crecv + ((uint64_t)t * K + k) * cmsg;
      q[k] = *reinterpret_cast<const uint2*>(m + 8ull * i);
      sc[k] = *reinterpret_cast<const float*>(m + H + 4ull * (i / 16));
    }
  }
  const float* w = reinterpret_cast<const float*>(weights) + (uint64_t)t * K;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < (int)K) {
      const float wk = w[k];
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const uint32_t word = h < 2 ? q[k].x : q[k].y;
        const __half2_raw hr = __nv_cvt_fp8x2_to_halfraw2((__nv_fp8x2_storage_t)((word >> ((h & 1) * 16)) & 0xFFFF), __NV_E4M3);
        const float2 f = __half22float2(__half2(hr));
        acc[2 * h] = __fadd_rn(acc[2 * h], __fmul_rn(wk, __fmul_rn(f.x, sc[k])));
        acc[2 * h + 1] = __fadd_rn(acc[2 * h + 1], __fmul_rn(wk, __fmul_rn(f.y, sc[k])));
      }
    }
  }
  uint32_t pk[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const __nv_bfloat162 r = __floats2bfloat162_rn(acc[2 * h], acc[2 * h + 1]);
    pk[h] = *reinterpret_cast<const uint32_t*>(&r);
  }
  return make_uint4(pk[0], pk[1], pk[2], pk[3]);
}

// out = sum_k w_k * y_k for one 16-byte vector (8 elements) of token t:
// u16 wraparound (harness_moe.cpp:227-242) or fp32 accumulate in k order
// with single rounding per op, rounded once to bf16.
template <int KMAX>
__device__ __forceinline__ uint4 reduce_vec(const uint4* y, uint32_t K, uint32_t mode, const void* weights, uint32_t t) {
  if (mode == 0) {
    const uint16_t* w = reinterpret_cast<const uint16_t*>(weights) + (uint64_t)t * K;
    uint32_t acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < KMAX; ++k) {
      if (k < (int)K) {
        const uint32_t wk = w[k];
        const uint32_t ys[4] = {y[k].x, y[k].y, y[k].z, y[k].w};
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          acc[2 * c] += wk * (ys[c] & 0xFFFFu);
          acc[2 * c + 1] += wk * (ys[c] >> 16);
        }
      }
    }
    return make_uint4((acc[0] & 0xFFFFu) | (acc[1] << 16), (acc[2] & 0xFFFFu) | (acc[3] << 16),
                      (acc[4] & 0xFFFFu) | (acc[5] << 16), (acc[6] & 0xFFFFu) | (acc[7] << 16));
  }
  const float* w = reinterpret_cast<const float*>(weights) + (uint64_t)t * K;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < KMAX; ++k) {
    if (k < (int)K) {
      const float wk = w[k];
      const uint32_t ys[4] = {y[k].x, y[k].y, y[k].z, y[k].w};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        acc[2 * c] = __fadd_rn(acc[2 * c], __fmul_rn(wk, __uint_as_float(ys[c] << 16)));
        acc[2 * c + 1] = __fadd_rn(acc[2 * c + 1], __fmul_rn(wk, __uint_as_float(ys[c] & 0xFFFF0000u)));
      }
    }
  }
  uint32_t pk[4];
#pragma unroll
  for (int c = 0; c < 4; ++c)
    pk[c] = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[2 * c])) |
            ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[2 * c + 1])) << 16);
  return make_uint4(pk[0], pk[1], pk[2], pk[3]);
}

// Grid-wide barrier among the G CTAs of one rank's cooperative launch: a
// monotone arrival counter (target = iteration * G), so it needs no reset.
__device__ __forceinline__ void rank_grid_barrier(unsigned int* ctr, unsigned int target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    gin::fence_acq_rel_gpu();
    atomicAdd(ctr, 1u);
    while (true) {
      unsigned cur;
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(ctr) : "memory");
      if (cur >= target) break;
      __nanosleep(20);
    }
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
  const unsigned int bar_target = (unsigned int)(R.iteration * G);
  // coop: route tables built cooperatively + work over all tokens (large T*K);
  // local: every CTA histograms the whole (small) route table and moves only
  // its own tokens -- no grid barrier on the latency-bound LL path
  const bool coop = L.coop != 0;
  MOE_STAMP(R, 0, 0);

  __shared__ uint32_t hist_all[kMaxExperts], run[kMaxExperts], prefix_e[kMaxExperts];
  __shared__ char* sbase[GIN_MAX_RANKS];
  __shared__ int is_last;
  extern __shared__ __align__(128) char dsm[];
  TmaSmem* ctl = reinterpret_cast<TmaSmem*>(dsm) + warp;
  // per stage: [dst pointers: Kp * 8 bytes, padded to 128][row chunk]
  const uint32_t dhead = (Kp * 8 + 127) & ~127u;
  // fp8: [dst row][bf16 chunk][e4m3 chunk/2][scales chunk/64, padded]
  const uint32_t qoff = dhead + chunk, soff = qoff + chunk / 2;
  const uint32_t sstride = fp8 ? ((soff + chunk / 64 + 15) & ~15u) : dhead + chunk;
  char* stage = dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)warp * kDispStages * sstride;
  uint32_t* own = reinterpret_cast<uint32_t*>(dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) +
                                              (size_t)kTmaWarps * kDispStages * sstride);  // [(t1-t0)*K]
  uint32_t* g_hist = R.route;                                  // [G][E]
  uint32_t* g_pre = R.route + (size_t)kMaxGrid * kMaxExperts;  // [G][E]
  uint32_t* g_tot = R.route + 2 * (size_t)kMaxGrid * kMaxExperts;  // [E]
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
  auto next_item = [&]() -> uint64_t {  // lane 0 only
    uint64_t it;
    if (!coop) {
      it = lbase + (ctl->cur++) * kTmaWarps;
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
    return it < items ? it : kNoItem;
  };
  // A stage's mbarrier expects the row chunk AND the token's destination row;
  // the row chunk does not depend on routing, so it can be requested first.
  auto issue_row = [&](int s, uint64_t it) {  // lane 0
    const uint32_t t = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + Kp * 8);
    gin::tma::load(sb + dhead, x + (uint64_t)t * payload + (uint64_t)p * chunk, len, &ctl->bar[s]);
  };
  auto issue_dst = [&](int s, uint64_t it) {  // lane 0, once dst_g is published
    const uint32_t t = (uint32_t)(it / parts);
    gin::tma::load(stage + (size_t)s * sstride, dst_g + (uint64_t)t * Kp, Kp * 8, &ctl->bar[s]);
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
  // A0: own routes -> smem + own histogram -> global row
  for (uint32_t q = tid; q < nq; q += kTmaThreads) {
    const uint32_t e = (uint32_t)__ldg(R.idx + (uint64_t)t0 * K + q);
    own[q] = e;
    atomicAdd(&hist_all[e], 1u);
  }
  __syncthreads();
  for (uint32_t e = tid; e < E; e += kTmaThreads) g_hist[(size_t)b * E + e] = hist_all[e];
  MOE_STAMP(R, 0, 1);
  rank_grid_barrier(R.ws + 3, bar_target);
  // A1: column scans, one warp per expert e = b + w*G
  for (uint32_t e = b + warp * G; e < E; e += kTmaWarps * G) {
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
  rank_grid_barrier(R.ws + 4, bar_target);
  // A2: this CTA's prefix row and the totals; reference slot numbers
  for (uint32_t e = tid; e < E; e += kTmaThreads) {
    run[e] = __ldcg(g_pre + (size_t)b * E + e);
    hist_all[e] = __ldcg(g_tot + e);
  }
  __syncthreads();
  }  // coop
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
  __syncthreads();
  if (warp == 0) {
    // Reference slot order (t, k ascending): 32 pairs at a time; lanes with the
    // same expert rank themselves by lane (match_any) and the group's lowest
    // lane advances the expert's running count.
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
    const uint32_t t = (uint32_t)(it / parts), p = (uint32_t)(it % parts);
    char* sb = stage + (size_t)s * sstride;
    char* const* dp = reinterpret_cast<char* const*>(sb);
    gin::tma::mbar_wait(&ctl->bar[s], (j / kDispStages) & 1);
    if (p == 0 && lane < K) gin::st_v4(dp[lane] + L.mpay, make_uint4(rank, t, lane, lane + 1));  // meta
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
  arrive_last(R.ws + 0, (unsigned)(R.iteration * G), &is_last);
  if (is_last) {
    if (tid == 0) *grab_ctr = 0;  // every CTA is past Phase B
    release_experts(gin, v, L.win_counts, hist_all, n, rank, e_local);
  }
  MOE_STAMP(R, 0, 6);
  if (tid == 0) {
    const uint64_t want = R.iteration * ((uint64_t)n << 32);
    if (!L.no_wait)
      for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) gin.wait_ge_signal(e_loc, want);
  }
  MOE_STAMP(R, 0, 7);
}

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
// Sender phases as moe_dispatch_tma_kernel (cooperative route tables with the
// n destination "row" bins appended to the E expert bins), then
//   C: per remote destination: counts + row count (relaxed) + fence.sys + one
//      release of the destination's rows cell; own experts released as usual.
//   F: every rank acquires the rows cell (n-1 sources), then fans the rows
//      out through the same TMA pipeline (bulk load header + row chunk, bulk
//      store to each listed slot), the last CTA releases the experts'
//      (1<<32)+count on behalf of each source (own GPU: GPU scope).
//   D: acquire every local expert as before.
constexpr uint32_t kRowHdr = 128;

template <int KMAX>
__global__ void __launch_bounds__(kTmaThreads, 1) moe_dispatch_dedup_kernel(MoeLaunch L, uint32_t chunk) {
  const MoeRankArgs& R = L.r[blockIdx.y];
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
  const unsigned int bar_target = (unsigned int)(R.iteration * G);
  MOE_STAMP(R, 0, 0);

  __shared__ uint32_t hist_all[kMaxExperts + GIN_MAX_RANKS], run[kMaxExperts + GIN_MAX_RANKS];
  __shared__ uint32_t prefix_e[kMaxExperts];
  __shared__ uint32_t cntv[kMaxExperts], src_prefix[kMaxExperts], rcnt[GIN_MAX_RANKS + 1];
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
  if (warp == 0) {
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
        ent_g[pi] = (uint64_t)slot | ((uint64_t)e_loc << 32);
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
  rank_grid_barrier(R.ws + 5, bar_target);
  MOE_STAMP(R, 0, 4);

  // ---- Phase B: one bulk store per (token, destination rank) for remote
  // rows, one per message for own experts
  const char* x = reinterpret_cast<const char*>(R.x);
  const uint64_t items = (uint64_t)T * parts;
  const uint64_t gw = (uint64_t)b * kTmaWarps + warp, wstride = (uint64_t)G * kTmaWarps;
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
    gin::tma::fence_proxy_async_global();
  }
  MOE_STAMP(R, 0, 5);

  // ---- Phase C: per remote destination: counts + row count, one fence, one
  // release of its rows cell; own experts as usual (GPU scope)
  arrive_last(R.ws + 0, bar_target, &is_last);
  if (is_last) {
    for (uint32_t d = warp; d < n; d += kTmaWarps) {
      uint32_t* cb = reinterpret_cast<uint32_t*>(v->win[L.win_counts].base[d]);
      for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
        gin::st_relaxed_sys32(cb + (uint64_t)e_loc * n + rank, hist_all[d * e_local + e_loc]);
      if (lane == 0) gin::st_relaxed_sys32(cb + (uint64_t)e_local * n + rank, hist_all[E + d]);
      if (d == rank) {
        gin::fence_acq_rel_gpu();
        for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
          gin::red_relaxed_sys_add(gin.sub_cell(d, rank, e_loc), (1ull << 32) + hist_all[d * e_local + e_loc]);
      } else {
        gin::fence_acq_rel_sys();
        if (lane == 0) gin::red_relaxed_sys_add(gin.sub_cell(d, rank, e_local + 1), 1ull);
      }
    }
  }
  MOE_STAMP(R, 0, 6);

  // ---- Phase F: receive side -- fan the rows of every source out into the
  // expert slots of this rank's dispatch window
  if (L.no_wait) return;  // profiling harness: the sender's part only
  if (tid == 0) gin.wait_ge_signal(e_local + 1, R.iteration * (uint64_t)(n - 1));
  __syncthreads();
  gin::tma::fence_proxy_async_global();  // rows/headers written by peers -> read by this CTA's bulk loads
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
  const uint32_t P = e_local * n;
  for (uint32_t i = tid; i < P; i += kTmaThreads) cntv[i] = gin::ld_acquire_sys32(counts + i);
  if (tid <= n) rcnt[tid] = 0;
  __syncthreads();
  if (tid < n) rcnt[tid] = tid == rank ? 0u : gin::ld_acquire_sys32(counts + P + tid);
  source_prefix<kTmaWarps>(cntv, src_prefix, n, e_local);
  __syncthreads();
  if (tid == 0) {  // rcnt -> exclusive prefix over sources (row order: source-major)
    uint32_t acc = 0;
    for (uint32_t s2 = 0; s2 < n; ++s2) {
      const uint32_t c = rcnt[s2];
      rcnt[s2] = acc;
      acc += c;
    }
    rcnt[n] = acc;
  }
  __syncthreads();
  const char* rows = v->win[L.win_rows].base[rank];
  char* mywin = v->win[L.win_dispatch].base[rank];
  const uint64_t fitems = (uint64_t)rcnt[n] * parts;
  auto locate_row = [&](uint64_t it, uint32_t& src, uint32_t& jr) {
    const uint32_t r = (uint32_t)(it / parts);
    uint32_t s2 = 0;
    while (s2 + 1 < n && rcnt[s2 + 1] <= r) ++s2;
    while (s2 < n && rcnt[s2 + 1] == rcnt[s2]) ++s2;  // skip sources with no rows
    src = s2;
    jr = r - rcnt[s2];
  };
  auto fissue = [&](int s, uint64_t it) {
    uint32_t src, jr;
    locate_row(it, src, jr);
    const uint32_t p = (uint32_t)(it % parts);
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_arrive_expect_tx(&ctl->bar[s], len + kRowHdr);
    gin::tma::load(sb, rows + rows_bytes + ((uint64_t)src * T + jr) * kRowHdr, kRowHdr, &ctl->bar[s]);
    gin::tma::load(sb + dhead, rows + ((uint64_t)src * T + jr) * payload + (uint64_t)p * chunk, len, &ctl->bar[s]);
  };
  __syncthreads();
  const uint32_t phase0 = (uint32_t)((items + wstride - 1 - gw) / wstride);  // items this warp ran in Phase B
  if (lane == 0) {
    for (int s = 0; s < kDispStages; ++s) {
      const uint64_t it = gw + s * wstride;
      if (it < fitems) fissue((int)((phase0 + s) % kDispStages), it);
    }
  }
  for (uint32_t j = 0;; ++j) {
    const uint64_t it = gw + (uint64_t)j * wstride;
    if (it >= fitems) break;
    const uint32_t jj = phase0 + j;  // continue the stage/parity sequence of Phase B
    const int s = (int)(jj % kDispStages);
    uint32_t src, jr;
    locate_row(it, src, jr);
    const uint32_t p = (uint32_t)(it % parts);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_wait(&ctl->bar[s], (jj / kDispStages) & 1);
    const uint32_t* h = reinterpret_cast<const uint32_t*>(sb);
    const uint32_t tok = h[0], mask = h[1];
    if (p == 0 && lane < K && ((mask >> lane) & 1)) {
      const uint32_t slot = h[2 + 2 * lane], e_loc = h[3 + 2 * lane] & 0xFFFFu;
      char* m = mywin + ((uint64_t)src * T * K + src_prefix[e_loc * n + src] + slot) * dmsg;
      gin::st_v4(m + payload, make_uint4(src, tok, lane, lane + 1));
    }
    if (lane == 0) {
      const uint32_t len = tma_chunk_len(payload, chunk, p);
      for (uint32_t k = 0; k < K; ++k) {
        if (!((mask >> k) & 1)) continue;
        const uint32_t slot = h[2 + 2 * k], e_loc = h[3 + 2 * k] & 0xFFFFu;
        char* m = mywin + ((uint64_t)src * T * K + src_prefix[e_loc * n + src] + slot) * dmsg;
        gin::tma::store(m + (uint64_t)p * chunk, sb + dhead, len);
      }
      gin::tma::commit();
      if (j >= 1) {
        gin::tma::wait_read<1>();
        const uint64_t nxt = it - wstride + kDispStages * wstride;
        if (nxt < fitems) fissue((int)((jj - 1) % kDispStages), nxt);
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    gin::tma::wait_all();
    gin::tma::fence_proxy_async_global();
  }
  // the last CTA releases every (local expert, remote source) pair on the
  // source's behalf: this GPU is the only reader (GPU scope)
  arrive_last(R.ws + 12, bar_target, &is_last);
  if (is_last) {
    gin::fence_acq_rel_gpu();
    for (uint32_t i = tid; i < P; i += kTmaThreads) {
      const uint32_t e_loc = i / n, src = i % n;
      if (src != rank) gin::red_relaxed_sys_add(gin.sub_cell(rank, src, e_loc), (1ull << 32) + cntv[i]);
    }
  }
  MOE_STAMP(R, 0, 7);
  if (tid == 0 && !L.no_wait) {
    const uint64_t want = R.iteration * ((uint64_t)n << 32);
    for (uint32_t e_loc = b; e_loc < e_local; e_loc += G) gin.wait_ge_signal(e_loc, want);
  }
}

template <int KMAX>
__global__ void __launch_bounds__(kCmbThreads, 1) moe_combine_tma_kernel(MoeLaunch L, uint32_t chunk) {
  // The transform pass keeps the SM busy between TMA waits, so this kernel
  // runs 16 warps with smaller (<= 4 KiB) chunks instead of the dispatch's 8.
  constexpr int kTmaThreads = kCmbThreads;
  constexpr int kTmaWarps = kCmbThreads / 32;
  const MoeRankArgs& R = L.r[blockIdx.y];
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, rank = v->rank, n_ctx = v->n_ctx;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint64_t dmsg = L.dmsg, cmsg = L.cmsg;
  const bool fp8 = L.mode >= 2, fp8c = L.mode == 3;
  const uint32_t payload = 2u * H, parts = L.cparts;
  MOE_STAMP(R, 1, 0);

  __shared__ uint32_t cnt[kMaxExperts], pair_start[kMaxExperts + 1], src_prefix[kMaxExperts];
  __shared__ uint32_t warp_tot[kMoeWarps];
  __shared__ uint32_t total_msgs;
  __shared__ int is_last;
  extern __shared__ __align__(128) char dsm[];
  TmaSmem* ctl = reinterpret_cast<TmaSmem*>(dsm) + warp;
  // per stage: [128-byte header: the message's 16-byte meta][chunk]; fp8:
  // [header][e4m3 chunk/2][scales chunk/64][bf16 output chunk]
  // mode 3 adds the re-quantized output: [..][bf16 y chunk][e4m3 chunk/2][scales chunk/64]
  const uint32_t q_off = 128, s_off = 128 + chunk / 2, o_off = fp8 ? s_off + chunk / 64 : 128;
  const uint32_t oq_off = o_off + chunk, os_off = oq_off + chunk / 2;
  const uint32_t sstride = fp8c ? os_off + chunk / 64 : (fp8 ? o_off + chunk : 128 + chunk);
  char* stage = dsm + ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)warp * kTmaStages * sstride;

  const uint32_t P = e_local * n;
  const uint32_t* counts = reinterpret_cast<const uint32_t*>(v->win[L.win_counts].base[rank]);
  for (uint32_t i = tid; i < P; i += kTmaThreads) {
    const uint32_t c = gin::ld_acquire_sys32(counts + i);
    cnt[i] = c;
    pair_start[i] = c;
  }
  if (tid < kMoeWarps) warp_tot[tid] = 0;
  if (lane == 0) {
    for (int s = 0; s < kTmaStages; ++s) gin::tma::mbar_init(&ctl->bar[s], 1);
    gin::tma::fence_mbar_init();
  }
  __syncthreads();
  if (L.layout != 0) source_prefix<kTmaWarps>(cnt, src_prefix, n, e_local);
  // exclusive scan of P <= 1024 entries with 256 threads (4 per thread)
  {
    const uint32_t per = (P + kTmaThreads - 1) / kTmaThreads;
    const uint32_t lo = tid * per, hi = min(lo + per, P);
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
    if (tid == 0) pair_start[P] = total_msgs;
    __syncthreads();
  }

  MOE_STAMP(R, 1, 1);
  const char* recv = v->win[L.win_dispatch].base[rank];
  char* const* cbases = v->win[L.win_combine].base;
  const uint64_t items = (uint64_t)total_msgs * parts;
  const uint64_t gw = (uint64_t)b * kTmaWarps + warp, stride = (uint64_t)G * kTmaWarps;
  auto locate = [&](uint32_t m, uint32_t& lo_pair) -> const char* {
    uint32_t lo = 0, hi = P;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (pair_start[mid] <= m) lo = mid; else hi = mid;
    }
    lo_pair = lo;
    const uint32_t e_loc = lo / n, src = lo % n, slot = m - pair_start[lo];
    const uint64_t moff = L.layout == 0 ? (((uint64_t)e_loc * n + src) * T + slot) * dmsg
                                        : ((uint64_t)src * T * K + src_prefix[lo] + slot) * dmsg;
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
    const uint32_t pr = (uint32_t)reinterpret_cast<uint64_t>(ctl->dptr[s]);
    const uint32_t e = rank * e_local + pr / n, src = pr % n;
    const uint32_t len = tma_chunk_len(payload, chunk, p);
    char* sb = stage + (size_t)s * sstride;
    gin::tma::mbar_wait(&ctl->bar[s], (uint32_t)((j / kTmaStages) & 1));
    uint4* buf = reinterpret_cast<uint4*>(sb + o_off);
    {
      const uint32_t nv = len / 16;
      uint32_t i = lane;
      if (fp8) {  // expand: 8 codes -> one 16-byte bf16 vector; scale per 128 elements
        const float sc = 1.0f + (float)(e % 7u) / 8.0f, cc = ((float)(e % 9u) - 4.0f) / 16.0f;
        const uint2* qin = reinterpret_cast<const uint2*>(sb + q_off);
        const float* scl = reinterpret_cast<const float*>(sb + s_off);
        for (; i < nv; i += 32) buf[i] = fp8x8_transform(qin[i], scl[i / 16], sc, cc);
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
    if (fp8c) {  // re-quantize the expert output, 128 elements per warp step
      __syncwarp();
      for (uint32_t blk = 0; blk < len / 256; ++blk)
        fp8_quant_block(reinterpret_cast<const uint16_t*>(sb + o_off + blk * 256),
                        reinterpret_cast<uint8_t*>(sb + oq_off + blk * 128), reinterpret_cast<float*>(sb + os_off) + blk,
                        lane);
    }
    gin::tma::fence_proxy_async_shared();
    __syncwarp();
    if (lane == 0) {
      const uint4 meta = *reinterpret_cast<const uint4*>(sb);  // {src, token, k, tag}
      char* cdst = cbases[src] + ((uint64_t)meta.y * K + meta.z) * cmsg;
      if (fp8c) {
        gin::tma::store(cdst + (uint64_t)p * (chunk / 2), sb + oq_off, len / 2);
        gin::tma::store(cdst + H + (uint64_t)p * (chunk / 64), sb + os_off, len / 64);
      } else {
        gin::tma::store(cdst + (uint64_t)p * chunk, buf, len);
      }
      gin::tma::commit();
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
  }
  MOE_STAMP(R, 1, 2);

  arrive_last(R.ws + 1, (unsigned)(R.iteration * G), &is_last);
  if (is_last) {
    if (tid == 0) *grab_ctr = 0;  // every CTA is past its loop: ready for the next launch
    for (uint32_t sc = tid; sc < n * n_ctx; sc += kTmaThreads) {
      const uint32_t src = sc / n_ctx, ctx = sc % n_ctx;
      uint32_t c = 0;
      for (uint32_t e_loc = 0; e_loc < e_local; ++e_loc)
        if ((rank * e_local + e_loc) % n_ctx == ctx) c += cnt[e_loc * n + src];
      if (c) {
        if (src == rank) {  // own tokens: the reducer is on this GPU
          gin::fence_acq_rel_gpu();
          gin::red_relaxed_sys_add(gin.sub_cell(src, rank, e_local), c);
        } else {
          gin.release_signal_raw(src, e_local, c);
        }
      }
    }
  }
  MOE_STAMP(R, 1, 3);
  if (L.fuse_reduce) {
    // small launches: the source-side reduction right here (saves the second
    // launch); same arithmetic as moe_combine_reduce_kernel
    if (tid == 0) gin.wait_ge_signal(e_local, R.iteration * (uint64_t)T * K);
    __syncthreads();
    const char* crecv = v->win[L.win_combine].base[rank];
    const uint32_t nvec = payload / 16;
    const uint64_t ritems = (uint64_t)T * nvec, rstride = (uint64_t)G * kTmaThreads;
    for (uint64_t q = (uint64_t)b * kTmaThreads + tid; q < ritems; q += rstride) {
      const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
      uint4 y[KMAX];
#pragma unroll
      for (int k = 0; k < KMAX; ++k)
        if (k < (int)K && !fp8c) y[k] = gin::ld_nc_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i);
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
// this launch, so it needs no co-residency.
template <int KMAX, bool FP8C>
__global__ void __launch_bounds__(kMoeThreads, 2) moe_combine_reduce_kernel(MoeLaunch L, uint32_t /*chunk*/) {
  const MoeRankArgs& R = L.r[blockIdx.y];
  const GinDevCommView* v = R.view;
  gin::Gin gin(v, 0);
  const uint32_t rank = v->rank;
  const uint32_t K = L.K, T = L.T, H = L.H, e_local = L.e_local;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const uint64_t cmsg = L.cmsg;
  constexpr bool fp8c = FP8C;  // mode 3 (a separate instantiation keeps the bf16 path spill-free)
  const uint32_t payload = 2u * H;
  MOE_STAMP(R, 2, 0);
  if (tid == 0) gin.wait_ge_signal(e_local, R.iteration * (uint64_t)T * K);
  __syncthreads();
  MOE_STAMP(R, 2, 1);
  const char* crecv = v->win[L.win_combine].base[rank];
  const uint32_t nvec = payload / 16;
  const uint64_t ritems = (uint64_t)T * nvec, rstride = (uint64_t)G * kMoeThreads;
  for (uint64_t q = (uint64_t)b * kMoeThreads + tid; q < ritems; q += rstride) {
    const uint32_t t = (uint32_t)(q / nvec), i = (uint32_t)(q % nvec);
    if (fp8c) {
      gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
                 reduce_fp8_vec<KMAX>(crecv, cmsg, H, t, i, K, R.weights));
      continue;
    }
    uint4 y[KMAX];
#pragma unroll
    for (int k = 0; k < KMAX; ++k)
      if (k < (int)K) y[k] = gin::ld_nc_v4(crecv + ((uint64_t)t * K + k) * cmsg + 16ull * i);
    gin::st_v4(reinterpret_cast<char*>(R.out) + (uint64_t)t * payload + 16ull * i,
               reduce_vec<KMAX>(y, K, L.mode, R.weights, t));
  }
  MOE_STAMP(R, 2, 2);
}

// ------------------------------------------------------------------ synthetic inputs
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// route_token (harness_moe.cpp:25-30): std::mt19937_64 seeded with
// mix64(seed ^ mix64(src*100003 + token)), draws % E until K distinct, sorted.
__global__ void moe_route_kernel(int32_t* idx, uint64_t seed, uint32_t src, uint32_t T, uint32_t E, uint32_t K) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint64_t mt[312];
  mt[0] = mix64(seed ^ mix64((uint64_t)src * 100003ull + t));
  for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  int pos = 312;
  int32_t picked[32];
  uint32_t got = 0;
  while (got < K) {
    if (pos >= 312) {
      for (int i = 0; i < 312; ++i) {
        const uint64_t y = (mt[i] & 0xFFFFFFFF80000000ull) | (mt[(i + 1) % 312] & 0x7FFFFFFFull);
        uint64_t nv = mt[(i + 156) % 312] ^ (y >> 1);
        if (y & 1) nv ^= 0xB5026F5AA96619E9ull;
        mt[i] = nv;
      }
      pos = 0;
    }
    uint64_t x = mt[pos++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    const int32_t e = (int32_t)(x % E);
    uint32_t p = 0;
    while (p < got && picked[p] < e) ++p;
    if (p < got && picked[p] == e) continue;
    for (uint32_t j = got; j > p; --j) picked[j] = picked[j - 1];
    picked[p] = e;
    ++got;
  }
  for (uint32_t k = 0; k < K; ++k) idx[(uint64_t)t * K + k] = picked[k];
}

// token_element (harness_moe.cpp:32-34) or the bf16 generator.
__global__ void moe_tokens_kernel(uint16_t* x, uint64_t seed, uint32_t src, uint32_t T, uint32_t H, uint32_t mode) {
  const uint64_t total = (uint64_t)T * H;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < total; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(j / H), i = (uint32_t)(j % H);
    if (mode == 0) {
      x[j] = (uint16_t)(seed + src * 7919u + t * 131u + i * 13u);
    } else {
      const uint64_t h = mix64(seed ^ mix64(((uint64_t)src << 40) ^ ((uint64_t)t << 20) ^ i));
      const uint16_t sign = (uint16_t)((h >> 63) << 15);
      const uint16_t expo = (uint16_t)(120u + (uint32_t)((h >> 8) % 12u));
      x[j] = (uint16_t)(sign | (expo << 7) | (uint16_t)(h & 0x7Fu));
    }
  }
}

// combine_weight (harness_moe.cpp:40-42); bf16 mode uses w/8 as fp32.
__global__ void moe_weights_kernel(void* w, uint32_t src, uint32_t T, uint32_t K, uint32_t mode) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T * K) return;
  const uint32_t t = j / K, k = j % K;
  const uint16_t cw = (uint16_t)(1u + (src + 3u * t + 5u * k) % 7u);
  if (mode == 0) reinterpret_cast<uint16_t*>(w)[j] = cw;
  else reinterpret_cast<float*>(w)[j] = (float)cw / 8.0f;
}

}  // namespace ginsim_b200

// ------------------------------------------------------------------ C ABI
using namespace ginsim_b200;

struct ginsim_cuda_moe_s {
  Comm* comm = nullptr;
  ginsim_cuda_moe_config cfg{};
  uint32_t e_local = 0, parts = 4, G = 0, Gc = 0, Gr = 0, chunk = 0, cparts = 1, cchunk = 0;
  uint32_t win_dispatch = 0, win_counts = 0, win_combine = 0, win_stage = 0, win_cstage = 0, win_mirror = 0;
  bool proxy = false;
  void* buf_mirror = nullptr;
  uint32_t* midx = nullptr;
  uint32_t win_rows = 0;
  void* buf_rows = nullptr;
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
};

extern "C" {

int ginsim_cuda_moe_create(ginsim_cuda_comm_t comm, const ginsim_cuda_moe_config* cfg, ginsim_cuda_moe_t* out) {
  GIN_API_BEGIN
  Comm* c = &comm->impl;
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
  if (e_local + 1 > c->cfg.signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS)
    fail(GINSIM_E_USAGE, "per-expert signals plus the combine flag exceed the signal table");
  auto m = std::make_unique<ginsim_cuda_moe_s>();
  m->comm = c;
  m->cfg = *cfg;
  m->e_local = e_local;
  m->parts = cfg->hidden >= 1024 ? 4 : 1;
  const uint64_t dmsg = (cfg->mode >= 2 ? (uint64_t)cfg->hidden + cfg->hidden / 32 : 2ull * cfg->hidden) + 16;
  const uint64_t cmsg = cfg->mode == 3 ? (uint64_t)cfg->hidden + cfg->hidden / 32 : 2ull * cfg->hidden;
  const uint64_t n = c->world, T = cfg->tokens, K = cfg->top_k;
  const uint64_t dbytes = cfg->layout == 0 ? (uint64_t)e_local * n * T * dmsg : n * T * K * dmsg;
  if (cfg->layout == 2 && e_local + 2 > c->cfg.signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS)
    fail(GINSIM_E_USAGE, "per-expert signals plus the combine flag and rows cell exceed the signal table");
  const uint64_t nbytes = ((uint64_t)e_local * n + n) * 4;  // counts [e_loc][src] + row counts [src] (layout 2)
  const uint64_t cbytes = T * K * cmsg;
  if (ginsim_cuda_mem_alloc(comm, dbytes, &m->buf_dispatch)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
  if (ginsim_cuda_mem_alloc(comm, nbytes, &m->buf_counts)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
  if (ginsim_cuda_mem_alloc(comm, cbytes, &m->buf_combine)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
  int rc;
  if ((rc = ginsim_cuda_window_register(comm, m->buf_dispatch, dbytes, &m->win_dispatch))) fail(rc, ginsim_cuda_last_error());
  if ((rc = ginsim_cuda_window_register(comm, m->buf_counts, nbytes, &m->win_counts))) fail(rc, ginsim_cuda_last_error());
  if ((rc = ginsim_cuda_window_register(comm, m->buf_combine, cbytes, &m->win_combine))) fail(rc, ginsim_cuda_last_error());
  m->proxy = c->cfg.backend == GIN_BACKEND_PROXY;
  if (cfg->layout == 2) {
    // row staging: [src][j] rows of 2H bytes, then [src][j] 128-byte headers
    const uint64_t rbytes = n * T * (2ull * cfg->hidden + 128);
    if (ginsim_cuda_mem_alloc(comm, rbytes, &m->buf_rows)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if ((rc = ginsim_cuda_window_register(comm, m->buf_rows, rbytes, &m->win_rows))) fail(rc, ginsim_cuda_last_error());
    DeviceGuard dgr(c->device);
    GIN_CUDA(cudaMalloc(&m->aux_g, 2 * (size_t)T * ((K + 1) & ~1ull) * sizeof(uint64_t)));
  }
  if (m->proxy) {
    // Proxy backend: dispatch rows and combine results are staged in local
    // registered windows the host agent copies from (the reference's staging
    // windows, harness_moe.cpp:122-130).  Separate windows, so a combine never
    // overwrites rows the agent may still be copying out for the dispatch.
    const uint64_t sbytes = T * K * dmsg, cbytes2 = n * T * K * cmsg;
    if (ginsim_cuda_mem_alloc(comm, sbytes, &m->buf_stage)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if ((rc = ginsim_cuda_window_register(comm, m->buf_stage, sbytes, &m->win_stage))) fail(rc, ginsim_cuda_last_error());
    if (ginsim_cuda_mem_alloc(comm, cbytes2, &m->buf_cstage)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if ((rc = ginsim_cuda_window_register(comm, m->buf_cstage, cbytes2, &m->win_cstage))) fail(rc, ginsim_cuda_last_error());
    // combine results in send order ([dst][expert prefix][slot]): one put per run
    if (ginsim_cuda_mem_alloc(comm, cbytes2, &m->buf_mirror)) fail(GINSIM_E_CUDA, ginsim_cuda_last_error());
    if ((rc = ginsim_cuda_window_register(comm, m->buf_mirror, cbytes2, &m->win_mirror))) fail(rc, ginsim_cuda_last_error());
    DeviceGuard dgm(c->device);
    GIN_CUDA(cudaMalloc(&m->midx, (size_t)T * K * 4));
  }
  DeviceGuard g(c->device);
  GIN_CUDA(cudaMalloc(&m->ws, 256));
  GIN_CUDA(cudaMalloc(&m->route, (2 * (size_t)kMaxGrid + 1) * kMaxExperts * 4));
  GIN_CUDA(cudaMalloc(&m->dst_g, (size_t)cfg->tokens * ((cfg->top_k + 1) & ~1u) * sizeof(char*)));
  GIN_CUDA(cudaMemset(m->ws, 0, 256));
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
  *out = m.release();
  GIN_API_END
}

int ginsim_cuda_moe_destroy(ginsim_cuda_moe_t moe) {
  GIN_API_BEGIN
  if (!moe) return GINSIM_OK;
  {
    DeviceGuard g(moe->comm->device);
    cudaDeviceSynchronize();
    if (moe->ws) cudaFree(moe->ws);
    if (moe->route) cudaFree(moe->route);
    if (moe->midx) cudaFree(moe->midx);
    if (moe->aux_g) cudaFree(moe->aux_g);
    if (moe->dst_g) cudaFree(moe->dst_g);
    if (moe->prof) cudaFree(moe->prof);
  }
  // window memory stays mapped until the comm is destroyed (windows are
  // never deregistered in the reference either).
  delete moe;
  GIN_API_END
}

int ginsim_cuda_moe_windows(ginsim_cuda_moe_t moe, uint32_t* d, uint32_t* c, uint32_t* cb) {
  if (d) *d = moe->win_dispatch;
  if (c) *c = moe->win_counts;
  if (cb) *cb = moe->win_combine;
  return GINSIM_OK;
}

int ginsim_cuda_moe_generate(ginsim_cuda_moe_t moe, uint64_t seed, uint32_t src, void* x, int32_t* idx, void* w,
                             void* stream) {
  GIN_API_BEGIN
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
  L.fuse_reduce = moes[0]->coop ? 0u : 1u;
  L.mpay = cfg.mode >= 2 ? cfg.hidden + cfg.hidden / 32 : 2u * cfg.hidden;
  L.dmsg = (uint64_t)L.mpay + 16;
  L.cmsg = cfg.mode == 3 ? (uint64_t)cfg.hidden + cfg.hidden / 32 : 2ull * cfg.hidden;
  for (uint32_t i = 0; i < n; ++i) {
    if (std::memcmp(&moes[i]->cfg, &cfg, sizeof(cfg)) != 0 || moes[i]->win_dispatch != L.win_dispatch)
      fail(GINSIM_E_USAGE, "moe handles in one launch must share a config");
    L.r[i].view = moes[i]->comm->dev_view;
    L.r[i].ws = moes[i]->ws;
    L.r[i].route = moes[i]->route;
    L.r[i].dst_g = moes[i]->dst_g;
    L.r[i].midx = moes[i]->midx;
    L.r[i].aux_g = moes[i]->aux_g;
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
  int threads;           // of dispatch / combine
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
  if (e == 1 && m->proxy) {
    k.dispatch = k8 ? (const void*)moe_dispatch_kernel<8, true> : (const void*)moe_dispatch_kernel<32, true>;
    k.combine = (const void*)moe_combine_kernel<true>;
    k.threads = kMoeThreads;
    return k;
  }
  if (e == 1) {
    k.dispatch = k8 ? (const void*)moe_dispatch_kernel<8, false> : (const void*)moe_dispatch_kernel<32, false>;
    k.combine = (const void*)moe_combine_kernel<false>;
    k.threads = kMoeThreads;
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
  } else {
    k.combine = k8 ? (const void*)moe_combine_tma_kernel<8> : (const void*)moe_combine_tma_kernel<32>;
    if (m->cfg.mode == 3)
      k.reduce = k8 ? (const void*)moe_combine_reduce_kernel<8, true> : (const void*)moe_combine_reduce_kernel<32, true>;
    else
      k.reduce = k8 ? (const void*)moe_combine_reduce_kernel<8, false> : (const void*)moe_combine_reduce_kernel<32, false>;
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
  if (m->cfg.mode >= 2) {  // + e4m3 chunk + scales per stage
    const size_t sst = (dhead + m->chunk + m->chunk / 2 + m->chunk / 64 + 15) & ~(size_t)15;
    return ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)kTmaWarps * kDispStages * sst + pairs * 4;
  }
  const size_t tokens = (size_t)((m->cfg.tokens + G - 1) / G + 1);
  const size_t rowj = m->cfg.layout == 2 ? tokens * m->comm->world * 4 : 0;  // dedup: (t, dst) row indices
  return ((sizeof(TmaSmem) * kTmaWarps + 127) & ~(size_t)127) + (size_t)kTmaWarps * kDispStages * (dhead + m->chunk) +
         pairs * 4 + rowj;
}
static size_t combine_smem(const ginsim_cuda_moe_t m) {
  if (!kernels_of(m).tma_combine) return 0;
  // fp8: [hdr][e4m3 in][scales][bf16 out] per stage
  const size_t c = m->cchunk;
  const size_t sst = m->cfg.mode == 3 ? 128 + 2 * (c / 2 + c / 64) + c
                                      : (m->cfg.mode == 2 ? 128 + c / 2 + c / 64 + c : 128 + c);
  return ((sizeof(TmaSmem) * kCmbWarps + 127) & ~(size_t)127) + (size_t)kCmbWarps * kTmaStages * sst;
}
static int combine_threads(const MoeKernels& k) { return k.tma_combine ? kCmbThreads : kMoeThreads; }

static void plan(const ginsim_cuda_moe_t* moes, uint32_t n) {
  ginsim_cuda_moe_t m = moes[0];
  if (m->G) return;
  const MoeKernels k = kernels_of(m);
  const uint32_t payload = 2u * m->cfg.hidden;
  uint32_t parts = 1, chunk = 0, cparts = 1, cchunk = 0;
  if (use_tma(m)) {
    parts = (payload + 8191) / 8192;
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
      cchunk = 2048;  // combine stages also hold the expanded bf16 output
      cparts = (payload + cchunk - 1) / cchunk;
    }
    m->chunk = chunk;
    m->cchunk = cchunk;
  }
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
  if (k.reduce) Gr = std::max<uint32_t>(1, (uint32_t)max_coresident_ctas(k.reduce, kMoeThreads, 0, m->comm->device) / n);
  if (!use_tma(m) || !k.tma_combine) {
    // LSU combine: (message, part) work items sized to the warp count
    const uint32_t nvec = payload % 16u == 0 ? payload / 16u : 0u;
    if (nvec >= 32 && !k.tma_dispatch) {
      const uint32_t want = (2u * Gd * kMoeWarps + m->cfg.tokens - 1) / m->cfg.tokens;
      parts = std::max(1u, std::min(want, nvec / 32u));
    }
  }
  for (uint32_t i = 0; i < n; ++i) {
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
  for (uint32_t i = 1; i < n; ++i)
    if (moes[i]->comm->device != moes[0]->comm->device) fail(GINSIM_E_USAGE, "emulated ranks must share a device");
}

int ginsim_cuda_moe_dispatch(const ginsim_cuda_moe_t* moes, uint32_t n, const void* const* x,
                             const int32_t* const* idx, void* stream) {
  GIN_API_BEGIN
  check_launch_set(moes, n);
  MoeLaunch L = make_launch(moes, n);
  DeviceGuard g(moes[0]->comm->device);
  plan(moes, n);
  const MoeKernels k = kernels_of(moes[0]);
  L.parts = moes[0]->parts;
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
  void* args[] = {&L, &chunk};
  const uint32_t Gc = moes[0]->Gc;
  launch_coop(k.combine, Gc, n, combine_threads(k), combine_smem(moes[0]), args, (cudaStream_t)stream);
  if (k.reduce && !L.no_wait && !L.fuse_reduce) {  // profiling harness: the reduce would wait on every source's flag
    GIN_CUDA(cudaLaunchKernel(k.reduce, dim3(moes[0]->Gr, n), dim3(kMoeThreads), args, 0, (cudaStream_t)stream));
  }
  moes[0]->last_ctas = Gc * n;
  GIN_API_END
}

int ginsim_cuda_moe_phase_times(ginsim_cuda_moe_t moe, uint32_t kernel, uint64_t* out, uint32_t* ctas) {
  GIN_API_BEGIN
  if (!moe->prof) fail(GINSIM_E_USAGE, "phase stamps need GINSIM_PROFILE_PHASES=1 at moe_create");
  if (kernel > 2) fail(GINSIM_E_USAGE, "kernel: 0 dispatch, 1 combine send, 2 combine reduce");
  DeviceGuard g(moe->comm->device);
  GIN_CUDA(cudaDeviceSynchronize());
  GIN_CUDA(cudaMemcpy(out, moe->prof + (uint64_t)kernel * 1024 * 8, 1024 * 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost));
  if (ctas) *ctas = kernel == 0 ? moe->G : (kernel == 1 ? moe->Gc : moe->Gr);
  GIN_API_END
}

int ginsim_cuda_moe_last_launch(ginsim_cuda_moe_t moe, uint32_t* ctas, uint32_t* threads) {
  if (ctas) *ctas = moe->last_ctas;
  if (threads) *threads = (uint32_t)kernels_of(moe).threads;
  return GINSIM_OK;
}

}  // extern "C"

extern "C" int ginsim_cuda_moe_create_all(const ginsim_cuda_comm_t* comms, uint32_t n,
                                          const ginsim_cuda_moe_config* cfg, ginsim_cuda_moe_t* out) {
  GIN_API_BEGIN
  std::vector<int> rcs(n, 0);
  std::vector<std::string> msgs(n);
  std::vector<std::thread> ts;
  for (uint32_t r = 0; r < n; ++r) {
    ts.emplace_back([&, r] {
      rcs[r] = ginsim_cuda_moe_create(comms[r], cfg, &out[r]);
      if (rcs[r]) msgs[r] = ginsim_cuda_last_error();
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < n; ++r)
    if (rcs[r]) fail(rcs[r], "rank " + std::to_string(r) + ": " + msgs[r]);
  GIN_API_END
}
