// moe_common.cuh -- launch structs, constants and device helpers of the MoE kernels.
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
#pragma once

namespace ginsim_b200 {


constexpr int kMoeThreads = 512;
constexpr int kMoeWarps = kMoeThreads / 32;
constexpr uint32_t kMaxExperts = 1024;
constexpr uint32_t kMaxGrid = 1024;  // CTAs per rank of one launch
constexpr uint32_t kDedupChunks = 4;      // layout 2: row chunks per source (moe_dedup.cuh)
constexpr uint32_t kCombineChunks = 8;    // pipelined combine: at most this many source-token chunks
constexpr uint32_t kEarlyRedSms = 64;     // pipelined combine: SMs the send kernel leaves to the early reducer
constexpr size_t kWsBytes = 512;          // per-handle workspace words (MoeRankArgs::ws); [64, 64 + kCombineChunks) chunk arrivals

struct MoeRankArgs {
  const GinDevCommView* view;
  unsigned int* ws;           // per-moe arrival counters [0] dispatch [1] combine [2] slot barrier
  uint32_t* route;            // TMA dispatch scratch: hist [kMaxGrid][E], prefix [kMaxGrid][E], totals [E]
  char** dst_g;               // TMA dispatch: [T][Kp] destination pointer of every (t, k) pair
  uint32_t* midx;             // proxy: [T][K] index of (t, k)'s result in the combine mirror window
  uint64_t* aux_g;            // layout 2: [2][T][Kp] row-header address and (slot, e_loc) per pair
  uint32_t* pipe;             // proxy pipeline: [T*K] staging position -> pair, then chunk counters
  const uint16_t* x;          // [T][H]
  const int32_t* idx;         // [T][K]
  const void* weights;        // [T][K] u16 (mode 0) / f32 (mode 1)
  uint16_t* out;              // [T][H]
  uint64_t iteration;         // 1-based
  uint64_t* cell_acc;         // [e_local] counts consumed by earlier iterations per local expert cell
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
  uint32_t share;                // TMA dispatch, every rank of the comm in this launch (emulated): after their
                                 // static first round, warps take tokens of ANY lane from one launch-wide counter
  uint32_t stage_ctas;           // Proxy pipeline: CTAs that stage (the rest leave the copy engines the HBM)
  uint32_t fanout_ctas;          // layout 2: CTAs that fan received rows out while the others put (0 = all, in turn)
  uint32_t cell0;                // first signal cell of this handle: expert cells, combine flag, rows/chunk cells
  uint32_t cchunks;              // pipelined combine: source-token chunks C (0 = one combine flag at the end)
  uint32_t dgrid;                // dispatch grid (CTAs per rank): chunk c = the tokens of CTAs [c*dgrid/C, ...)
  uint32_t red_first, red_last;  // reduce launch: chunks [red_first, red_last) (pipelined combine)
};

// Pipelined combine (L.cchunks = C > 1; one rank per GPU, cooperative route
// tables).  Source tokens are cut into C chunks aligned with the dispatch's
// CTA token ranges (combine_chunk_cta), so chunk c's slot bound for expert e
// is the prefix row g_pre[first CTA of c][e] the route tables already hold.  The dispatch's
// releasing CTA writes those bounds next to the counts; the combine's send
// kernel then walks its messages chunk-major, and whoever completes chunk
// c's sends releases cell e_local + 3 + kDedupChunks + c at each source by
// the number of messages it sent there.  The source reduces chunk c once
// the cell holds iteration * tokens(c) * K -- chunks 0..C-2 by a reducer on
// kEarlyRedSms SMs the send kernel leaves free, started while it runs
// (programmatic dependent launch), the last chunk by the full-occupancy
// reducer after it.
// First dispatch CTA of chunk c: equal chunks.  (A last chunk half as long,
// so less is left for after the send kernel, measured worse -- N=2 combine
// 402 vs 392 us: the early reducer then still holds the larger third chunk
// when the send ends.)
__device__ __forceinline__ uint32_t combine_chunk_cta(uint32_t c, uint32_t C, uint32_t G) {
  return c >= C ? G : c * G / C;
}
__device__ __forceinline__ uint32_t combine_chunk_t0(uint32_t c, uint32_t C, uint32_t dgrid, uint32_t T) {
  return c >= C ? T : (uint32_t)((uint64_t)combine_chunk_cta(c, C, dgrid) * T / dgrid);
}
// count-window offset (u32 words) of the bounds: [src][c-1][e_loc] for c = 1..C-1
__device__ __forceinline__ uint64_t combine_bounds_index(uint32_t n, uint32_t e_local, uint32_t src, uint32_t c,
                                                         uint32_t C) {
  return (uint64_t)e_local * n + n + (uint64_t)n * (kDedupChunks + 1) + ((uint64_t)src * (C - 1) + (c - 1)) * e_local;
}
__device__ __forceinline__ uint32_t combine_chunk_cell(uint32_t cell0, uint32_t e_local, uint32_t c) {
  return cell0 + e_local + 3 + kDedupChunks + c;
}

// Per-handle launch counters in device memory (ws words 56..59: [0]
// dispatch, [1] combine).  A dispatch/combine launch's iteration is the
// stored value + 1 (read by every CTA at its start); the CTA that completes
// the launch's grid-wide arrival -- after every CTA has read it -- stores it
// back.  The host therefore passes no per-launch value, and a step captured
// in a CUDA graph advances on every replay.
__device__ __forceinline__ uint64_t* moe_iter_ptr(const MoeRankArgs& R, int kind) {
  return reinterpret_cast<uint64_t*>(R.ws + 56) + kind;
}
__device__ __forceinline__ uint64_t moe_iteration(const MoeRankArgs& R, int kind, bool next) {
  return *reinterpret_cast<volatile uint64_t*>(moe_iter_ptr(R, kind)) + (next ? 1u : 0u);
}

// Acquire local expert e_loc's dispatch cell for `iteration` (one thread).
// The cell accumulates (n<<32) + count per source per iteration
// (harness_moe.cpp:163-167) and is never reset, so once the counts of all
// iterations sum past 2^32 they carry into the arrival field, and a bare
// "cell >= it*(n<<32)" would pass before every source has released.  The
// target therefore adds the counts consumed by earlier iterations
// (cell_acc): cell >= it*(n<<32) + acc holds only when all n sources of this
// iteration have released (one iteration's counts stay below 2^32), and the
// value read after the wait advances acc exactly (modular arithmetic).
__device__ __forceinline__ void acquire_expert_cell(const gin::Gin& gin, const MoeRankArgs& R, uint32_t cell,
                                                    uint32_t e_loc, uint64_t iteration, uint32_t n) {
  const uint64_t arrivals = iteration * ((uint64_t)n << 32);
  const uint64_t acc = R.cell_acc[e_loc];
  gin.wait_ge_signal(cell, arrivals + acc);
  R.cell_acc[e_loc] = gin.read_signal(cell) - arrivals;
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t u16x2_transform(uint32_t two, uint32_t add) {
  // two u16 lanes: y = 3x + (17e+1), each lane mod 2^16
  const uint32_t lo = ((two & 0xFFFFu) * 3u + add) & 0xFFFFu;
  const uint32_t hi = ((two >> 16) * 3u + add) & 0xFFFFu;
  return lo | (hi << 16);
}

// 8 bf16 lanes: y = bf16(fp32(x)*s + c), single-rounded mul and add, packed
// back two at a time (cvt.rn.bf16x2.f32) -- same rounding as bf16x2_transform.
// The pair's multiply goes through the sm_100 packed fp32 pipe (FMUL2: each
// lane an IEEE rn multiply).  The add stays scalar: ptxas 12.9 contracts a
// mul.rn.f32x2 + add.rn.f32x2 pair into FFMA2 (single rounding -- measured in
// SASS), which would break bit-exactness; a scalar FADD after FMUL2 is kept.
__device__ __forceinline__ float2 mul_add2_rn(float2 v, float s, float c) {
  const float2 m = __fmul2_rn(v, make_float2(s, s));
  return make_float2(__fadd_rn(m.x, c), __fadd_rn(m.y, c));
}
__device__ __forceinline__ uint32_t bf16x2_transform(uint32_t two, float s, float c) {
  const float2 y = mul_add2_rn(make_float2(__uint_as_float(two << 16), __uint_as_float(two & 0xFFFF0000u)), s, c);
  const __nv_bfloat16 ya = __float2bfloat16_rn(y.x), yb = __float2bfloat16_rn(y.y);
  return (uint32_t)__bfloat16_as_ushort(ya) | ((uint32_t)__bfloat16_as_ushort(yb) << 16);
}

__device__ __forceinline__ uint32_t bf16x2_pack_transform(uint32_t two, float s, float c) {
  const float2 y = mul_add2_rn(make_float2(__uint_as_float(two << 16), __uint_as_float(two & 0xFFFF0000u)), s, c);
  const __nv_bfloat162 r = __floats2bfloat162_rn(y.x, y.y);  // .x = low half, .y = high half
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
  const float2 iv = make_float2(inv, inv);
  const __nv_fp8x2_storage_t lo =
      __nv_cvt_float2_to_fp8x2(__fmul2_rn(make_float2(f[0], f[1]), iv), __NV_SATFINITE, __NV_E4M3);
  const __nv_fp8x2_storage_t hi =
      __nv_cvt_float2_to_fp8x2(__fmul2_rn(make_float2(f[2], f[3]), iv), __NV_SATFINITE, __NV_E4M3);
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
    const float2 y = mul_add2_rn(__fmul2_rn(f, make_float2(scale, scale)), s, c);
    const __nv_bfloat162 r = __floats2bfloat162_rn(y.x, y.y);
    out[h] = *reinterpret_cast<const uint32_t*>(&r);
  }
  return make_uint4(out[0], out[1], out[2], out[3]);
}

// Mode-2 combine: a lane holds at most this many 8-code vectors of a chunk
// (chunk <= 4096 payload bytes = 256 vectors over 32 lanes).
constexpr int kFp8MaxVec = 8;

// Mode-3 combine, one lane's 16 elements of a 128-element block (8 lanes per
// block): the same arithmetic as fp8x8_transform + fp8_quant_block -- y =
// bf16(deq*s + c), block amax over the bf16 values, scale = amax/448 and
// codes = e4m3(y * (448/amax)), all single-rounded -- kept in registers; the
// codes overwrite the lane's own 16 input codes.
__device__ __forceinline__ void fp8_requant16(uint4* cp, uint4 codes, float scale_in, float s, float c,
                                              float* scale_out, uint32_t sub8) {
  const uint4 y0 = fp8x8_transform(make_uint2(codes.x, codes.y), scale_in, s, c);
  const uint4 y1 = fp8x8_transform(make_uint2(codes.z, codes.w), scale_in, s, c);
  const uint32_t w[8] = {y0.x, y0.y, y0.z, y0.w, y1.x, y1.y, y1.z, y1.w};
  float f[16];
#pragma unroll
  for (int h = 0; h < 8; ++h) {
    f[2 * h] = __uint_as_float(w[h] << 16);
    f[2 * h + 1] = __uint_as_float(w[h] & 0xFFFF0000u);
  }
  float amax = 0.0f;
#pragma unroll
  for (int h = 0; h < 16; ++h) amax = fmaxf(amax, fabsf(f[h]));
#pragma unroll
  for (int o = 4; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const float scale = amax > 0.0f ? __fdiv_rn(amax, 448.0f) : 1.0f;
  const float inv = amax > 0.0f ? __fdiv_rn(448.0f, amax) : 1.0f;
  uint32_t q[4];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const float2 iv = make_float2(inv, inv);
    const __nv_fp8x2_storage_t lo =
        __nv_cvt_float2_to_fp8x2(__fmul2_rn(make_float2(f[4 * h], f[4 * h + 1]), iv), __NV_SATFINITE, __NV_E4M3);
    const __nv_fp8x2_storage_t hi =
        __nv_cvt_float2_to_fp8x2(__fmul2_rn(make_float2(f[4 * h + 2], f[4 * h + 3]), iv), __NV_SATFINITE, __NV_E4M3);
    q[h] = (uint32_t)lo | ((uint32_t)hi << 16);
  }
  *cp = make_uint4(q[0], q[1], q[2], q[3]);
  if (sub8 == 0) *scale_out = scale;
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
// Count window: cnt[src][e_loc] u32 (source-major, so one source's counts
// for a destination's experts are one contiguous run -- a single put on the
// Proxy backend), then the dedup row counts [src] at e_local*n.  Kernels scan
// (e_loc, src) pairs in e_loc-major order (harness_moe.cpp:174-179): pair i
// = e_loc*n + src lives at count_index(i).
__device__ __forceinline__ uint32_t count_index(uint32_t i, uint32_t n, uint32_t e_local) {
  return (i % n) * e_local + i / n;
}

__device__ __forceinline__ void release_experts(const gin::Gin& gin, const GinDevCommView* v, uint32_t win_counts,
                                                const uint32_t* hist, uint32_t n, uint32_t rank, uint32_t e_local,
                                                uint32_t cell0, uint32_t C = 0, const uint32_t* g_pre = nullptr,
                                                uint32_t pre_stride = 0, uint32_t G = 0) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (uint32_t d = warp; d < n; d += nw) {
    uint32_t* cb = reinterpret_cast<uint32_t*>(v->win[win_counts].base[d]);
    // the counts need no ordering against the puts, only before the cells:
    // one fence between them releases both the puts (by cumulativity) and
    // the counts; for own experts the acquirer is on this GPU (GPU scope)
    for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
      gin::st_relaxed_sys32(cb + (uint64_t)rank * e_local + e_loc, hist[d * e_local + e_loc]);
    // pipelined combine: the slot bound of every source-token chunk (the
    // prefix row of the chunk's first CTA), released by the same fence
    for (uint32_t c = 1; c < C; ++c)
      for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
        gin::st_relaxed_sys32(cb + combine_bounds_index(n, e_local, rank, c, C) + e_loc,
                              __ldcg(g_pre + (size_t)combine_chunk_cta(c, C, G) * pre_stride + d * e_local + e_loc));
    gin.fence_toward(d);  // (own experts and emulated peers: GPU scope)
    for (uint32_t e_loc = lane; e_loc < e_local; e_loc += 32)
      gin::red_relaxed_sys_add(gin.sub_cell(d, rank, cell0 + e_loc), (1ull << 32) + hist[d * e_local + e_loc]);
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

}  // namespace ginsim_b200
