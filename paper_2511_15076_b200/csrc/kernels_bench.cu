// kernels_bench.cu — raw NVLink / HBM copy engines used as roofline probes:
// the same put path the MoE kernels use (128-bit LSU stores or TMA bulk
// copies staged through shared memory) over one window region into a peer's
// (or the local) window, no signals.  Gives the measured NVLink write floor
// that BASELINE's "fraction of 900 GB/s" sits next to.
#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <vector>

#include "gin_device.cuh"
#include "runtime_internal.h"
#include "tma.cuh"

namespace ginsim_b200 {

constexpr int kCopyThreads = 256;
constexpr int kCopyStages = 4;

__global__ void __launch_bounds__(kCopyThreads) lsu_copy_kernel(char* dst, const char* src, uint64_t bytes) {
  const uint64_t nv = bytes / 16;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < nv; i += 4 * stride) {
    const uint4 a = gin::ld_nc_v4(src + 16 * i), b = gin::ld_nc_v4(src + 16 * (i + stride));
    const uint4 c = gin::ld_nc_v4(src + 16 * (i + 2 * stride)), d = gin::ld_nc_v4(src + 16 * (i + 3 * stride));
    gin::st_v4(dst + 16 * i, a);
    gin::st_v4(dst + 16 * (i + stride), b);
    gin::st_v4(dst + 16 * (i + 2 * stride), c);
    gin::st_v4(dst + 16 * (i + 3 * stride), d);
  }
  for (; i < nv; i += stride) gin::st_v4(dst + 16 * i, gin::ld_nc_v4(src + 16 * i));
}

// One pipeline per warp (lane 0 drives it): kCopyStages chunks in flight,
// TMA load global->smem on an mbarrier, TMA store smem->dst.
__global__ void __launch_bounds__(kCopyThreads) tma_copy_kernel(char* dst, const char* src, uint64_t bytes,
                                                              uint32_t chunk) {
  extern __shared__ __align__(128) char smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * kCopyStages;
  char* buf = smem + 1024 + (size_t)warp * kCopyStages * chunk;
  const uint64_t total = (bytes + chunk - 1) / chunk;
  const uint64_t gw = (uint64_t)blockIdx.x * nw + warp, stride = (uint64_t)gridDim.x * nw;
  if (lane != 0) return;
  for (int s = 0; s < kCopyStages; ++s) gin::tma::mbar_init(bars + s, 1);
  gin::tma::fence_mbar_init();
  auto len = [&](uint64_t c) { return (uint32_t)std::min<uint64_t>(chunk, bytes - c * chunk); };
  for (int s = 0; s < kCopyStages; ++s) {
    const uint64_t c = gw + s * stride;
    if (c < total) {
      gin::tma::mbar_arrive_expect_tx(bars + s, len(c));
      gin::tma::load(buf + (size_t)s * chunk, src + c * chunk, len(c), bars + s);
    }
  }
  for (uint64_t i = 0;; ++i) {
    const uint64_t c = gw + i * stride;
    if (c >= total) break;
    const int s = (int)(i % kCopyStages);
    gin::tma::mbar_wait(bars + s, (uint32_t)((i / kCopyStages) & 1));
    gin::tma::store(dst + c * chunk, buf + (size_t)s * chunk, len(c));
    gin::tma::commit();
    gin::tma::wait_read<0>();
    const uint64_t cn = c + kCopyStages * stride;
    if (cn < total) {
      gin::tma::mbar_arrive_expect_tx(bars + s, len(cn));
      gin::tma::load(buf + (size_t)s * chunk, src + cn * chunk, len(cn), bars + s);
    }
  }
  gin::tma::wait_all();
}

// 256-bit LSU copy (LDG/STG .256 on sm_100a): half the instructions of the
// 128-bit path for the same bytes in flight.
__global__ void __launch_bounds__(kCopyThreads) lsu256_copy_kernel(char* dst, const char* src, uint64_t bytes) {
  const uint64_t nv = bytes / 32;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + stride < nv; i += 2 * stride) {
    const gin::u32x8 a = gin::ld_nc_v8(src + 32 * i), b = gin::ld_nc_v8(src + 32 * (i + stride));
    gin::st_v8(dst + 32 * i, a);
    gin::st_v8(dst + 32 * (i + stride), b);
  }
  for (; i < nv; i += stride) gin::st_v8(dst + 32 * i, gin::ld_nc_v8(src + 32 * i));
}

// Store-only TMA: every warp bulk-stores one shared-memory chunk over and
// over to consecutive destination chunks -- no HBM reads, so it measures the
// write path (NVLink egress or HBM write) alone.
__global__ void __launch_bounds__(kCopyThreads) tma_store_only_kernel(char* dst, uint64_t bytes, uint32_t chunk) {
  extern __shared__ __align__(128) char smem[];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  char* buf = smem + (size_t)warp * chunk;
  for (uint32_t i = lane * 16; i < chunk; i += 32 * 16) *reinterpret_cast<uint4*>(buf + i) = make_uint4(i, warp, 1, 2);
  gin::tma::fence_proxy_async_shared();
  __syncwarp();
  if (lane != 0) return;
  const uint64_t total = (bytes + chunk - 1) / chunk;
  const uint64_t gw = (uint64_t)blockIdx.x * nw + warp, stride = (uint64_t)gridDim.x * nw;
  uint32_t n = 0;
  for (uint64_t c = gw; c < total; c += stride) {
    gin::tma::store(dst + c * chunk, buf, (uint32_t)std::min<uint64_t>(chunk, bytes - c * chunk));
    gin::tma::commit();
    if (++n >= 8) gin::tma::wait_read<8>();
  }
  gin::tma::wait_all();
}

// Occupies every SM (ctas_per_sm CTAs of 1024 threads each) until the
// host-mapped release word becomes nonzero: used to check that the proxy
// agent's copies and stream memops progress while a persistent kernel holds
// the whole GPU (they must run on the copy engines / front end, not on SMs).
__global__ void __launch_bounds__(1024) occupy_kernel(const volatile uint32_t* release, uint64_t timeout_ns) {
  if (threadIdx.x == 0) {
    const uint64_t t0 = gin::globaltimer();
    while (*release == 0 && gin::globaltimer() - t0 < timeout_ns) __nanosleep(1000);
  }
  __syncthreads();
}

__global__ void spin_kernel(uint64_t ns) {
  const uint64_t t0 = gin::globaltimer();
  while (gin::globaltimer() - t0 < ns) __nanosleep(1000);
}

}  // namespace ginsim_b200

using namespace ginsim_b200;

extern "C" {

// Copies `bytes` from this rank's src window (offset 0) into `peer`'s dst
// window (offset 0) `iters` times; engine 0 = LSU 128-bit stores, 1 = TMA
// bulk.  Returns the mean milliseconds per copy (CUDA events on `stream`).
int ginsim_cuda_copy_bench(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                           uint64_t bytes, uint32_t engine, uint32_t ctas, uint32_t iters, float* ms_out,
                           void* stream) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->window_live(src_win) || !c->window_live(dst_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
  if (peer >= c->world) fail(GINSIM_E_INVALID_PEER, "peer out of range");
  if (c->windows[src_win].sizes[c->rank] < bytes || c->windows[dst_win].sizes[peer] < bytes)
    fail(GINSIM_E_OUT_OF_BOUNDS, "copy exceeds window capacity");
  if (bytes % 16) fail(GINSIM_E_USAGE, "copy size must be a multiple of 16");
  DeviceGuard g(c->device);
  char* dst = c->windows[dst_win].bases[peer];
  const char* src = c->windows[src_win].bases[c->rank];
  cudaStream_t s = (cudaStream_t)stream;
  int sms = 0;
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const uint32_t G = ctas ? ctas : (uint32_t)sms;
  const uint32_t tchunk = 4096;
  const size_t smem = 1024 + (size_t)(kCopyThreads / 32) * kCopyStages * tchunk;
  if (engine == 1) {
    GIN_CUDA(cudaFuncSetAttribute((const void*)tma_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  }
  cudaEvent_t e0, e1;
  GIN_CUDA(cudaEventCreate(&e0));
  GIN_CUDA(cudaEventCreate(&e1));
  auto launch = [&] {
    if (engine == 0) lsu_copy_kernel<<<G, kCopyThreads, 0, s>>>(dst, src, bytes);
    else tma_copy_kernel<<<G, kCopyThreads, smem, s>>>(dst, src, bytes, tchunk);
  };
  launch();
  GIN_CUDA(cudaGetLastError());
  GIN_CUDA(cudaEventRecord(e0, s));
  for (uint32_t i = 0; i < iters; ++i) launch();
  GIN_CUDA(cudaEventRecord(e1, s));
  GIN_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  GIN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *ms_out = ms / (float)std::max(1u, iters);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  GIN_API_END
}

// Extended probe: engine 0 = LSU 128-bit, 1 = TMA load+store (chunk bytes,
// 4 stages per warp), 2 = LSU 256-bit, 3 = copy engine (cudaMemcpyAsync over
// the peer mapping), 4 = TMA store-only (no reads).
// chunk = TMA chunk bytes; CTAs of 256 threads.
int ginsim_cuda_copy_bench_ex(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                              uint64_t bytes, uint32_t engine, uint32_t ctas, uint32_t chunk, uint32_t iters,
                              float* ms_out, void* stream) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->window_live(src_win) || !c->window_live(dst_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
  if (peer >= c->world) fail(GINSIM_E_INVALID_PEER, "peer out of range");
  if (c->windows[src_win].sizes[c->rank] < bytes || c->windows[dst_win].sizes[peer] < bytes)
    fail(GINSIM_E_OUT_OF_BOUNDS, "copy exceeds window capacity");
  if (bytes % 32 || engine > 8) fail(GINSIM_E_USAGE, "copy size must be a multiple of 32; engine 0..8");
  if (chunk == 0 || chunk % 16 || chunk > 16384) fail(GINSIM_E_USAGE, "chunk must be a multiple of 16 in 16..16384");
  DeviceGuard g(c->device);
  // engines 5/7 pull: read the peer's src window, write this rank's dst window
  const bool pull = engine == 5 || engine == 7;
  if (pull && (c->windows[src_win].sizes[peer] < bytes || c->windows[dst_win].sizes[c->rank] < bytes))
    fail(GINSIM_E_OUT_OF_BOUNDS, "copy exceeds window capacity");
  char* dst = c->windows[dst_win].bases[pull ? c->rank : peer];
  const char* src = c->windows[src_win].bases[pull ? peer : c->rank];
  // engine 6: the copy engine moves the last GINSIM_HYBRID_CE_PCT percent
  // (default 25) on a side stream while TMA copies the rest
  uint64_t ce_bytes = 0;
  if (engine == 6) {
    const char* e = std::getenv("GINSIM_HYBRID_CE_PCT");
    const uint64_t pct = std::min<uint64_t>(100, e ? std::strtoull(e, nullptr, 10) : 25);
    ce_bytes = (bytes * pct / 100) & ~uint64_t(4095);
  }
  const uint64_t sm_bytes = bytes - ce_bytes;
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  // engine 8: copy engine toward EVERY other rank at once, one stream per peer
  // (bytes / (world-1) each, from disjoint slices): do peer copies overlap?
  std::vector<cudaStream_t> ps;
  std::vector<cudaEvent_t> pj;
  if (engine == 8) {
    if (c->world < 2) fail(GINSIM_E_USAGE, "engine 8 needs peers");
    for (uint32_t q = 0; q + 1 < c->world; ++q) {
      cudaStream_t st;
      cudaEvent_t ev;
      GIN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
      GIN_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      ps.push_back(st);
      pj.push_back(ev);
    }
    GIN_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
  }
  if (engine == 6) {
    GIN_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    GIN_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    GIN_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
  }
  cudaStream_t s = (cudaStream_t)stream;
  int sms = 0;
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
  const uint32_t G = ctas ? ctas : (uint32_t)sms;
  const size_t smem_ld = 1024 + (size_t)(kCopyThreads / 32) * kCopyStages * chunk;
  const size_t smem_st = (size_t)(kCopyThreads / 32) * chunk;
  if (engine == 1 || engine == 5 || engine == 6) {
    if (smem_ld > 227 * 1024) fail(GINSIM_E_USAGE, "chunk too large for 4 stages x 8 warps");
    GIN_CUDA(cudaFuncSetAttribute((const void*)tma_copy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_ld));
  }
  if (engine == 4)
    GIN_CUDA(cudaFuncSetAttribute((const void*)tma_store_only_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_st));
  cudaEvent_t e0, e1;
  GIN_CUDA(cudaEventCreate(&e0));
  GIN_CUDA(cudaEventCreate(&e1));
  auto launch = [&] {
    switch (engine) {
      case 0: lsu_copy_kernel<<<G, kCopyThreads, 0, s>>>(dst, src, bytes); break;
      case 1: tma_copy_kernel<<<G, kCopyThreads, smem_ld, s>>>(dst, src, bytes, chunk); break;
      case 2: lsu256_copy_kernel<<<G, kCopyThreads, 0, s>>>(dst, src, bytes); break;
      case 3: GIN_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, s)); break;
      case 4: tma_store_only_kernel<<<G, kCopyThreads, smem_st, s>>>(dst, bytes, chunk); break;
      case 5: tma_copy_kernel<<<G, kCopyThreads, smem_ld, s>>>(dst, src, bytes, chunk); break;
      case 6:
        GIN_CUDA(cudaEventRecord(fork, s));
        GIN_CUDA(cudaStreamWaitEvent(side, fork, 0));
        if (ce_bytes) GIN_CUDA(cudaMemcpyAsync(dst + sm_bytes, src + sm_bytes, ce_bytes, cudaMemcpyDefault, side));
        if (sm_bytes) tma_copy_kernel<<<G, kCopyThreads, smem_ld, s>>>(dst, src, sm_bytes, chunk);
        GIN_CUDA(cudaEventRecord(join, side));
        GIN_CUDA(cudaStreamWaitEvent(s, join, 0));
        break;
      case 8: {
        GIN_CUDA(cudaEventRecord(fork, s));
        const uint64_t per = (bytes / (c->world - 1)) & ~uint64_t(4095);
        for (uint32_t q = 0, i = 0; q < c->world; ++q) {
          if (q == c->rank) continue;
          GIN_CUDA(cudaStreamWaitEvent(ps[i], fork, 0));
          GIN_CUDA(cudaMemcpyAsync(c->windows[dst_win].bases[q] + per * i, src + per * i, per, cudaMemcpyDefault, ps[i]));
          GIN_CUDA(cudaEventRecord(pj[i], ps[i]));
          GIN_CUDA(cudaStreamWaitEvent(s, pj[i], 0));
          ++i;
        }
        break;
      }
      default: lsu256_copy_kernel<<<G, kCopyThreads, 0, s>>>(dst, src, bytes); break;
    }
  };
  launch();
  GIN_CUDA(cudaGetLastError());
  GIN_CUDA(cudaEventRecord(e0, s));
  for (uint32_t i = 0; i < iters; ++i) launch();
  GIN_CUDA(cudaEventRecord(e1, s));
  GIN_CUDA(cudaEventSynchronize(e1));
  GIN_CUDA(cudaGetLastError());
  float ms = 0;
  GIN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  *ms_out = ms / (float)std::max(1u, iters);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (side) {
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    cudaStreamDestroy(side);
  }
  for (auto st : ps) cudaStreamDestroy(st);
  for (auto ev : pj) cudaEventDestroy(ev);
  if (engine == 8) cudaEventDestroy(fork);
  GIN_API_END
}

// Host-issued operation cost (the proxy agent's building blocks): n_ops
// stream memops (kind 0: 64-bit writes, batched `batch` per
// cuStreamBatchMemOp) or copies (kind 1: cudaMemcpyAsync of `bytes` each)
// into `peer`'s dst window.  out[0] = device us per op (events), out[1] =
// host us per op spent issuing.
int ginsim_cuda_host_op_bench(ginsim_cuda_comm_t comm, uint32_t src_win, uint32_t dst_win, uint32_t peer,
                              uint32_t kind, uint32_t n_ops, uint32_t batch, uint64_t bytes, float* out,
                              void* stream) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->window_live(src_win) || !c->window_live(dst_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
  if (peer >= c->world || kind > 1 || n_ops == 0 || batch == 0 || batch > 256) fail(GINSIM_E_USAGE, "bad probe arguments");
  const uint64_t span = kind == 0 ? 8ull * n_ops : bytes * n_ops;
  if (c->windows[dst_win].sizes[peer] < span || c->windows[src_win].sizes[c->rank] < span)
    fail(GINSIM_E_OUT_OF_BOUNDS, "probe exceeds window capacity");
  DeviceGuard g(c->device);
  char* dst = c->windows[dst_win].bases[peer];
  const char* src = c->windows[src_win].bases[c->rank];
  cudaStream_t s = (cudaStream_t)stream, own = nullptr;
  if (!s) {  // stream memops need an explicit stream
    GIN_CUDA(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
    s = own;
  }
  std::vector<CUstreamBatchMemOpParams> ops;
  auto issue = [&](uint64_t v) {
    if (kind == 0) {
      for (uint32_t i = 0; i < n_ops; i += batch) {
        ops.clear();
        for (uint32_t j = i; j < std::min(n_ops, i + batch); ++j) {
          CUstreamBatchMemOpParams op{};
          op.writeValue.operation = CU_STREAM_MEM_OP_WRITE_VALUE_64;
          op.writeValue.address = (CUdeviceptr)(dst + 8ull * j);
          op.writeValue.value64 = v + j;
          op.writeValue.flags = CU_STREAM_WRITE_VALUE_DEFAULT;
          ops.push_back(op);
        }
        GIN_CU(cuapi().cuStreamBatchMemOp((CUstream)s, (unsigned)ops.size(), ops.data(), 0));
      }
    } else {
      for (uint32_t j = 0; j < n_ops; ++j)
        GIN_CUDA(cudaMemcpyAsync(dst + bytes * j, src + bytes * j, bytes, cudaMemcpyDefault, s));
    }
  };
  issue(1);
  GIN_CUDA(cudaStreamSynchronize(s));
  cudaEvent_t e0, e1;
  GIN_CUDA(cudaEventCreate(&e0));
  GIN_CUDA(cudaEventCreate(&e1));
  // a short spin kernel first so the whole sequence is queued before it runs
  spin_kernel<<<1, 32, 0, s>>>(2000000ull);
  GIN_CUDA(cudaEventRecord(e0, s));
  const auto h0 = std::chrono::steady_clock::now();
  issue(1000);
  const auto h1 = std::chrono::steady_clock::now();
  GIN_CUDA(cudaEventRecord(e1, s));
  GIN_CUDA(cudaEventSynchronize(e1));
  float ms = 0;
  GIN_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  out[0] = ms * 1000.f / (float)n_ops;
  out[1] = (float)std::chrono::duration<double, std::micro>(h1 - h0).count() / (float)n_ops;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (own) cudaStreamDestroy(own);
  GIN_API_END
}

int ginsim_cuda_occupy(int device, uint32_t ctas_per_sm, const uint32_t* release_word, uint64_t timeout_ms,
                       void* stream) {
  GIN_API_BEGIN
  DeviceGuard g(device);
  int sms = 0;
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  const uint32_t per = std::max(1u, std::min(ctas_per_sm, 2u));
  occupy_kernel<<<sms * per, 1024, 0, (cudaStream_t)stream>>>(reinterpret_cast<const volatile uint32_t*>(release_word),
                                                              timeout_ms * 1000000ull);
  GIN_CUDA(cudaGetLastError());
  GIN_API_END
}

}  // extern "C"
