// kernels_bench.cu — raw NVLink / HBM copy engines used as roofline probes:
// the same put path the MoE kernels use (128-bit LSU stores or TMA bulk
// copies staged through shared memory) over one window region into a peer's
// (or the local) window, no signals.  Gives the measured NVLink write floor
// that BASELINE's "fraction of 900 GB/s" sits next to.
#include <algorithm>

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
  Comm* c = &comm->impl;
  if (src_win >= c->windows.size() || dst_win >= c->windows.size()) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
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

}  // extern "C"
