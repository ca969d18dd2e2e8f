// runtime.cu — host runtime behind the C ABI: bootstrap, communicator setup,
// VMM window registration and peer mapping, completion cells, host-issued ops.
//
// Reference counterparts (/root/reference-relative):
//   InProcGroup rendezvous          proj/core/src/runtime.cpp:66-175
//   DevComm ctor / tables           proj/core/src/runtime.cpp:197-213
//   window_register / finalize      proj/core/src/runtime.cpp:347-380
//   cells read/wait/reset           proj/core/src/runtime.cpp:404-443
//   Gin put / put_value / signal    proj/core/src/runtime.cpp:604-633
//   comm_init                       proj/core/src/runtime.cpp:582-599
// B200 design: every rank's signal table and every window region is a
// cuMemCreate allocation exported as a POSIX FD; peers import it (same
// process: reuse the VA and grant access; other process: pidfd_getfd +
// cuMemImportFromShareableHandle + cuMemMap) so a device put is a plain
// NVLink store and a signal is one red.release.sys.
#include <sys/syscall.h>
#include <unistd.h>

#include <chrono>
#include <cstdlib>
#include <cstring>

#include "gin_device.cuh"
#include "runtime_internal.h"

namespace ginsim_b200 {

static thread_local std::string g_last_error = "no error";
void set_last_error(const char* m) { g_last_error = m; }

void fail(int code, const std::string& msg) { throw GinError(code, msg); }

const CuApi& cuapi() {
  static CuApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", reinterpret_cast<void**>(&api.cuStreamWriteValue64), cudaEnableDefault, &q) != cudaSuccess || !api.cuStreamWriteValue64)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuStreamWriteValue64 unavailable");
    if (cudaGetDriverEntryPoint("cuStreamBatchMemOp", reinterpret_cast<void**>(&api.cuStreamBatchMemOp), cudaEnableDefault, &q) != cudaSuccess || !api.cuStreamBatchMemOp)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuStreamBatchMemOp unavailable");
    if (cudaGetDriverEntryPoint("cuGetErrorString", reinterpret_cast<void**>(&api.cuGetErrorString), cudaEnableDefault, &q) != cudaSuccess || !api.cuGetErrorString)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuGetErrorString unavailable");
    if (cudaGetDriverEntryPoint("cuMemAddressFree", reinterpret_cast<void**>(&api.cuMemAddressFree), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemAddressFree)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemAddressFree unavailable");
    if (cudaGetDriverEntryPoint("cuMemAddressReserve", reinterpret_cast<void**>(&api.cuMemAddressReserve), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemAddressReserve)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemAddressReserve unavailable");
    if (cudaGetDriverEntryPoint("cuMemCreate", reinterpret_cast<void**>(&api.cuMemCreate), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemCreate)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemCreate unavailable");
    if (cudaGetDriverEntryPoint("cuMemExportToShareableHandle", reinterpret_cast<void**>(&api.cuMemExportToShareableHandle), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemExportToShareableHandle)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemExportToShareableHandle unavailable");
    if (cudaGetDriverEntryPoint("cuMemGetAllocationGranularity", reinterpret_cast<void**>(&api.cuMemGetAllocationGranularity), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemGetAllocationGranularity)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemGetAllocationGranularity unavailable");
    if (cudaGetDriverEntryPoint("cuMemImportFromShareableHandle", reinterpret_cast<void**>(&api.cuMemImportFromShareableHandle), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemImportFromShareableHandle)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemImportFromShareableHandle unavailable");
    if (cudaGetDriverEntryPoint("cuMemMap", reinterpret_cast<void**>(&api.cuMemMap), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemMap)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemMap unavailable");
    if (cudaGetDriverEntryPoint("cuMemRelease", reinterpret_cast<void**>(&api.cuMemRelease), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemRelease)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemRelease unavailable");
    if (cudaGetDriverEntryPoint("cuMemSetAccess", reinterpret_cast<void**>(&api.cuMemSetAccess), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemSetAccess)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemSetAccess unavailable");
    if (cudaGetDriverEntryPoint("cuMemUnmap", reinterpret_cast<void**>(&api.cuMemUnmap), cudaEnableDefault, &q) != cudaSuccess || !api.cuMemUnmap)
      throw GinError(GINSIM_E_CUDA, "driver entry point cuMemUnmap unavailable");
    // optional (multicast): left null when absent
    cudaGetDriverEntryPoint("cuMulticastCreate", reinterpret_cast<void**>(&api.cuMulticastCreate), cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuMulticastAddDevice", reinterpret_cast<void**>(&api.cuMulticastAddDevice), cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuMulticastBindMem", reinterpret_cast<void**>(&api.cuMulticastBindMem), cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuMulticastUnbind", reinterpret_cast<void**>(&api.cuMulticastUnbind), cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuMulticastGetGranularity", reinterpret_cast<void**>(&api.cuMulticastGetGranularity), cudaEnableDefault, &q);
    cudaGetDriverEntryPoint("cuDeviceGetAttribute", reinterpret_cast<void**>(&api.cuDeviceGetAttribute), cudaEnableDefault, &q);
    cudaGetLastError();
  });
  return api;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) fail(GINSIM_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
void cu_check(CUresult r, const char* what) {
  if (r != CUDA_SUCCESS) {
    const char* s = nullptr;
    if (cuapi().cuGetErrorString) cuapi().cuGetErrorString(r, &s);
    fail(GINSIM_E_CUDA, std::string(what) + ": " + (s ? s : "unknown CUresult"));
  }
}

DeviceGuard::DeviceGuard(int dev) {
  cudaGetDevice(&prev);
  if (prev != dev) GIN_CUDA(cudaSetDevice(dev));
}
DeviceGuard::~DeviceGuard() {
  if (prev >= 0) cudaSetDevice(prev);
}

// ------------------------------------------------------------------ in-process group
struct InProcGroup {
  uint32_t world;
  uint64_t timeout_ms = 60000;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<uint8_t> buf;
  size_t bytes = 0;
  uint32_t arrived = 0, left = 0;
  bool draining = false;

  int allgather(uint32_t rank, const void* send, void* recv, size_t n) {
    std::unique_lock<std::mutex> lk(mu);
    auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(timeout_ms);
    if (!cv.wait_until(lk, deadline, [&] { return !draining; })) return 1;
    if (arrived == 0) {
      buf.assign((size_t)world * n, 0);
      bytes = n;
    } else if (bytes != n) {
      return 2;
    }
    std::memcpy(buf.data() + (size_t)rank * n, send, n);
    if (++arrived == world) {
      draining = true;
      cv.notify_all();
    } else if (!cv.wait_until(lk, deadline, [&] { return draining; })) {
      return 1;
    }
    std::memcpy(recv, buf.data(), (size_t)world * n);
    if (++left == world) {
      left = 0;
      arrived = 0;
      draining = false;
      cv.notify_all();
    }
    return 0;
  }
};

struct InProcEndpoint {
  InProcGroup* g;
  uint32_t rank;
};

static int inproc_allgather(void* ctx, const void* send, void* recv, size_t bytes) {
  auto* ep = static_cast<InProcEndpoint*>(ctx);
  return ep->g->allgather(ep->rank, send, recv, bytes);
}

}  // namespace ginsim_b200

struct ginsim_cuda_group_s {
  ginsim_b200::InProcGroup g;
  std::vector<ginsim_b200::InProcEndpoint> eps;
};

namespace ginsim_b200 {

// ------------------------------------------------------------------ comm plumbing
void Comm::allgather(const void* send, void* recv, size_t bytes) {
  int rc = boot.allgather(boot.ctx, send, recv, bytes);
  if (rc != 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "bootstrap allgather failed (rc " + std::to_string(rc) + ")");
}
void Comm::barrier() {
  std::vector<uint8_t> all(world);
  uint8_t one = 1;
  allgather(&one, all.data(), 1);
}
void Comm::sync_view() {
  DeviceGuard g(device);
  GIN_CUDA(cudaMemcpy(dev_view, &host_view, sizeof(GinDevCommView), cudaMemcpyHostToDevice));
}

static uint64_t granularity(int device) {
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  GIN_CU(cuapi().cuMemGetAllocationGranularity(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  return g;
}

static VmmAlloc vmm_alloc(int device, uint64_t bytes) {
  DeviceGuard dg(device);
  GIN_CUDA(cudaFree(nullptr));  // make sure the primary context exists
  VmmAlloc a;
  a.device = device;
  const uint64_t g = granularity(device);
  a.size = ((bytes ? bytes : 1) + g - 1) / g * g;
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = device;
  prop.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  GIN_CU(cuapi().cuMemCreate(&a.handle, a.size, &prop, 0));
  GIN_CU(cuapi().cuMemAddressReserve(&a.ptr, a.size, g, 0, 0));
  GIN_CU(cuapi().cuMemMap(a.ptr, a.size, 0, a.handle, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  GIN_CU(cuapi().cuMemSetAccess(a.ptr, a.size, &acc, 1));
  int fd = -1;
  GIN_CU(cuapi().cuMemExportToShareableHandle(&fd, a.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  a.fd = fd;
  GIN_CUDA(cudaMemset((void*)a.ptr, 0, a.size));
  GIN_CUDA(cudaDeviceSynchronize());
  return a;
}

static void vmm_free(VmmAlloc& a) {
  if (!a.ptr) return;
  cuapi().cuMemUnmap(a.ptr, a.size);
  cuapi().cuMemAddressFree(a.ptr, a.size);
  cuapi().cuMemRelease(a.handle);
  if (a.fd >= 0) close(a.fd);
  a = VmmAlloc{};
}

char* Comm::map_blob(const ExportBlob& b, std::vector<Mapping>* maps) {
  if (b.bytes == 0 && b.alloc_size == 0) return nullptr;
  if (b.pid == (int32_t)getpid()) {
    if (b.device != device) {
      if (b.is_vmm) {
        CUmemAccessDesc acc{};
        acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
        acc.location.id = device;
        acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
        std::lock_guard<std::mutex> lk(mu);
        GIN_CU(cuapi().cuMemSetAccess((CUdeviceptr)(b.ptr - b.offset), b.alloc_size, &acc, 1));
      } else {
        DeviceGuard g(device);
        cudaError_t e = cudaDeviceEnablePeerAccess(b.device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) {
          cudaGetLastError();
        } else {
          GIN_CUDA(e);
        }
      }
    }
    return reinterpret_cast<char*>(b.ptr);
  }
  if (!b.is_vmm) {
    fail(GINSIM_E_USAGE, "window memory shared across processes must come from ginsim_cuda_mem_alloc");
  }
  int pidfd = (int)syscall(SYS_pidfd_open, b.pid, 0);
  if (pidfd < 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "pidfd_open of peer process failed");
  int fd = (int)syscall(SYS_pidfd_getfd, pidfd, b.fd, 0);
  close(pidfd);
  if (fd < 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "pidfd_getfd of peer allocation failed");
  DeviceGuard g(device);
  Mapping m;
  m.size = b.alloc_size;
  GIN_CU(cuapi().cuMemImportFromShareableHandle(&m.handle, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
  close(fd);
  GIN_CU(cuapi().cuMemAddressReserve(&m.ptr, m.size, granularity(device), 0, 0));
  GIN_CU(cuapi().cuMemMap(m.ptr, m.size, 0, m.handle, 0));
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  GIN_CU(cuapi().cuMemSetAccess(m.ptr, m.size, &acc, 1));
  {
    std::lock_guard<std::mutex> lk(mu);
    (maps ? *maps : imported).push_back(m);
  }
  return reinterpret_cast<char*>(m.ptr + b.offset);
}

void check_same_device(const ginsim_cuda_comm_t* comms, uint32_t n) {
  if (n == 0 || n > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "launch needs 1..8 comms");
  if (!comms) fail(GINSIM_E_USAGE, "null communicator list");
  for (uint32_t i = 0; i < n; ++i) comm_impl(comms[i]);  // null handles -> UsageError
  for (uint32_t i = 1; i < n; ++i) {
    if (comms[i]->impl.device != comms[0]->impl.device) {
      fail(GINSIM_E_USAGE, "emulated ranks in one launch must share a device; launch per device instead");
    }
  }
}

int max_coresident_ctas(const void* kernel, int threads, size_t smem, int device) {
  int per_sm = 0, sms = 0;
  GIN_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  return per_sm * sms;
}

void check_device_error(Comm* c) {
  uint32_t code = 0;
  DeviceGuard g(c->device);
  GIN_CUDA(cudaMemcpy(&code, c->host_view.error, 4, cudaMemcpyDeviceToHost));
  if (code) {
    uint32_t zero = 0;
    GIN_CUDA(cudaMemcpy(c->host_view.error, &zero, 4, cudaMemcpyHostToDevice));
    fail((int)code, "device-side error " + std::to_string(code) + " on rank " + std::to_string(c->rank));
  }
}

// ------------------------------------------------------------------ host-issued ops
struct HostOp {
  uint32_t kind;  // 0 put, 1 put_value, 2 signal
  uint32_t ctx, peer, dst_win, src_win, width;
  uint64_t dst_off, src_off_or_value, bytes;
  gin::Action action;
};

__global__ void host_op_kernel(const GinDevCommView* v, HostOp op) {
  gin::Gin gin(v, op.ctx);
  gin::CoopWarp w;
  const gin::Team world = gin::WorldTeam(v->world);
  switch (op.kind) {
    case 0:
      gin.put(w, world, op.peer, op.dst_win, op.dst_off, op.src_win, op.src_off_or_value, op.bytes, op.action);
      break;
    default:
      gin.put_value_raw(w, world, op.peer, op.dst_win, op.dst_off, op.src_off_or_value, op.width, op.action);
      break;
  }
}

// Bulk part of a large host-issued direct put: every SM moves a slice with
// 128-bit vectors (a one-warp put would crawl); the op's completion action
// then follows as a zero-byte put in stream order (the kernel boundary orders
// this kernel's stores before that release).
__global__ void __launch_bounds__(512) host_copy_kernel(char* dst, const char* src, uint64_t bytes) {
  const uint64_t per = ((bytes + gridDim.x - 1) / gridDim.x + 15) & ~15ull;
  const uint64_t lo = min(bytes, per * blockIdx.x), hi = min(bytes, lo + per);
  if (hi > lo) gin::coop_copy(gin::CoopCta{}, dst + lo, src + lo, hi - lo);
}

__global__ void host_signal_kernel(const GinDevCommView* v, uint32_t ctx, uint32_t peer, uint32_t id,
                                   gin::SignalOp op, int32_t counter) {
  gin::Gin gin(v, ctx);
  gin::CoopWarp w;
  gin::Action extra = gin::NoAction();
  extra.counter_id = counter;
  gin.signal(w, gin::WorldTeam(v->world), peer, id, op, extra);
}

static gin::Action to_action(const ginsim_cuda_action* a) {
  gin::Action r = gin::NoAction();
  if (!a) return r;
  r.signal_id = a->signal_id;
  r.counter_id = a->counter_id;
  r.op = a->signal_add ? gin::SignalAdd(a->operand) : gin::SignalInc();
  return r;
}

static void validate_action(Comm* c, const ginsim_cuda_action* a) {
  if (!a) return;
  if (a->signal_id >= 0 && (uint32_t)a->signal_id >= c->cfg.signal_cells)
    fail(GINSIM_E_INVALID_SIGNAL, "signal " + std::to_string(a->signal_id) + " out of range");
  if (a->counter_id >= 0 && (uint32_t)a->counter_id >= c->cfg.counter_cells)
    fail(GINSIM_E_INVALID_COUNTER, "counter " + std::to_string(a->counter_id) + " out of range");
  if (a->signal_id >= 0 && !a->signal_add && a->operand != 1 && a->operand != 0) {
    // SignalInc carries operand 1 (types.hpp:33-37); any other value is ignored.
  }
}

static void validate_common(Comm* c, uint32_t ctx, uint32_t peer) {
  if (ctx >= c->cfg.n_contexts) fail(GINSIM_E_INVALID_CONTEXT, "context out of range");
  if (peer >= c->world)
    fail(GINSIM_E_INVALID_PEER, "peer " + std::to_string(peer) + " outside team of " + std::to_string(c->world));
}

static const Comm::Window& lookup_window(Comm* c, uint32_t w) {
  if (!c->window_live(w)) fail(GINSIM_E_UNKNOWN_WINDOW, "window " + std::to_string(w) + " is not registered");
  return c->windows[w];
}

static void check_range(Comm* c, uint32_t w, uint32_t rank, uint64_t off, uint64_t len) {
  const auto& win = lookup_window(c, w);
  const uint64_t cap = win.sizes[rank];
  if (off > cap || len > cap - off) {
    fail(GINSIM_E_OUT_OF_BOUNDS, "window " + std::to_string(w) + " rank " + std::to_string(rank) + ": [" +
                                     std::to_string(off) + ", +" + std::to_string(len) + ") exceeds capacity " +
                                     std::to_string(cap));
  }
}

static void encode_host_op(Comm* c, uint8_t opcode, uint32_t peer, uint32_t dst_win, uint64_t dst_off,
                           uint32_t src_win, uint64_t src, uint64_t bytes, const ginsim_cuda_action* a,
                           uint8_t out[64]) {
  ginsim_cuda_descriptor d{};
  d.opcode = opcode;
  d.team = 0;
  d.peer = peer;
  d.dst_window = dst_win;
  d.src_window = src_win;
  d.dst_offset = dst_off;
  d.src_offset_or_value = src;
  d.bytes = bytes;
  if (a && a->signal_id >= 0) {
    d.flags |= GIN_FLAG_HAS_SIGNAL;
    d.signal_id = (uint32_t)a->signal_id;
    if (a->signal_add) {
      d.flags |= GIN_FLAG_SIGNAL_IS_ADD;
      d.signal_operand = a->operand;
    } else {
      d.signal_operand = 1;
    }
  }
  if (a && a->counter_id >= 0) {
    d.flags |= GIN_FLAG_HAS_COUNTER;
    d.counter_id = (uint32_t)a->counter_id;
  }
  (void)c;
  descriptor_encode(&d, out);
}

// Direct backend: a host-issued op carrying a local counter is outstanding
// until the stream has executed it (counter_pending, runtime.cpp:431-438).
static void note_direct_counter(Comm* c, const ginsim_cuda_action* a, cudaStream_t s) {
  if (!a || a->counter_id < 0) return;
  std::lock_guard<std::mutex> lk(c->mu);
  cudaEvent_t e;
  if (!c->free_op_events.empty()) {
    e = c->free_op_events.back();
    c->free_op_events.pop_back();
  } else {
    GIN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  GIN_CUDA(cudaEventRecord(e, s));
  c->direct_pending.emplace_back(e, (uint32_t)a->counter_id);
}
static bool direct_counter_pending(Comm* c, uint32_t id) {
  std::lock_guard<std::mutex> lk(c->mu);
  bool pending = false;
  std::vector<std::pair<cudaEvent_t, uint32_t>> keep;
  for (auto& pe : c->direct_pending) {
    const cudaError_t q = cudaEventQuery(pe.first);
    if (q == cudaSuccess) {
      c->free_op_events.push_back(pe.first);
      continue;
    }
    if (q != cudaErrorNotReady) GIN_CUDA(q);
    if (pe.second == id) pending = true;
    keep.push_back(pe);
  }
  c->direct_pending.swap(keep);
  return pending;
}

// submit_op (runtime.cpp:474-544) for a host-issued op: validation (ctx, peer,
// bounds against the peer's capacity and our own, inline width, cell ids),
// then the direct path (a one-warp device op on `stream`) or the proxy path
// (a descriptor for the host agent).  Returns the proxy host ticket of the
// op on its context (0 on the direct backend).
constexpr uint64_t kHostCopyBulk = 256ull << 10;  // host puts from this size spread over the SMs

uint64_t host_op(Comm* c, uint32_t ctx, uint8_t opcode, uint32_t peer, uint32_t dst_win, uint64_t dst_off,
                 uint32_t src_win, uint64_t src_or_value, uint64_t bytes, const ginsim_cuda_action* action,
                 cudaStream_t stream) {
  NvtxRange nv(opcode == GIN_OP_PUT ? "ginsim.put" : (opcode == GIN_OP_PUT_INLINE ? "ginsim.put_value" : "ginsim.signal"));
  validate_common(c, ctx, peer);
  if (opcode == GIN_OP_PUT_INLINE && (bytes == 0 || bytes > 8))
    fail(GINSIM_E_INVALID_DESCRIPTOR, "put_value width must be 1..8 bytes");
  if (opcode != GIN_OP_SIGNAL_ONLY) check_range(c, dst_win, peer, dst_off, bytes);
  if (opcode == GIN_OP_PUT) check_range(c, src_win, c->rank, src_or_value, bytes);
  validate_action(c, action);
  if (c->cfg.backend == GIN_BACKEND_PROXY) {
    uint8_t d[64];
    encode_host_op(c, opcode, peer, opcode == GIN_OP_SIGNAL_ONLY ? 0 : dst_win, dst_off, src_win, src_or_value, bytes,
                   action, d);
    return proxy_host_submit(c, ctx, d);
  }
  DeviceGuard g(c->device);
  if (opcode == GIN_OP_SIGNAL_ONLY) {
    host_signal_kernel<<<1, 32, 0, stream>>>(c->dev_view, ctx, peer, (uint32_t)action->signal_id,
                                              action->signal_add ? gin::SignalAdd(action->operand) : gin::SignalInc(),
                                              action->counter_id);
  } else {
    HostOp op{};
    op.kind = opcode == GIN_OP_PUT ? 0 : 1;
    op.ctx = ctx;
    op.peer = peer;
    op.dst_win = dst_win;
    op.src_win = src_win;
    op.dst_off = dst_off;
    op.src_off_or_value = src_or_value;
    op.bytes = bytes;
    if (opcode == GIN_OP_PUT && bytes >= kHostCopyBulk) {
      int sms = 0;
      GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
      const uint32_t G = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms, bytes / kHostCopyBulk));
      host_copy_kernel<<<G, 512, 0, stream>>>(c->windows[dst_win].bases[peer] + dst_off,
                                              c->windows[src_win].bases[c->rank] + src_or_value, bytes);
      GIN_CUDA(cudaGetLastError());
      op.bytes = 0;  // the completion action rides on a zero-byte put after the copy
    }
    op.width = (uint32_t)bytes;
    op.action = to_action(action);
    host_op_kernel<<<1, 32, 0, stream>>>(c->dev_view, op);
  }
  GIN_CUDA(cudaGetLastError());
  note_direct_counter(c, action, stream);
  return 0;
}

}  // namespace ginsim_b200

using namespace ginsim_b200;

extern "C" {

const char* ginsim_cuda_last_error(void) { return g_last_error.c_str(); }
int ginsim_cuda_abi_version(void) { return GINSIM_CUDA_ABI_VERSION; }

void ginsim_cuda_config_default(ginsim_cuda_config* cfg) {
  cfg->n_contexts = 4;
  cfg->backend = GIN_BACKEND_DIRECT;
  cfg->signal_cells = 256;
  cfg->counter_cells = 256;
  cfg->queue_depth = 1024;
  cfg->transport = 0;
  cfg->timeout_ms = 30000;
}

static bool env_u64(const char* name, uint64_t* out) {
  const char* v = std::getenv(name);
  if (!v || !*v) return false;
  char* end = nullptr;
  unsigned long long x = std::strtoull(v, &end, 0);
  if (end == v || *end != '\0') fail(GINSIM_E_USAGE, std::string(name) + ": cannot parse '" + v + "' as an integer");
  *out = x;
  return true;
}

int ginsim_cuda_config_from_env(ginsim_cuda_config* cfg) {
  GIN_API_BEGIN
  if (const char* b = std::getenv("GINSIM_BACKEND"); b && *b) {
    std::string s(b);
    if (s == "direct") cfg->backend = GIN_BACKEND_DIRECT;
    else if (s == "proxy") cfg->backend = GIN_BACKEND_PROXY;
    else fail(GINSIM_E_USAGE, "GINSIM_BACKEND must be 'direct' or 'proxy', got '" + s + "'");
  }
  if (const char* t = std::getenv("GINSIM_TRANSPORT"); t && *t) {
    std::string s(t);
    if (s == "fabric" || s == "nvlink") cfg->transport = 0;
    else if (s == "socket") cfg->transport = 1;
    else fail(GINSIM_E_USAGE, "GINSIM_TRANSPORT must be 'fabric' or 'socket', got '" + s + "'");
  }
  uint64_t v;
  if (env_u64("GINSIM_QUEUE_DEPTH", &v)) cfg->queue_depth = (uint32_t)v;
  if (env_u64("GINSIM_TIMEOUT_MS", &v)) cfg->timeout_ms = v;
  GIN_API_END
}

int ginsim_cuda_inproc_group_create(uint32_t world_size, ginsim_cuda_group_t* out) {
  GIN_API_BEGIN
  if (world_size == 0) fail(GINSIM_E_USAGE, "world size must be positive");
  if (world_size > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "world size above 8 (one NVSwitch domain)");
  auto* g = new ginsim_cuda_group_s;
  g->g.world = world_size;
  g->eps.resize(world_size);
  for (uint32_t r = 0; r < world_size; ++r) g->eps[r] = InProcEndpoint{&g->g, r};
  *out = g;
  GIN_API_END
}

int ginsim_cuda_inproc_group_destroy(ginsim_cuda_group_t group) {
  delete group;
  return GINSIM_OK;
}

int ginsim_cuda_inproc_bootstrap(ginsim_cuda_group_t group, uint32_t rank, ginsim_cuda_bootstrap* out) {
  GIN_API_BEGIN
  if (rank >= group->g.world) fail(GINSIM_E_USAGE, "rank outside group");
  out->ctx = &group->eps[rank];
  out->allgather = &inproc_allgather;
  GIN_API_END
}

int ginsim_cuda_comm_create(uint32_t rank, uint32_t world, int device, const ginsim_cuda_config* cfg_in,
                            const ginsim_cuda_bootstrap* boot, ginsim_cuda_comm_t* out) {
  GIN_API_BEGIN
  if (world == 0 || world > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "world size must be 1..8");
  if (rank >= world) fail(GINSIM_E_USAGE, "rank " + std::to_string(rank) + " outside world of " + std::to_string(world));
  ginsim_cuda_config cfg;
  if (cfg_in) cfg = *cfg_in; else ginsim_cuda_config_default(&cfg);
  if (cfg.signal_cells < GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS)
    fail(GINSIM_E_USAGE, "signal table smaller than the reserved barrier region");
  if (cfg.n_contexts == 0 || cfg.n_contexts > GIN_MAX_CONTEXTS) fail(GINSIM_E_USAGE, "n_contexts must be 1..16");
  if (cfg.transport > 1) fail(GINSIM_E_USAGE, "transport must be 0 (fabric) or 1 (socket)");
  if (cfg.transport == 1 && cfg.backend != GIN_BACKEND_PROXY)
    fail(GINSIM_E_BACKEND_MISMATCH, "the socket transport runs on the Proxy backend (device stores need the fabric)");
  if (cfg.queue_depth == 0 || (cfg.queue_depth & (cfg.queue_depth - 1)))
    fail(GINSIM_E_USAGE, "ring capacity must be a power of two, got " + std::to_string(cfg.queue_depth));
  if (cfg.backend > 1) fail(GINSIM_E_USAGE, "backend must be 0 (direct) or 1 (proxy)");
  auto holder = std::make_unique<ginsim_cuda_comm_s>();
  Comm* c = &holder->impl;
  c->rank = rank;
  c->world = world;
  c->device = device;
  c->cfg = cfg;
  c->boot = *boot;
  // Config equality (runtime.cpp:86-105): compare against rank 0's.
  std::vector<ginsim_cuda_config> all(world);
  c->allgather(&cfg, all.data(), sizeof(cfg));
  for (uint32_t r = 0; r < world; ++r) {
    if (std::memcmp(&all[r], &all[0], sizeof(cfg)) != 0) {
      fail(GINSIM_E_CONFIG_MISMATCH, "rank " + std::to_string(r) + " passed a configuration differing from rank 0");
    }
  }
  DeviceGuard dg(device);
  GIN_CUDA(cudaFree(nullptr));
  const uint64_t cells = cfg.signal_cells;
  c->signal_alloc = vmm_alloc(device, (uint64_t)world * cells * 8);
  // local block: signal_base | counters | counter_base | error | tickets | completed | workspace
  const size_t sz_sig_base = cells * 8, sz_ctr = (size_t)cfg.counter_cells * 8;
  const size_t off_ctr = sz_sig_base, off_ctr_base = off_ctr + sz_ctr, off_err = off_ctr_base + sz_ctr;
  const size_t off_tk = (off_err + 256), off_done = off_tk + GIN_MAX_CONTEXTS * 8, off_ws = (off_done + GIN_MAX_CONTEXTS * 8 + 255) / 256 * 256;
  const size_t total = off_ws + 65536;
  GIN_CUDA(cudaMalloc(&c->local_block, total));
  GIN_CUDA(cudaMemset(c->local_block, 0, total));
  char* lb = static_cast<char*>(c->local_block);
  GinDevCommView& v = c->host_view;
  std::memset(&v, 0, sizeof(v));
  v.rank = rank;
  v.world = world;
  v.n_ctx = cfg.n_contexts;
  v.signal_cells = cfg.signal_cells;
  v.counter_cells = cfg.counter_cells;
  v.backend = cfg.backend;
  v.device = (uint32_t)device;
  v.timeout_ns = cfg.timeout_ms * 1000000ull;
  v.signal_base = reinterpret_cast<uint64_t*>(lb);
  v.counters = reinterpret_cast<uint64_t*>(lb + off_ctr);
  v.counter_base = reinterpret_cast<uint64_t*>(lb + off_ctr_base);
  v.error = reinterpret_cast<unsigned int*>(lb + off_err);
  v.proxy.tickets = reinterpret_cast<unsigned long long*>(lb + off_tk);
  v.proxy.completed = reinterpret_cast<uint64_t*>(lb + off_done);
  v.proxy.mask = cfg.queue_depth - 1;
  v.workspace = reinterpret_cast<unsigned int*>(lb + off_ws);
  // teams: slot 0 is the world team (id 0, identity; types.cpp:8-14)
  v.teams[0].id = 0;
  v.teams[0].n = world;
  for (uint32_t r = 0; r < GIN_MAX_RANKS; ++r) v.teams[0].members[r] = (uint8_t)r;
  // Exchange and map every rank's signal table.
  ExportBlob mine{};
  mine.pid = (int32_t)getpid();
  mine.fd = c->signal_alloc.fd;
  mine.device = device;
  mine.is_vmm = 1;
  mine.alloc_size = c->signal_alloc.size;
  mine.offset = 0;
  mine.bytes = (uint64_t)world * cells * 8;
  mine.ptr = c->signal_alloc.ptr;
  std::vector<ExportBlob> blobs(world);
  c->allgather(&mine, blobs.data(), sizeof(ExportBlob));
  for (uint32_t r = 0; r < world; ++r) {
    // (the socket transport reaches peers only through their agents: their
    // signal tables and windows are not mapped into this process)
    v.signals[r] = r == rank ? reinterpret_cast<uint64_t*>(c->signal_alloc.ptr)
                             : (cfg.transport == 1 ? nullptr : reinterpret_cast<uint64_t*>(c->map_blob(blobs[r])));
    if (r != rank && blobs[r].pid == mine.pid && blobs[r].device == device) c->shares_device = true;
    if (blobs[r].pid == mine.pid && blobs[r].device == device) v.same_gpu |= 1u << r;
  }
  GIN_CUDA(cudaMalloc(&c->dev_view, sizeof(GinDevCommView)));
  GIN_CUDA(cudaStreamCreateWithFlags(&c->op_stream, cudaStreamNonBlocking));
  if (cfg.backend == GIN_BACKEND_PROXY) c->proxy = proxy_start(c);
  nvls_setup(c);  // collective; leaves nvls.on = false where multicast is unavailable
  // Load the host-op kernels now.  Under CUDA's lazy module loading the first
  // launch of a kernel loads it, and that load waits for the device: a
  // host-issued put made while a long-running kernel holds the GPU (e.g. a
  // user kernel spinning on a signal this put delivers) would block until
  // that kernel ends.
  {
    cudaFuncAttributes fa{};
    GIN_CUDA(cudaFuncGetAttributes(&fa, (const void*)host_op_kernel));
    GIN_CUDA(cudaFuncGetAttributes(&fa, (const void*)host_signal_kernel));
    GIN_CUDA(cudaFuncGetAttributes(&fa, (const void*)host_copy_kernel));
  }
  c->sync_view();
  GIN_CUDA(cudaDeviceSynchronize());
  c->barrier();  // nobody signals a peer before every table is mapped
  *out = holder.release();
  GIN_API_END
}

int ginsim_cuda_comm_create_all(uint32_t world, const int* devices, const ginsim_cuda_config* cfg,
                                ginsim_cuda_comm_t* out) {
  GIN_API_BEGIN
  ginsim_cuda_group_t g = nullptr;
  int rc = ginsim_cuda_inproc_group_create(world, &g);
  if (rc) fail(rc, g_last_error);
  // The group must outlive the comms only for setup; later collectives
  // (window_register) reuse it, so it is intentionally kept (leaked per set).
  std::vector<int> rcs(world, 0);
  std::vector<std::string> msgs(world);
  std::vector<std::thread> ts;
  for (uint32_t r = 0; r < world; ++r) {
    ts.emplace_back([&, r] {
      ginsim_cuda_bootstrap b;
      ginsim_cuda_inproc_bootstrap(g, r, &b);
      rcs[r] = ginsim_cuda_comm_create(r, world, devices[r], cfg, &b, &out[r]);
      if (rcs[r]) msgs[r] = ginsim_cuda_last_error();
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < world; ++r)
    if (rcs[r]) fail(rcs[r], "rank " + std::to_string(r) + ": " + msgs[r]);
  GIN_API_END
}

int ginsim_cuda_comm_destroy(ginsim_cuda_comm_t comm) {
  GIN_API_BEGIN
  if (!comm) return GINSIM_OK;
  Comm* c = comm_impl(comm);
  {
    DeviceGuard g(c->device);
    cudaDeviceSynchronize();
    if (c->proxy) proxy_stop(c->proxy);
    nvls_teardown(c);
    for (auto& w : c->windows) {
      c->imported.insert(c->imported.end(), w.maps.begin(), w.maps.end());
      if (w.host_registered) cudaHostUnregister(w.host_registered);
    }
    for (auto& m : c->imported) {
      cuapi().cuMemUnmap(m.ptr, m.size);
      cuapi().cuMemAddressFree(m.ptr, m.size);
      cuapi().cuMemRelease(m.handle);
    }
    for (auto& pe : c->direct_pending) cudaEventDestroy(pe.first);
    for (auto e : c->free_op_events) cudaEventDestroy(e);
    for (auto& kv : c->allocs) vmm_free(kv.second);
    vmm_free(c->signal_alloc);
    if (c->dev_view) cudaFree(c->dev_view);
    if (c->local_block) cudaFree(c->local_block);
    if (c->op_stream) cudaStreamDestroy(c->op_stream);
  }
  delete comm;
  GIN_API_END
}

int ginsim_cuda_comm_info(ginsim_cuda_comm_t comm, uint32_t* rank, uint32_t* world, int* device, uint32_t* backend) {
  GIN_API_BEGIN
  const Comm* c = comm_impl(comm);
  if (rank) *rank = c->rank;
  if (world) *world = c->world;
  if (device) *device = c->device;
  if (backend) *backend = c->cfg.backend;
  GIN_API_END
}

int ginsim_cuda_comm_config(ginsim_cuda_comm_t comm, ginsim_cuda_config* out) {
  GIN_API_BEGIN
  const Comm* c = comm_impl(comm);
  if (!out) fail(GINSIM_E_USAGE, "comm_config: null argument");
  *out = c->cfg;
  GIN_API_END
}

int ginsim_cuda_devcomm_view(ginsim_cuda_comm_t comm, const void** view) {
  GIN_API_BEGIN
  const Comm* c = comm_impl(comm);
  if (!view) fail(GINSIM_E_USAGE, "devcomm_view: null argument");
  *view = c->dev_view;
  GIN_API_END
}

int ginsim_cuda_mem_alloc(ginsim_cuda_comm_t comm, uint64_t bytes, void** ptr) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  VmmAlloc a = vmm_alloc(c->device, bytes);
  std::lock_guard<std::mutex> lk(c->mu);
  c->allocs[a.ptr] = a;
  *ptr = reinterpret_cast<void*>(a.ptr);
  GIN_API_END
}

int ginsim_cuda_mem_free(ginsim_cuda_comm_t comm, void* ptr) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  DeviceGuard g(c->device);
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(c->mu);
  auto it = c->allocs.find((CUdeviceptr)ptr);
  if (it == c->allocs.end()) fail(GINSIM_E_UNKNOWN_HANDLE, "pointer was not allocated by ginsim_cuda_mem_alloc");
  vmm_free(it->second);
  c->allocs.erase(it);
  GIN_API_END
}

int ginsim_cuda_window_register(ginsim_cuda_comm_t comm, void* local, uint64_t bytes, uint32_t* window_id) {
  GIN_API_BEGIN
  NvtxRange nv("ginsim.window_register");
  Comm* c = comm_impl(comm);
  if (!window_id) fail(GINSIM_E_USAGE, "window_register: null window id pointer");
  // Dense ids in call order (runtime.cpp:347-371); an id freed by
  // window_deregister is reused (lowest first), so every rank that registers
  // and deregisters in the same order agrees on the ids.
  uint32_t id = 0;
  while (id < c->windows.size() && c->windows[id].live) ++id;
  if (id >= GIN_MAX_WINDOWS)
    fail(GINSIM_E_USAGE, "too many live windows (max " + std::to_string(GIN_MAX_WINDOWS) + "; deregister unused ones)");
  // Host-memory windows (compatibility with the reference's host programs,
  // whose windows are std::vector bytes): pageable host memory is pinned and
  // mapped (cudaHostRegister), so device ops and peers reach it through UVA
  // while the host keeps reading and writing it directly.  In-process ranks
  // only: host pages cannot be imported by another process.
  void* host_registered = nullptr;
  if (bytes > 0 && local) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, local) != cudaSuccess) {
      cudaGetLastError();
      at.type = cudaMemoryTypeUnregistered;
    }
    if (at.type == cudaMemoryTypeUnregistered) {
      DeviceGuard dg(c->device);
      GIN_CUDA(cudaHostRegister(local, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
      host_registered = local;
    }
    if (at.type == cudaMemoryTypeUnregistered || at.type == cudaMemoryTypeHost) {
      void* dptr = nullptr;
      GIN_CUDA(cudaHostGetDevicePointer(&dptr, local, 0));
      if (dptr != local) {
        if (host_registered) cudaHostUnregister(host_registered);
        fail(GINSIM_E_USAGE, "host-memory window without a unified address (device pointer differs)");
      }
    }
  }
  // a failure below (bootstrap, mismatch, peer mapping) must not leave the
  // host pages pinned or the peers' regions mapped
  Comm::Window w;
  struct Undo {
    void* host = nullptr;
    std::vector<Mapping>* maps = nullptr;
    ~Undo() {
      if (maps)
        for (auto& m : *maps) {
          cuapi().cuMemUnmap(m.ptr, m.size);
          cuapi().cuMemAddressFree(m.ptr, m.size);
          cuapi().cuMemRelease(m.handle);
        }
      if (host) cudaHostUnregister(host);
    }
  } undo{host_registered, &w.maps};
  ExportBlob mine{};
  mine.pid = (int32_t)getpid();
  mine.device = c->device;
  mine.bytes = bytes;
  mine.ptr = (uint64_t)local;
  mine.window_id = id;
  mine.fd = -1;
  if (bytes > 0) {
    std::lock_guard<std::mutex> lk(c->mu);
    for (auto& kv : c->allocs) {
      const VmmAlloc& a = kv.second;
      if ((uint64_t)local >= a.ptr && (uint64_t)local + bytes <= a.ptr + a.size) {
        mine.is_vmm = 1;
        mine.fd = a.fd;
        mine.alloc_size = a.size;
        mine.offset = (uint64_t)local - a.ptr;
        break;
      }
    }
    if (!local) fail(GINSIM_E_USAGE, "window of nonzero size with a null pointer");
  }
  std::vector<ExportBlob> blobs(c->world);
  c->allgather(&mine, blobs.data(), sizeof(ExportBlob));
  for (uint32_t r = 0; r < c->world; ++r) {
    if (blobs[r].window_id != mine.window_id) {
      fail(GINSIM_E_REGISTRATION_MISMATCH, "window_register call counts differ: rank " + std::to_string(c->rank) +
                                               " at " + std::to_string(mine.window_id) + ", rank " +
                                               std::to_string(r) + " at " + std::to_string(blobs[r].window_id));
    }
  }
  w.live = true;
  w.host_registered = host_registered;
  w.sizes.resize(c->world);
  w.bases.resize(c->world);
  for (uint32_t r = 0; r < c->world; ++r) {
    w.sizes[r] = blobs[r].bytes;
    w.bases[r] = r == c->rank ? static_cast<char*>(local)
                              : (blobs[r].bytes && c->cfg.transport == 0 ? c->map_blob(blobs[r], &w.maps) : nullptr);
  }
  undo.host = nullptr;  // the window owns them from here
  undo.maps = nullptr;
  for (uint32_t r = 0; r < c->world; ++r) {
    c->host_view.win[id].base[r] = w.bases[r];
    c->host_view.win[id].size[r] = w.sizes[r];
  }
  // (release: the socket transport's receiver thread reads base/size once it sees the bit)
  __atomic_fetch_or(&c->host_view.win_live, 1ull << id, __ATOMIC_RELEASE);
  c->host_view.n_windows = std::max<uint32_t>(c->host_view.n_windows, id + 1);
  if (id == c->windows.size()) c->windows.push_back(std::move(w));
  else c->windows[id] = std::move(w);
  c->sync_view();
  c->barrier();  // no rank leaves before every rank has mapped (runtime.cpp:364-367)
  *window_id = id;
  GIN_API_END
}

int ginsim_cuda_window_deregister(ginsim_cuda_comm_t comm, uint32_t window_id) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  lookup_window(c, window_id);
  DeviceGuard g(c->device);
  GIN_CUDA(cudaDeviceSynchronize());  // no kernel of this rank still uses the window
  Comm::Window& w = c->windows[window_id];
  for (auto& m : w.maps) {
    cuapi().cuMemUnmap(m.ptr, m.size);
    cuapi().cuMemAddressFree(m.ptr, m.size);
    cuapi().cuMemRelease(m.handle);
  }
  if (w.host_registered) cudaHostUnregister(w.host_registered);
  w = Comm::Window{};
  c->host_view.win[window_id] = GinWindowView{};
  c->host_view.win_live &= ~(1ull << window_id);
  c->sync_view();
  GIN_API_END
}

int ginsim_cuda_register_team(ginsim_cuda_comm_t comm, uint32_t team_id, const uint32_t* members, uint32_t n) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  // DevComm::register_team (runtime.cpp:329-337): local, members must be in
  // the world, ids unique (world = id 0 is always present).
  if (n == 0 || !members) fail(GINSIM_E_USAGE, "team must have members");
  if (n > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "team larger than the world");
  for (uint32_t i = 0; i < n; ++i)
    if (members[i] >= c->world) fail(GINSIM_E_INVALID_PEER, "team member " + std::to_string(members[i]) + " out of world");
  if (team_id > 0xFFFFu) fail(GINSIM_E_USAGE, "team id must fit the descriptor's 16-bit team field");
  std::lock_guard<std::mutex> lk(c->mu);
  uint32_t slot = GIN_MAX_TEAMS;
  for (uint32_t i = 0; i < GIN_MAX_TEAMS; ++i) {
    if (c->host_view.teams[i].n && c->host_view.teams[i].id == team_id) fail(GINSIM_E_USAGE, "team id already registered");
    if (!c->host_view.teams[i].n && slot == GIN_MAX_TEAMS) slot = i;
  }
  if (slot == GIN_MAX_TEAMS) fail(GINSIM_E_USAGE, "team table full (" + std::to_string(GIN_MAX_TEAMS) + " teams)");
  GinTeamView t{};
  t.id = team_id;
  t.n = n;
  for (uint32_t i = 0; i < n; ++i) t.members[i] = (uint8_t)members[i];
  c->host_view.teams[slot] = t;  // the proxy agent reads host_view.teams (written before any op names the team)
  {
    DeviceGuard g(c->device);
    GIN_CUDA(cudaMemcpy(&c->dev_view->teams[slot], &t, sizeof(t), cudaMemcpyHostToDevice));
  }
  GIN_API_END
}

int ginsim_cuda_team(ginsim_cuda_comm_t comm, uint32_t team_id, uint32_t* members, uint32_t* n) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  std::lock_guard<std::mutex> lk(c->mu);
  for (uint32_t i = 0; i < GIN_MAX_TEAMS; ++i) {
    const GinTeamView& t = c->host_view.teams[i];
    if (t.n && t.id == team_id) {
      if (n) *n = t.n;
      if (members)
        for (uint32_t j = 0; j < t.n; ++j) members[j] = t.members[j];
      return GINSIM_OK;
    }
  }
  fail(GINSIM_E_USAGE, "team " + std::to_string(team_id) + " not registered");
  GIN_API_END
}

int ginsim_cuda_window_size(ginsim_cuda_comm_t comm, uint32_t window_id, uint32_t rank, uint64_t* bytes) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  const auto& w = lookup_window(c, window_id);
  if (rank >= c->world) fail(GINSIM_E_RANK_OUT_OF_RANGE, "rank not registered in window");
  *bytes = w.sizes[rank];
  GIN_API_END
}

int ginsim_cuda_window_ptr(ginsim_cuda_comm_t comm, uint32_t window_id, uint32_t rank, void** ptr) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  const auto& w = lookup_window(c, window_id);
  if (rank >= c->world) fail(GINSIM_E_RANK_OUT_OF_RANGE, "rank not registered in window");
  *ptr = w.bases[rank];
  GIN_API_END
}

// ------------------------------------------------------------------ host ops
int ginsim_cuda_put(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t dst_win, uint64_t dst_off,
                    uint32_t src_win, uint64_t src_off, uint64_t bytes, const ginsim_cuda_action* action,
                    void* stream) {
  GIN_API_BEGIN
  host_op(comm_impl(comm), ctx, GIN_OP_PUT, peer, dst_win, dst_off, src_win, src_off, bytes, action, (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_put_value(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t dst_win, uint64_t dst_off,
                          uint64_t le_value, uint32_t width, const ginsim_cuda_action* action, void* stream) {
  GIN_API_BEGIN
  host_op(comm_impl(comm), ctx, GIN_OP_PUT_INLINE, peer, dst_win, dst_off, GIN_INLINE_WINDOW, le_value, width, action,
          (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_signal(ginsim_cuda_comm_t comm, uint32_t ctx, uint32_t peer, uint32_t signal_id, uint32_t signal_add,
                       uint64_t operand, const ginsim_cuda_action* extra, void* stream) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (signal_id >= c->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal " + std::to_string(signal_id) + " out of range");
  ginsim_cuda_action a{};
  a.signal_id = (int32_t)signal_id;
  a.signal_add = signal_add;
  a.operand = signal_add ? operand : 1;
  a.counter_id = extra ? extra->counter_id : -1;
  host_op(c, ctx, GIN_OP_SIGNAL_ONLY, peer, 0, 0, GIN_INLINE_WINDOW, 0, 0, &a, (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_flush(ginsim_cuda_comm_t comm, uint32_t ctx, void* stream) {
  GIN_API_BEGIN
  NvtxRange nv("ginsim.flush");
  Comm* c = comm_impl(comm);
  if (ctx >= c->cfg.n_contexts) fail(GINSIM_E_INVALID_CONTEXT, "flush: context out of range");
  if (c->cfg.backend == GIN_BACKEND_PROXY) {
    proxy_host_flush(c, ctx);
  } else {
    DeviceGuard g(c->device);
    GIN_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
  }
  check_device_error(c);
  GIN_API_END
}

static uint64_t read_cells_sum(Comm* c, uint32_t id) {
  DeviceGuard g(c->device);
  std::vector<uint64_t> sub(c->world);
  uint64_t base = 0;
  // the world sub-cells of the cell are a strided column: one 2-D copy
  GIN_CUDA(cudaMemcpy2D(sub.data(), 8, c->host_view.signals[c->rank] + id, (size_t)c->cfg.signal_cells * 8, 8, c->world,
                        cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(&base, c->host_view.signal_base + id, 8, cudaMemcpyDeviceToHost));
  uint64_t sum = 0;
  for (uint64_t x : sub) sum += x;
  return sum - base;
}

static void wait_until(Comm* c, const std::function<bool()>& pred, const char* what) {
  auto deadline = std::chrono::steady_clock::now() + std::chrono::milliseconds(c->cfg.timeout_ms);
  uint32_t idle = 0;
  while (!pred()) {
    proxy_check_failed(c);  // a dead agent is a failure now, not a timeout later (runtime.cpp:280-294)
    if (std::chrono::steady_clock::now() > deadline)
      fail(GINSIM_E_TIMEOUT, std::string(what) + ": exceeded " + std::to_string(c->cfg.timeout_ms) + " ms");
    if (++idle < 128) std::this_thread::yield();
    else std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}

int ginsim_cuda_read_signal(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal " + std::to_string(id) + " out of range");
  *value = read_cells_sum(c, id);
  GIN_API_END
}

int ginsim_cuda_wait_signal(ginsim_cuda_comm_t comm, uint32_t id, uint64_t expected) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal " + std::to_string(id) + " out of range");
  wait_until(c, [&] { return read_cells_sum(c, id) >= expected; }, "wait_signal");
  GIN_API_END
}

int ginsim_cuda_reset_signal(ginsim_cuda_comm_t comm, uint32_t id) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal " + std::to_string(id) + " out of range");
  DeviceGuard g(c->device);
  uint64_t base = 0, sum = 0;
  GIN_CUDA(cudaMemcpy(&base, c->host_view.signal_base + id, 8, cudaMemcpyDeviceToHost));
  sum = read_cells_sum(c, id) + base;
  GIN_CUDA(cudaMemcpy(c->host_view.signal_base + id, &sum, 8, cudaMemcpyHostToDevice));
  GIN_API_END
}

static uint64_t read_counter_raw(Comm* c, uint32_t id) {
  DeviceGuard g(c->device);
  uint64_t v = 0, b = 0;
  GIN_CUDA(cudaMemcpy(&v, c->host_view.counters + id, 8, cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(&b, c->host_view.counter_base + id, 8, cudaMemcpyDeviceToHost));
  return v - b;
}

int ginsim_cuda_read_counter(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.counter_cells) fail(GINSIM_E_INVALID_COUNTER, "counter " + std::to_string(id) + " out of range");
  *value = read_counter_raw(c, id);
  GIN_API_END
}

int ginsim_cuda_wait_counter(ginsim_cuda_comm_t comm, uint32_t id, uint64_t expected) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.counter_cells) fail(GINSIM_E_INVALID_COUNTER, "counter " + std::to_string(id) + " out of range");
  wait_until(c, [&] { return read_counter_raw(c, id) >= expected; }, "wait_counter");
  GIN_API_END
}

int ginsim_cuda_reset_counter(ginsim_cuda_comm_t comm, uint32_t id) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (id >= c->cfg.counter_cells) fail(GINSIM_E_INVALID_COUNTER, "counter " + std::to_string(id) + " out of range");
  if (proxy_counter_pending(c, id) || direct_counter_pending(c, id)) {
    fail(GINSIM_E_RESET_WHILE_OUTSTANDING, "counter " + std::to_string(id) + " still has operations in flight");
  }
  DeviceGuard g(c->device);
  uint64_t v = 0;
  GIN_CUDA(cudaMemcpy(&v, c->host_view.counters + id, 8, cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(c->host_view.counter_base + id, &v, 8, cudaMemcpyHostToDevice));
  GIN_API_END
}

int ginsim_cuda_snapshot_cells(ginsim_cuda_comm_t comm, uint64_t* signals, uint64_t* counters) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  DeviceGuard g(c->device);
  GIN_CUDA(cudaDeviceSynchronize());
  const uint32_t cells = c->cfg.signal_cells;
  std::vector<uint64_t> sub((size_t)c->world * cells), base(cells), ctr(c->cfg.counter_cells), cb(c->cfg.counter_cells);
  GIN_CUDA(cudaMemcpy(sub.data(), c->host_view.signals[c->rank], sub.size() * 8, cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(base.data(), c->host_view.signal_base, cells * 8, cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(ctr.data(), c->host_view.counters, ctr.size() * 8, cudaMemcpyDeviceToHost));
  GIN_CUDA(cudaMemcpy(cb.data(), c->host_view.counter_base, cb.size() * 8, cudaMemcpyDeviceToHost));
  if (signals) {
    for (uint32_t i = 0; i < cells; ++i) {
      uint64_t s = 0;
      for (uint32_t r = 0; r < c->world; ++r) s += sub[(size_t)r * cells + i];
      signals[i] = s - base[i];
    }
  }
  if (counters)
    for (uint32_t i = 0; i < c->cfg.counter_cells; ++i) counters[i] = ctr[i] - cb[i];
  GIN_API_END
}

int ginsim_cuda_device_error(ginsim_cuda_comm_t comm, uint32_t* code, int clear) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  DeviceGuard g(c->device);
  GIN_CUDA(cudaMemcpy(code, c->host_view.error, 4, cudaMemcpyDeviceToHost));
  if (clear) {
    uint32_t z = 0;
    GIN_CUDA(cudaMemcpy(c->host_view.error, &z, 4, cudaMemcpyHostToDevice));
  }
  GIN_API_END
}

int ginsim_cuda_proxy_trace(ginsim_cuda_comm_t comm, double* out, uint32_t max_records, uint32_t* n_out) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->proxy) fail(GINSIM_E_BACKEND_MISMATCH, "proxy_trace on a direct-backend comm");
  DeviceGuard g(c->device);
  *n_out = proxy_trace(c, out, max_records);
  GIN_API_END
}

int ginsim_cuda_proxy_stats(ginsim_cuda_comm_t comm, uint64_t* descriptors, uint64_t* copies, uint64_t* busy_ns,
                            uint64_t* wall_ns) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->proxy) fail(GINSIM_E_BACKEND_MISMATCH, "proxy_stats on a direct-backend comm");
  proxy_stats(c, descriptors, copies, busy_ns, wall_ns);
  GIN_API_END
}

}  // extern "C"

extern "C" int ginsim_cuda_window_register_all(const ginsim_cuda_comm_t* comms, uint32_t n, void* const* ptrs,
                                               const uint64_t* bytes, uint32_t* window_id) {
  GIN_API_BEGIN
  if (n == 0 || n > GIN_MAX_RANKS) fail(GINSIM_E_USAGE, "need 1..8 comms");
  if (!comms || !ptrs || !bytes || !window_id) fail(GINSIM_E_USAGE, "window_register_all: null argument");
  // every handle checked before any rank enters the collective (a null one would leave the others waiting)
  for (uint32_t r = 0; r < n; ++r) comm_impl(comms[r]);
  std::vector<int> rcs(n, 0);
  std::vector<std::string> msgs(n);
  std::vector<uint32_t> ids(n, 0);
  std::vector<std::thread> ts;
  for (uint32_t r = 0; r < n; ++r) {
    ts.emplace_back([&, r] {
      rcs[r] = ginsim_cuda_window_register(comms[r], ptrs[r], bytes[r], &ids[r]);
      if (rcs[r]) msgs[r] = ginsim_cuda_last_error();
    });
  }
  for (auto& t : ts) t.join();
  for (uint32_t r = 0; r < n; ++r) {
    if (!rcs[r]) continue;
    // one rank failed: the ranks that registered release the window again
    for (uint32_t q = 0; q < n; ++q)
      if (!rcs[q]) ginsim_cuda_window_deregister(comms[q], ids[q]);
    fail(rcs[r], "rank " + std::to_string(r) + ": " + msgs[r]);
  }
  *window_id = ids[0];
  GIN_API_END
}
