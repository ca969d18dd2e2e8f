// runtime_internal.h — host-side communicator state behind the C ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/ginsim_cuda.h"
#include "gin_types.h"

namespace ginsim_b200 {

// Internal exception carrying a C-ABI status; the C layer converts it.
struct GinError : std::runtime_error {
  int code;
  GinError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] void fail(int code, const std::string& msg);
void set_last_error(const char* msg);
#define GIN_API_BEGIN try {
#define GIN_API_END                                      \
  return GINSIM_OK;                                      \
  }                                                      \
  catch (const ::ginsim_b200::GinError& e) {             \
    ::ginsim_b200::set_last_error(e.what());             \
    return e.code;                                       \
  }                                                      \
  catch (const std::exception& e) {                      \
    ::ginsim_b200::set_last_error(e.what());             \
    return GINSIM_E_GENERIC;                             \
  }
void cuda_check(cudaError_t e, const char* what);
void cu_check(CUresult r, const char* what);
#define GIN_CUDA(x) ::ginsim_b200::cuda_check((x), #x)
#define GIN_CU(x) ::ginsim_b200::cu_check((x), #x)


// Driver API through cudaGetDriverEntryPoint: the library never links
// libcuda, so it loads (and its host-only codec runs) on a machine without a
// GPU driver; the first driver call resolves the table or fails loudly.
struct CuApi {
  decltype(&::cuStreamWriteValue64) cuStreamWriteValue64 = nullptr;
  decltype(&::cuStreamBatchMemOp) cuStreamBatchMemOp = nullptr;
  decltype(&::cuGetErrorString) cuGetErrorString = nullptr;
  decltype(&::cuMemAddressFree) cuMemAddressFree = nullptr;
  decltype(&::cuMemAddressReserve) cuMemAddressReserve = nullptr;
  decltype(&::cuMemCreate) cuMemCreate = nullptr;
  decltype(&::cuMemExportToShareableHandle) cuMemExportToShareableHandle = nullptr;
  decltype(&::cuMemGetAllocationGranularity) cuMemGetAllocationGranularity = nullptr;
  decltype(&::cuMemImportFromShareableHandle) cuMemImportFromShareableHandle = nullptr;
  decltype(&::cuMemMap) cuMemMap = nullptr;
  decltype(&::cuMemRelease) cuMemRelease = nullptr;
  decltype(&::cuMemSetAccess) cuMemSetAccess = nullptr;
  decltype(&::cuMemUnmap) cuMemUnmap = nullptr;
  // NVLink SHARP multicast (optional: null when the driver lacks them)
  decltype(&::cuMulticastCreate) cuMulticastCreate = nullptr;
  decltype(&::cuMulticastAddDevice) cuMulticastAddDevice = nullptr;
  decltype(&::cuMulticastBindMem) cuMulticastBindMem = nullptr;
  decltype(&::cuMulticastUnbind) cuMulticastUnbind = nullptr;
  decltype(&::cuMulticastGetGranularity) cuMulticastGetGranularity = nullptr;
  decltype(&::cuDeviceGetAttribute) cuDeviceGetAttribute = nullptr;
};
const CuApi& cuapi();

// NVTX range over a host entry point (header-only NVTX v3: a no-op unless a
// tool such as nsys / ncu --nvtx injects itself), so a profile shows which
// ginsim call launched what (SURVEY.md §5 tracing).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

// Scoped current-device switch.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev);
  ~DeviceGuard();
};

// One exportable VMM allocation (cuMemCreate + cuMemMap) owned by this process.
struct VmmAlloc {
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr ptr = 0;
  uint64_t size = 0;  // granularity-rounded
  int device = 0;
  int fd = -1;        // exported POSIX FD, kept open while the allocation lives
};

// Blob exchanged through the bootstrap for every window / signal table.
struct ExportBlob {
  int32_t pid;
  int32_t fd;
  int32_t device;
  int32_t is_vmm;
  uint64_t alloc_size;
  uint64_t offset;      // of the region inside the allocation
  uint64_t bytes;       // region size (window capacity)
  uint64_t ptr;         // owner's VA of the region (valid in the owner process)
  uint32_t window_id;
  uint32_t pad;
};

struct Mapping {  // an imported peer allocation
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr ptr = 0;
  uint64_t size = 0;
};

struct ProxyAgent;  // proxy.cu
struct ProxyDeleter {
  void operator()(ProxyAgent* p) const;
};
using ProxyPtr = std::unique_ptr<ProxyAgent, ProxyDeleter>;
struct NetTransport;  // net.cu: the Proxy backend's socket transport (Config.transport = 1)
struct NetDeleter {
  void operator()(NetTransport* t) const;
};
using NetPtr = std::unique_ptr<NetTransport, NetDeleter>;

struct Comm {
  uint32_t rank = 0, world = 1;
  int device = 0;
  ginsim_cuda_config cfg{};
  ginsim_cuda_bootstrap boot{};

  VmmAlloc signal_alloc;                      // [world][signal_cells] u64, exported
  void* local_block = nullptr;                // cudaMalloc: bases, counters, error, workspace
  std::vector<Mapping> imported;              // peer mappings owned by this comm
  std::vector<std::pair<uint64_t, uint64_t>> window_sizes_dummy;

  struct Window {
    bool live = false;                       // false after window_deregister (the id is free again)
    std::vector<uint64_t> sizes;
    std::vector<char*> bases;
    std::vector<Mapping> maps;               // peer regions imported for this window (other processes)
    void* host_registered = nullptr;         // host-memory window: the pages this rank cudaHostRegister'ed
  };
  std::vector<Window> windows;                // indexed by window id
  bool window_live(uint32_t w) const { return w < windows.size() && windows[w].live; }

  // host-issued direct-backend ops carrying a local counter, not yet known
  // complete: (event after the op, counter id); reset_counter refuses while
  // one is outstanding (runtime.cpp:431-438)
  std::vector<std::pair<cudaEvent_t, uint32_t>> direct_pending;
  std::vector<cudaEvent_t> free_op_events;

  GinDevCommView host_view{};
  GinDevCommView* dev_view = nullptr;         // device copy

  std::map<CUdeviceptr, VmmAlloc> allocs;     // ginsim_cuda_mem_alloc'd regions
  std::mutex mu;

  // NVLS multicast barrier region (nvls.cu): one granule bound on every rank
  struct Nvls {
    bool on = false, shared = false;  // shared: rank 0's handle object in this process
    CUmemGenericAllocationHandle mc = 0, local = 0;
    CUdeviceptr mc_va = 0, uc_va = 0;
    uint64_t size = 0;
  } nvls;

  cudaStream_t op_stream = nullptr;           // host-issued ops / cell reads
  bool shares_device = false;                 // another rank of this comm runs on this device in this process
  uint32_t moe_cells_next = 0;                // next never-used signal cell for a MoE handle
  std::vector<std::pair<uint32_t, uint32_t>> moe_cells_free;  // (first, span) ranges released by moe_destroy
  uint64_t op_counter[16] = {};                // per-workload launch/round counters (host side)
  ProxyPtr proxy;

  void allgather(const void* send, void* recv, size_t bytes);
  void barrier();
  void sync_view();                           // push host_view to dev_view
  // import a peer region into this process; a new mapping is recorded in
  // *maps (or in `imported` when maps is null)
  char* map_blob(const ExportBlob& b, std::vector<Mapping>* maps = nullptr);
};

// Launch helpers shared by the kernel translation units.
void check_same_device(const ginsim_cuda_comm_t* comms, uint32_t n);
int max_coresident_ctas(const void* kernel, int threads, size_t smem, int device);
void check_device_error(Comm* c);

// NVLS multicast barrier (nvls.cu): collective setup after the signal tables,
// teardown at comm destroy.  Disabled (nvls.on = false) without multicast
// support, with ranks sharing a device, or with GINSIM_NVLS=0.
void nvls_setup(Comm* c);
void nvls_teardown(Comm* c);

// Proxy agent lifecycle (proxy.cu).
ProxyPtr proxy_start(Comm* c);
void proxy_stop(ProxyPtr& p);
uint64_t proxy_host_submit(Comm* c, uint32_t ctx, const uint8_t desc[64]);  // returns the op's host ticket on ctx
bool proxy_host_done(Comm* c, uint32_t ctx, uint64_t ticket);
void proxy_check_failed(Comm* c);  // throws the agent's failure (no-op without an agent)
// A host-issued op through submit_op's validation (runtime.cu); returns the
// proxy host ticket (0 on the direct backend, which launches on `stream`).
uint64_t host_op(Comm* c, uint32_t ctx, uint8_t opcode, uint32_t peer, uint32_t dst_win, uint64_t dst_off,
                 uint32_t src_win, uint64_t src_or_value, uint64_t bytes, const ginsim_cuda_action* action,
                 cudaStream_t stream);
void proxy_host_flush(Comm* c, uint32_t ctx);
bool proxy_counter_pending(Comm* c, uint32_t id);
// Waits until the agent has consumed and completed every descriptor the GPU
// has submitted so far (all contexts) and every host-submitted op.
void proxy_quiesce(Comm* c);
// Zeroes the agent's running values of signal cells [first, first+span) toward
// every peer (the cells' owners zero their sub-cells at the same time).
void proxy_reset_cells(Comm* c, uint32_t first, uint32_t span);
void proxy_stats(Comm* c, uint64_t* descs, uint64_t* copies, uint64_t* busy_ns, uint64_t* wall_ns);
uint32_t proxy_trace(Comm* c, double* out, uint32_t max_records);
NetTransport* proxy_net(Comm* c);  // the agent's socket transport (null on the fabric)

// Socket transport (net.cu), driven by the proxy agent's thread.  Collective
// setup over the comm's bootstrap; puts return the peer connection's last
// sequence number (acked[peer] reaches it once the peer has performed them).
NetPtr net_start(Comm* c);
uint64_t net_put(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t win, uint64_t off, const char* dev_src,
                 uint64_t bytes, cudaStream_t stream);
uint64_t net_put_inline(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t win, uint64_t off, uint64_t value,
                        uint32_t bytes);
void net_signal(NetTransport* t, uint32_t peer, uint32_t ctx, uint32_t id, bool add, uint64_t operand);
uint64_t* net_acked_device(NetTransport* t, uint32_t peer);
uint64_t net_last_seq(NetTransport* t, uint32_t peer);
void net_release_waits(NetTransport* t);  // teardown past the timeout: unblock the completion stream
void net_reset_cells(NetTransport* t, uint32_t first, uint32_t span);
void net_check_failed(NetTransport* t);
void net_stats(NetTransport* t, uint64_t* tx_frames, uint64_t* rx_puts, uint64_t* rx_bytes);

// Descriptor codec (descriptor.cpp).
int descriptor_check(const ginsim_cuda_descriptor* d);
void descriptor_encode(const ginsim_cuda_descriptor* d, uint8_t out[64]);  // throws InvalidDescriptor
void descriptor_decode(const uint8_t in[64], ginsim_cuda_descriptor* d);   // throws MalformedDescriptor

}  // namespace ginsim_b200

struct ginsim_cuda_comm_s {
  ginsim_b200::Comm impl;
};

// The runtime behind a C-ABI comm handle; a null handle is a UsageError
// (inside GIN_API_BEGIN / GIN_API_END, so the caller gets GINSIM_E_USAGE).
inline ginsim_b200::Comm* comm_impl(ginsim_cuda_comm_t comm) {
  if (!comm) ginsim_b200::fail(GINSIM_E_USAGE, "null communicator handle");
  return &comm->impl;
}
