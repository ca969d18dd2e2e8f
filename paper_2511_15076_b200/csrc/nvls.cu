// nvls.cu — NVLink SHARP (multicast) barrier, SURVEY.md §8(f) f1.
//
// The reference's BarrierSession (proj/core/src/runtime.cpp:638-666) is a
// dissemination barrier: ceil(log2 n) rounds of zero-byte signals on reserved
// cells.  On an NVSwitch box the switch can reduce: every rank binds one
// granule of its memory to a multicast object (cuMulticastCreate /
// AddDevice / BindMem), and one `multimem.red.release.sys.add` through the
// multicast mapping increments the cell on EVERY rank at once.  A barrier is
// then one arrival plus a local acquire-poll for n arrivals per round --
// one round for any n instead of log2(n).  Arrival-only semantics, as the
// reference's (runtime.hpp:308-311).
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>

#include "gin_device.cuh"
#include "runtime_internal.h"

namespace ginsim_b200 {

// Ranks of one process share rank 0's multicast handle object; the last of
// them to tear down releases it (a rank released first would leave the
// others unbinding a dead handle).
static std::mutex g_mc_mu;
static std::map<CUmemGenericAllocationHandle, int> g_mc_refs;

struct NvlsBlob {
  int32_t pid, device, supported, fd;
  uint64_t handle, size;
};

void nvls_setup(Comm* c) {
  const char* env = std::getenv("GINSIM_NVLS");
  // (the socket transport models peers outside the NVLink domain: no multicast)
  const bool want = !(env && env[0] == '0') && c->cfg.transport == 0;
  const CuApi& api = cuapi();
  NvlsBlob me{};
  me.pid = (int32_t)getpid();
  me.device = c->device;
  int sup = 0;
  if (want && c->world > 1 && api.cuMulticastCreate && api.cuDeviceGetAttribute)
    api.cuDeviceGetAttribute(&sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, (CUdevice)c->device);
  me.supported = sup;
  std::vector<NvlsBlob> all(c->world);
  c->allgather(&me, all.data(), sizeof(me));
  // collective decision: every rank supports it and no two ranks share a device
  bool on = c->world > 1;
  for (uint32_t r = 0; r < c->world && on; ++r) {
    if (!all[r].supported) on = false;
    for (uint32_t q = 0; q < r && on; ++q)
      if (all[q].pid == all[r].pid && all[q].device == all[r].device) on = false;
  }
  if (!on) return;
  DeviceGuard g(c->device);
  // Every step is agreed collectively: a rank whose driver refuses a step
  // makes every rank fall back to the dissemination barrier (a rank that
  // threw mid-way would leave the others blocked in the bootstrap).
  auto agree = [&](bool mine_ok) {
    std::vector<uint8_t> oks(c->world);
    uint8_t m = mine_ok ? 1 : 0;
    c->allgather(&m, oks.data(), 1);
    for (uint8_t o : oks)
      if (!o) return false;
    return true;
  };
  auto step = [&](auto&& fn) {
    bool ok = true;
    try {
      fn();
    } catch (const std::exception&) {
      ok = false;
    }
    return agree(ok);
  };
  auto abandon = [&] {
    const CuApi& a = cuapi();
    if (c->nvls.mc_va) { a.cuMemUnmap(c->nvls.mc_va, c->nvls.size); a.cuMemAddressFree(c->nvls.mc_va, c->nvls.size); }
    if (c->nvls.uc_va) { a.cuMemUnmap(c->nvls.uc_va, c->nvls.size); a.cuMemAddressFree(c->nvls.uc_va, c->nvls.size); }
    if (c->nvls.local) a.cuMemRelease(c->nvls.local);
    if (c->nvls.mc) a.cuMemRelease(c->nvls.mc);
    c->nvls = Comm::Nvls{};
    cudaGetLastError();
  };
  CUmulticastObjectProp prop{};
  prop.numDevices = c->world;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  prop.size = 1;
  size_t gran = 0;
  NvlsBlob mc{};
  mc.pid = me.pid;
  mc.fd = -1;
  if (!step([&] {
        GIN_CU(api.cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
        prop.size = gran;
        c->nvls.size = gran;
        if (c->rank == 0) {
          GIN_CU(api.cuMulticastCreate(&c->nvls.mc, &prop));
          int fd = -1;
          GIN_CU(api.cuMemExportToShareableHandle(&fd, c->nvls.mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
          mc.fd = fd;
          mc.handle = c->nvls.mc;
        }
      })) {
    abandon();
    return;
  }
  std::vector<NvlsBlob> mcs(c->world);
  c->allgather(&mc, mcs.data(), sizeof(mc));
  bool shared_handle = false;
  const bool ok_import = step([&] {
    if (c->rank == 0) return;
    const NvlsBlob& o = mcs[0];
    if (o.pid == me.pid) {
      c->nvls.mc = o.handle;  // same process: the very same object (rank 0 releases it)
      shared_handle = true;
      return;
    }
    int pidfd = (int)syscall(SYS_pidfd_open, o.pid, 0);
    if (pidfd < 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "nvls: pidfd_open of rank 0 failed");
    int fd = (int)syscall(SYS_pidfd_getfd, pidfd, o.fd, 0);
    close(pidfd);
    if (fd < 0) fail(GINSIM_E_BOOTSTRAP_TIMEOUT, "nvls: pidfd_getfd of the multicast handle failed");
    GIN_CU(api.cuMemImportFromShareableHandle(&c->nvls.mc, (void*)(uintptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR));
    close(fd);
  });
  if (c->rank == 0 && mc.fd >= 0) close(mc.fd);
  if (!ok_import) {
    if (shared_handle) c->nvls.mc = 0;
    abandon();
    return;
  }
  // every device joins before any memory is bound
  if (!step([&] { GIN_CU(api.cuMulticastAddDevice(c->nvls.mc, (CUdevice)c->device)); })) {
    if (shared_handle) c->nvls.mc = 0;
    abandon();
    return;
  }
  const bool ok_bind = step([&] {
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = c->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    GIN_CU(api.cuMemCreate(&c->nvls.local, gran, &ap, 0));
    GIN_CU(api.cuMulticastBindMem(c->nvls.mc, 0, c->nvls.local, 0, gran, 0));
  });
  if (!ok_bind) {
    if (shared_handle) c->nvls.mc = 0;
    abandon();
    return;
  }
  const bool ok_map = step([&] {
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = c->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    GIN_CU(api.cuMemAddressReserve(&c->nvls.uc_va, gran, gran, 0, 0));
    GIN_CU(api.cuMemMap(c->nvls.uc_va, gran, 0, c->nvls.local, 0));
    GIN_CU(api.cuMemSetAccess(c->nvls.uc_va, gran, &acc, 1));
    GIN_CU(api.cuMemAddressReserve(&c->nvls.mc_va, gran, gran, 0, 0));
    GIN_CU(api.cuMemMap(c->nvls.mc_va, gran, 0, c->nvls.mc, 0));
    GIN_CU(api.cuMemSetAccess(c->nvls.mc_va, gran, &acc, 1));
    GIN_CUDA(cudaMemset((void*)c->nvls.uc_va, 0, gran));
    GIN_CUDA(cudaDeviceSynchronize());
  });  // (the agreement doubles as the barrier: every copy zeroed before anyone arrives)
  if (!ok_map) {
    api.cuMulticastUnbind(c->nvls.mc, (CUdevice)c->device, 0, gran);
    if (shared_handle) c->nvls.mc = 0;
    abandon();
    return;
  }
  c->nvls.on = true;
  c->nvls.shared = shared_handle;
  if (mcs[0].pid == me.pid) {  // rank 0's object, held by every rank of this process
    std::lock_guard<std::mutex> lk(g_mc_mu);
    g_mc_refs[c->nvls.mc] += 1;
  }
  c->host_view.nvls_mc = reinterpret_cast<uint64_t*>(c->nvls.mc_va);
  c->host_view.nvls_uc = reinterpret_cast<uint64_t*>(c->nvls.uc_va);
}

void nvls_teardown(Comm* c) {
  if (!c->nvls.on) return;
  const CuApi& api = cuapi();
  DeviceGuard g(c->device);
  cudaDeviceSynchronize();
  api.cuMemUnmap(c->nvls.mc_va, c->nvls.size);
  api.cuMemAddressFree(c->nvls.mc_va, c->nvls.size);
  api.cuMemUnmap(c->nvls.uc_va, c->nvls.size);
  api.cuMemAddressFree(c->nvls.uc_va, c->nvls.size);
  api.cuMulticastUnbind(c->nvls.mc, (CUdevice)c->device, 0, c->nvls.size);
  api.cuMemRelease(c->nvls.local);
  bool release = true;
  {
    std::lock_guard<std::mutex> lk(g_mc_mu);
    auto it = g_mc_refs.find(c->nvls.mc);
    if (it != g_mc_refs.end()) {  // shared within this process: the last holder releases
      release = --it->second == 0;
      if (release) g_mc_refs.erase(it);
    }
  }
  if (release) api.cuMemRelease(c->nvls.mc);
  c->nvls = Comm::Nvls{};
}

// ------------------------------------------------------------------ barrier bench
struct BarArgs {
  const GinDevCommView* v[GIN_MAX_RANKS];
  uint64_t round0[GIN_MAX_RANKS];  // barriers already completed on the slot
  uint32_t mode, iters, slot;
  uint64_t* ns;                    // [iters], written by lane 0
};

// One thread per rank runs `iters` back-to-back barriers and times each with
// %globaltimer: mode 0 = the reference's dissemination BarrierSession over
// reserved signal cells (runtime.cpp:651-666), mode 1 = NVLS (one
// multimem.red arrival, poll the local copy).
__global__ void barrier_bench_kernel(BarArgs A) {
  if (threadIdx.x != 0) return;
  const GinDevCommView* v = A.v[blockIdx.y];
  gin::Gin gin(v, 0);
  const gin::Team team = gin::WorldTeam(v->world);
  gin::BarrierSession bs(gin, team, A.slot, A.round0[blockIdx.y], /*allow_nvls=*/false);  // mode 0 = dissemination
  gin::CoopThread me;
  for (uint32_t i = 1; i <= A.iters; ++i) {
    const uint64_t t0 = gin::globaltimer();
    if (A.mode == 1) {
      uint64_t* cell = v->nvls_mc + A.slot;
      asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(cell), "l"(1ull) : "memory");
      gin.wait_ge(v->nvls_uc + A.slot, (A.round0[blockIdx.y] + i) * v->world);
    } else {
      bs.sync(me);
    }
    const uint64_t t1 = gin::globaltimer();
    if (blockIdx.y == 0) A.ns[i - 1] = t1 - t0;
  }
}

__global__ void broadcast_kernel(const GinDevCommView* v, uint32_t id, uint64_t amount) {
  gin::signal_broadcast(v, gin::CoopThread{}, id, amount);
}

}  // namespace ginsim_b200

using namespace ginsim_b200;

extern "C" {

int ginsim_cuda_signal_broadcast(ginsim_cuda_comm_t comm, uint32_t id, uint64_t amount, void* stream) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->nvls.on) fail(GINSIM_E_USAGE, "signal broadcast needs the NVLS multicast object (ginsim_cuda_nvls_enabled)");
  if (id >= GIN_BCAST_CELLS) fail(GINSIM_E_INVALID_SIGNAL, "broadcast cell " + std::to_string(id) + " out of range");
  DeviceGuard g(c->device);
  broadcast_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(c->dev_view, id, amount);
  GIN_CUDA(cudaGetLastError());
  GIN_API_END
}

int ginsim_cuda_read_broadcast(ginsim_cuda_comm_t comm, uint32_t id, uint64_t* value) {
  GIN_API_BEGIN
  Comm* c = comm_impl(comm);
  if (!c->nvls.on) fail(GINSIM_E_USAGE, "broadcast cells need the NVLS multicast object");
  if (id >= GIN_BCAST_CELLS) fail(GINSIM_E_INVALID_SIGNAL, "broadcast cell " + std::to_string(id) + " out of range");
  DeviceGuard g(c->device);
  GIN_CUDA(cudaMemcpy(value, reinterpret_cast<uint64_t*>(c->nvls.uc_va) + GIN_BCAST_BASE + id, 8, cudaMemcpyDeviceToHost));
  GIN_API_END
}

int ginsim_cuda_nvls_enabled(ginsim_cuda_comm_t comm, int* enabled) {
  GIN_API_BEGIN
  if (!enabled) fail(GINSIM_E_USAGE, "nvls_enabled: null argument");
  *enabled = comm_impl(comm)->nvls.on ? 1 : 0;
  GIN_API_END
}

int ginsim_cuda_barrier_bench(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t mode, uint32_t iters,
                              uint64_t* ns_out, void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  if (mode > 1) fail(GINSIM_E_USAGE, "mode: 0 dissemination, 1 NVLS");
  if (iters == 0) fail(GINSIM_E_USAGE, "iterations must be positive");
  BarArgs A{};
  A.mode = mode;
  A.iters = iters;
  // barrier slot 2: slot 0 is the world ring's, slot 1 the team ring's; every
  // slot's round count lives in its own host counter
  A.slot = 2;
  A.ns = ns_out;
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (mode == 1 && !c->nvls.on) fail(GINSIM_E_USAGE, "NVLS multicast is not enabled on this comm");
    A.v[i] = c->dev_view;
    std::lock_guard<std::mutex> lk(c->mu);
    A.round0[i] = c->op_counter[3 + mode];
    c->op_counter[3 + mode] += iters;
  }
  DeviceGuard g(comms[0]->impl.device);
  void* args[] = {&A};
  GIN_CUDA(cudaLaunchCooperativeKernel((const void*)barrier_bench_kernel, dim3(1, n), dim3(32), args, 0,
                                       (cudaStream_t)stream));
  GIN_API_END
}

}  // extern "C"
