// gin_device.cuh — sm_100a device-side GIN API (the paper's ncclGin object,
// PAPER.md:551-588), restated for NVLink 5 / NVSwitch peer memory.
//
// Reference semantics followed (all /root/reference-relative):
//   put / put_value / signal     proj/core/src/runtime.cpp:604-633 (Gin)
//   completion actions           proj/core/include/ginsim/types.hpp:45-72
//   ordering (watermark rule)    proj/core/src/fabric.cpp:63-79: when a signal
//       applies at its target, every earlier put on the same (ctx, src->dst)
//       channel is visible.  On NVLink this is a cumulative .sys release
//       issued after the cooperating threads' stores (bar.sync/__syncwarp).
//   waits use >=, reset is the only decrement  runtime.cpp:404-443
//   flush = local completion only              runtime.hpp:158-162
//   BarrierSession dissemination               runtime.cpp:651-666
// Direct backend  = the GDAKI analogue: the calling threads issue the NVLink
//                   stores themselves.
// Proxy backend   = 64-byte descriptors (descriptor.hpp:13-27) published into
//                   a per-context lock-free ring in pinned host memory and
//                   drained by a host thread (proxy.cpp).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gin_types.h"

namespace gin {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_relaxed_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_acquire_sys32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_release_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void red_relaxed_sys_add(uint64_t* p, uint64_t v) {
  asm volatile("red.relaxed.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_sys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// 128-bit streaming load that bypasses L1 allocation (source rows are read
// once per kernel; NVLink destinations are written once).
__device__ __forceinline__ uint4 ld_nc_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
// Coherent (weak, non-.nc) 128-bit load that skips L1 allocation: for data
// other GPUs write into this rank's windows while the reading kernel runs,
// read after the acquire of the flag that publishes it (.nc is only valid for
// data that is read-only for the kernel's whole lifetime).
__device__ __forceinline__ uint4 ld_na_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ uint4 ld_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}
__device__ __forceinline__ void st_v4(void* p, uint4 v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
// 256-bit (LDG/STG .256 on sm_100a) vector moves.
struct u32x8 {
  uint32_t v[8];
};
__device__ __forceinline__ u32x8 ld_nc_v8(const void* p) {
  u32x8 r;
  asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
                 "=r"(r.v[6]), "=r"(r.v[7])
               : "l"(p));
  return r;
}
__device__ __forceinline__ void st_v8(void* p, const u32x8& r) {
  asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r.v[0]),
               "r"(r.v[1]), "r"(r.v[2]), "r"(r.v[3]), "r"(r.v[4]), "r"(r.v[5]), "r"(r.v[6]), "r"(r.v[7])
               : "memory");
}

// ---------------------------------------------------------------- cooperation
// The paper's Coop parameter: which threads act
// together on one operation.  rank() == 0 is the leader that issues the
// signal / counter / descriptor.
struct CoopThread {
  __device__ int rank() const { return 0; }
  __device__ int size() const { return 1; }
  __device__ void sync() const {}
};
struct CoopWarp {
  __device__ int rank() const { return threadIdx.x & 31; }
  __device__ int size() const { return 32; }
  __device__ void sync() const { __syncwarp(); }
};
struct CoopCta {
  __device__ int rank() const {
    return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
  }
  __device__ int size() const { return blockDim.x * blockDim.y * blockDim.z; }
  __device__ void sync() const { __syncthreads(); }
};

// ---------------------------------------------------------------- actions
// proj/core/include/ginsim/types.hpp:27-72 (SignalOp, CompletionAction).
struct SignalOp {
  uint8_t is_add;
  uint64_t operand;
  __device__ __host__ uint64_t amount() const { return is_add ? operand : 1ull; }
};
__device__ __host__ inline SignalOp SignalInc() { return SignalOp{0, 1}; }
__device__ __host__ inline SignalOp SignalAdd(uint64_t v) { return SignalOp{1, v}; }

struct Action {
  int32_t signal_id;   // -1: no remote signal
  int32_t counter_id;  // -1: no local counter
  SignalOp op;
};
__device__ __host__ inline Action NoAction() { return Action{-1, -1, SignalOp{0, 1}}; }
__device__ __host__ inline Action SignalAction(uint32_t id, SignalOp op = SignalOp{0, 1}) {
  return Action{(int32_t)id, -1, op};
}
__device__ __host__ inline Action CounterAction(uint32_t id) { return Action{-1, (int32_t)id, SignalOp{0, 1}}; }
__device__ __host__ inline Action WithCounter(Action a, uint32_t id) {
  a.counter_id = (int32_t)id;
  return a;
}

// Team: an ordered subset of world ranks (types.hpp:75-84).  World = id 0,
// identity.  Sub-teams used on the Proxy backend must be registered on the
// comm (ginsim_cuda_register_team, runtime.cpp:329-343): the descriptor
// carries (team id, team-relative peer) and the host agent resolves it
// (proxy_backend.cpp:72).
struct Team {
  uint32_t id;
  uint32_t n;
  uint8_t members[GIN_MAX_RANKS];
  __device__ __host__ uint32_t world_rank(uint32_t team_rank) const { return members[team_rank]; }
};
__device__ __host__ inline Team WorldTeam(uint32_t world) {
  Team t;
  t.id = 0;
  t.n = world;
  for (uint32_t i = 0; i < GIN_MAX_RANKS; ++i) t.members[i] = (uint8_t)i;
  return t;
}
__device__ __host__ inline Team TeamFromView(const GinTeamView& tv) {
  Team t;
  t.id = tv.id;
  t.n = tv.n;
  for (uint32_t i = 0; i < GIN_MAX_RANKS; ++i) t.members[i] = tv.members[i];
  return t;
}

__device__ __forceinline__ void raise_error(const GinDevCommView* v, unsigned code) {
  atomicCAS(v->error, 0u, code);
}

// ---------------------------------------------------------------- bulk copy
// Cooperative byte copy from local memory to (possibly peer) memory with
// 128-bit vectors when both ends are 16-byte aligned.  Loads are issued
// ahead of stores (4 vectors per lane in flight) to keep NVLink saturated.
template <class Coop>
__device__ __forceinline__ void coop_copy(const Coop& c, char* dst, const char* src, uint64_t bytes) {
  const int r = c.rank(), n = c.size();
  if ((((uintptr_t)dst | (uintptr_t)src) & 15) == 0) {
    const uint64_t nv = bytes >> 4;
    const uint4* s = reinterpret_cast<const uint4*>(src);
    uint4* d = reinterpret_cast<uint4*>(dst);
    uint64_t i = r;
    for (; i + 3ull * n < nv; i += 4ull * n) {
      uint4 a = ld_v4(s + i), b = ld_v4(s + i + n), e = ld_v4(s + i + 2 * n), f = ld_v4(s + i + 3 * n);
      st_v4(d + i, a);
      st_v4(d + i + n, b);
      st_v4(d + i + 2 * n, e);
      st_v4(d + i + 3 * n, f);
    }
    for (; i < nv; i += n) st_v4(d + i, ld_v4(s + i));
    uint64_t j = nv << 4;
    if (j + 8 <= bytes) {  // an 8-byte tail word in one store (small puts: one NVLink write)
      if (r == 0) *reinterpret_cast<uint64_t*>(dst + j) = *reinterpret_cast<const uint64_t*>(src + j);
      j += 8;
    }
    for (j += r; j < bytes; j += n) dst[j] = src[j];
  } else if ((((uintptr_t)dst | (uintptr_t)src) & 7) == 0) {
    uint64_t j = 8ull * r;
    for (; j + 8 <= bytes; j += 8ull * n) *reinterpret_cast<uint64_t*>(dst + j) = *reinterpret_cast<const uint64_t*>(src + j);
    for (uint64_t k = (bytes & ~7ull) + r; k < bytes; k += n) dst[k] = src[k];
  } else {
    for (uint64_t j = r; j < bytes; j += n) dst[j] = src[j];
  }
}

// ---------------------------------------------------------------- the API
// One per-context handle, mirroring Gin (runtime.hpp:260-306) / ncclGin.
class Gin {
 public:
  __device__ Gin(const GinDevCommView* view, uint32_t ctx) : v_(view), ctx_(ctx) {}

  __device__ uint32_t rank() const { return v_->rank; }
  __device__ uint32_t world() const { return v_->world; }
  __device__ uint32_t context() const { return ctx_; }
  __device__ const GinDevCommView* view() const { return v_; }

  // Address of window `w` at `offset` in rank `r`'s region (mapped here).
  __device__ char* window_ptr(uint32_t w, uint32_t r, uint64_t offset) const {
    return v_->win[w].base[r] + offset;
  }

  // --- data movement -------------------------------------------------------
  template <class Coop>
  __device__ void put(const Coop& c, const Team& team, uint32_t peer, uint32_t dst_win,
                      uint64_t dst_off, uint32_t src_win, uint64_t src_off, uint64_t bytes,
                      Action a = NoAction()) const {
    if (!check_op(team, peer, a)) return;
    const uint32_t p = team.world_rank(peer);
    if (!check_range(dst_win, p, dst_off, bytes) || !check_range(src_win, v_->rank, src_off, bytes)) return;
    if (v_->backend == GIN_BACKEND_PROXY) {
      // Loopback (peer == self): a same-device cudaMemcpyAsync runs as a copy
      // KERNEL, which cannot start while the issuing kernel holds every SM
      // (tools/copy_engine_probe.py), so the coop moves the bytes itself and
      // the descriptor carries only the completion action (a zero-byte put).
      const bool loopback = p == v_->rank;
      if (loopback && bytes) coop_copy(c, window_ptr(dst_win, p, dst_off), window_ptr(src_win, v_->rank, src_off), bytes);
      c.sync();
      if (c.rank() == 0) {
        uint8_t flags = 0;
        submit(GIN_OP_PUT, team, peer, dst_win, dst_off, src_win, src_off, loopback ? 0 : bytes, a, flags);
      }
      c.sync();
      return;
    }
    if (bytes) coop_copy(c, window_ptr(dst_win, p, dst_off), window_ptr(src_win, v_->rank, src_off), bytes);
    complete(c, p, a);
  }

  // Inline write of 1..8 little-endian bytes (runtime.hpp:273-283).
  template <class Coop>
  __device__ void put_value_raw(const Coop& c, const Team& team, uint32_t peer, uint32_t dst_win,
                                uint64_t dst_off, uint64_t le_value, uint32_t width,
                                Action a = NoAction()) const {
    if (!check_op(team, peer, a)) return;
    const uint32_t p = team.world_rank(peer);
    if (width == 0 || width > 8) {
      if (c.rank() == 0) raise_error(v_, GIN_DEVERR_OUT_OF_BOUNDS);
      return;
    }
    if (!check_range(dst_win, p, dst_off, width)) return;
    if (v_->backend == GIN_BACKEND_PROXY) {
      c.sync();
      if (c.rank() == 0) {
        uint8_t flags = 0;
        submit(GIN_OP_PUT_INLINE, team, peer, dst_win, dst_off, GIN_INLINE_WINDOW, le_value, width, a, flags);
      }
      c.sync();
      return;
    }
    if (c.rank() == 0) {
      char* d = window_ptr(dst_win, p, dst_off);
      if (width == 8 && ((uintptr_t)d & 7) == 0) {
        *reinterpret_cast<volatile uint64_t*>(d) = le_value;
      } else if (width == 4 && ((uintptr_t)d & 3) == 0) {
        *reinterpret_cast<volatile uint32_t*>(d) = (uint32_t)le_value;
      } else {
        for (uint32_t i = 0; i < width; ++i) reinterpret_cast<volatile char*>(d)[i] = (char)(le_value >> (8 * i));
      }
    }
    complete(c, p, a);
  }
  template <class Coop, class T>
  __device__ void put_value(const Coop& c, const Team& team, uint32_t peer, uint32_t dst_win,
                            uint64_t dst_off, T value, Action a = NoAction()) const {
    static_assert(sizeof(T) <= 8, "inline values are at most 8 bytes");
    uint64_t packed = 0;
    memcpy(&packed, &value, sizeof(T));
    put_value_raw(c, team, peer, dst_win, dst_off, packed, sizeof(T), a);
  }

  // Standalone signal, ordered after every earlier put by this coop on this
  // (ctx, peer) channel (runtime.hpp:285-288).
  template <class Coop>
  __device__ void signal(const Coop& c, const Team& team, uint32_t peer, uint32_t id,
                         SignalOp op = SignalInc(), Action extra = NoAction()) const {
    Action a = extra;
    a.signal_id = (int32_t)id;
    a.op = op;
    if (!check_op(team, peer, a)) return;
    const uint32_t p = team.world_rank(peer);
    if (v_->backend == GIN_BACKEND_PROXY) {
      c.sync();
      if (c.rank() == 0) {
        uint8_t flags = 0;
        submit(GIN_OP_SIGNAL_ONLY, team, peer, 0, 0, GIN_INLINE_WINDOW, 0, 0, a, flags);
      }
      c.sync();
      return;
    }
    complete(c, p, a);
  }

  // Local completion of every op this coop issued on the context
  // (runtime.cpp:460-470).  Direct: the stores were issued by these threads;
  // a .sys fence after the coop barrier makes them performed.  Proxy: wait
  // until the host agent has completed every ticket issued before the call.
  template <class Coop>
  __device__ void flush(const Coop& c) const {
    c.sync();
    if (c.rank() == 0) {
      if (v_->backend == GIN_BACKEND_PROXY) {
        const uint64_t snap = atomicAdd(&v_->proxy.tickets[ctx_], 0ull);
        wait_ge(&v_->proxy.completed[ctx_], snap);
      } else {
        fence_acq_rel_sys();
      }
    }
    c.sync();
  }

  // --- completion state (ID-addressed cells) -------------
  __device__ uint64_t read_signal(uint32_t id) const {
    if (id >= v_->signal_cells) {
      raise_error(v_, GIN_DEVERR_INVALID_SIGNAL);
      return ~0ull;  // waits on an invalid cell end at once (the error word is set)
    }
    uint64_t s = 0;
    for (uint32_t src = 0; src < v_->world; ++src) s += ld_acquire_sys(sub_cell(v_->rank, src, id));
    return s - ld_relaxed_sys(v_->signal_base + id);
  }
  template <class Coop>
  __device__ void wait_signal(const Coop& c, uint32_t id, uint64_t expected) const {
    if (c.rank() == 0) {
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while (read_signal(id) < expected) {
        if (++spins > 64) __nanosleep(spins > 4096 ? 256 : 32);
        if (expired(t0, spins)) {
          raise_error(v_, GIN_DEVERR_TIMEOUT);
          break;
        }
      }
    }
    c.sync();
  }
  // Point-to-point waits for latency-critical handoffs with one known sender:
  // the raw value of the sub-cell `src` writes for cell `id` (its running sum
  // of signals to this rank, never reset by reset_signal), polled with ONE
  // acquire load per iteration and no backoff.  read_signal/wait_signal sum
  // every source's sub-cell instead.
  __device__ uint64_t read_signal_from(uint32_t src, uint32_t id) const {
    if (id >= v_->signal_cells || src >= v_->world) {
      raise_error(v_, id >= v_->signal_cells ? GIN_DEVERR_INVALID_SIGNAL : GIN_DEVERR_INVALID_PEER);
      return ~0ull;
    }
    return ld_acquire_sys(sub_cell(v_->rank, src, id));
  }
  __device__ void wait_signal_from(uint32_t src, uint32_t id, uint64_t raw_target) const {
    if (id >= v_->signal_cells || src >= v_->world) {
      raise_error(v_, id >= v_->signal_cells ? GIN_DEVERR_INVALID_SIGNAL : GIN_DEVERR_INVALID_PEER);
      return;
    }
    // acquire polls: measured cheaper than relaxed polls followed by one
    // fence.acq_rel.sys (rtt_floor modes 0 vs 2: 5.8 vs 8.9 us round trip)
    const uint64_t* p = sub_cell(v_->rank, src, id);
    const uint64_t t0 = globaltimer();
    for (uint32_t spins = 1; ld_acquire_sys(p) < raw_target; ++spins) {
      if ((spins & 4095) == 0 && expired(t0, 256)) {
        raise_error(v_, GIN_DEVERR_TIMEOUT);
        break;
      }
    }
  }

  // Reset sets the cell to 0 (runtime.cpp:414-418); only the owner may call
  // it, and only when no signal to the cell is in flight.
  __device__ void reset_signal(uint32_t id) const {
    if (id >= v_->signal_cells) {
      raise_error(v_, GIN_DEVERR_INVALID_SIGNAL);
      return;
    }
    uint64_t s = 0;
    for (uint32_t src = 0; src < v_->world; ++src) s += ld_acquire_sys(sub_cell(v_->rank, src, id));
    st_relaxed_sys(v_->signal_base + id, s);
  }
  __device__ uint64_t read_counter(uint32_t id) const {
    if (id >= v_->counter_cells) {
      raise_error(v_, GIN_DEVERR_INVALID_COUNTER);
      return ~0ull;
    }
    return ld_acquire_sys(v_->counters + id) - ld_relaxed_sys(v_->counter_base + id);
  }
  template <class Coop>
  __device__ void wait_counter(const Coop& c, uint32_t id, uint64_t expected) const {
    if (c.rank() == 0) {
      const uint64_t t0 = globaltimer();
      uint32_t spins = 0;
      while (read_counter(id) < expected) {
        if (++spins > 64) __nanosleep(32);
        if (expired(t0, spins)) {
          raise_error(v_, GIN_DEVERR_TIMEOUT);
          break;
        }
      }
    }
    c.sync();
  }
  __device__ void reset_counter(uint32_t id) const {
    if (id >= v_->counter_cells) {
      raise_error(v_, GIN_DEVERR_INVALID_COUNTER);
      return;
    }
    st_relaxed_sys(v_->counter_base + id, ld_acquire_sys(v_->counters + id));
  }

  // Raw signal cell of (dst rank, written by src) — the NVLink target of a
  // signal from src.  Exposed for fused kernels that batch their releases.
  __device__ uint64_t* sub_cell(uint32_t dst, uint32_t src, uint32_t id) const {
    return v_->signals[dst] + (uint64_t)src * v_->signal_cells + id;
  }

  // Release-add `amount` to cell `id` of world rank `dst` on behalf of this
  // rank; cumulative over everything that happens-before the calling thread.
  // GPU scope when dst lives on this GPU (emulated ranks), else system scope.
  __device__ void release_signal_raw(uint32_t dst, uint32_t id, uint64_t amount) const {
    if ((v_->same_gpu >> dst) & 1u) {
      fence_acq_rel_gpu();
      red_relaxed_sys_add(sub_cell(dst, v_->rank, id), amount);
    } else {
      red_release_sys_add(sub_cell(dst, v_->rank, id), amount);
    }
  }
  // The fence a release toward rank `dst` needs: GPU scope on this GPU.
  __device__ void fence_toward(uint32_t dst) const {
    if ((v_->same_gpu >> dst) & 1u) fence_acq_rel_gpu();
    else fence_acq_rel_sys();
  }

  // Single-thread wait until cell `id` >= expected (no coop barrier).
  __device__ void wait_ge_signal(uint32_t id, uint64_t expected) const {
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while (read_signal(id) < expected) {
      if (++spins > 64) __nanosleep(32);
      if (expired(t0, spins)) {
        raise_error(v_, GIN_DEVERR_TIMEOUT);
        break;
      }
    }
  }

  __device__ void wait_ge(const uint64_t* p, uint64_t expected) const {
    const uint64_t t0 = globaltimer();
    uint32_t spins = 0;
    while (ld_acquire_sys(p) < expected) {
      if (++spins > 64) __nanosleep(64);
      if (expired(t0, spins)) {
        raise_error(v_, GIN_DEVERR_TIMEOUT);
        break;
      }
    }
  }

  // Bounded spin: true once the comm timeout has elapsed (the caller raises
  // Timeout) or another thread has already raised a device error.
  __device__ bool expired(uint64_t t0, uint32_t spins) const {
    if ((spins & 255) != 0) return false;
    if (*reinterpret_cast<volatile unsigned int*>(v_->error) != 0) return true;
    return globaltimer() - t0 > v_->timeout_ns;
  }

  // A registered team of this comm by id (DevComm::team, runtime.cpp:338-343);
  // an unknown id yields an empty team (every op on it raises RankOutOfRange).
  __device__ Team team(uint32_t id) const {
    for (uint32_t i = 0; i < GIN_MAX_TEAMS; ++i)
      if (v_->teams[i].n && v_->teams[i].id == id) return TeamFromView(v_->teams[i]);
    Team t = WorldTeam(v_->world);
    t.id = id;
    t.n = 0;
    return t;
  }

 private:
  // submit_op validation (runtime.cpp:474-507): team-relative peer in range
  // (team_translate -> RankOutOfRange, types.cpp:14-20), world rank in range,
  // signal and counter ids inside their tables.
  __device__ bool check_op(const Team& team, uint32_t peer, const Action& a) const {
    unsigned code = 0;
    if (peer >= team.n) code = GIN_DEVERR_RANK_OUT_OF_RANGE;
    else if (team.members[peer] >= v_->world) code = GIN_DEVERR_INVALID_PEER;
    else if (a.signal_id >= 0 && (uint32_t)a.signal_id >= v_->signal_cells) code = GIN_DEVERR_INVALID_SIGNAL;
    else if (a.counter_id >= 0 && (uint32_t)a.counter_id >= v_->counter_cells) code = GIN_DEVERR_INVALID_COUNTER;
    if (code) raise_error(v_, code);
    return code == 0;
  }

  __device__ bool check_range(uint32_t w, uint32_t r, uint64_t off, uint64_t len) const {
    if (w >= GIN_MAX_WINDOWS || !((v_->win_live >> w) & 1ull) || r >= v_->world) {
      raise_error(v_, r >= v_->world ? GIN_DEVERR_INVALID_PEER : GIN_DEVERR_UNKNOWN_WINDOW);
      return false;
    }
    const uint64_t cap = v_->win[w].size[r];
    if (off > cap || len > cap - off) {  // overflow-safe, types.cpp:52-60
      raise_error(v_, GIN_DEVERR_OUT_OF_BOUNDS);
      return false;
    }
    return true;
  }

  // Direct completion: coop barrier, then the leader issues the cumulative
  // release (the signal) and/or the local-completion counter bump.
  template <class Coop>
  __device__ void complete(const Coop& c, uint32_t peer, const Action& a) const {
    if (a.signal_id < 0 && a.counter_id < 0) return;
    c.sync();
    if (c.rank() == 0) {
      if (a.signal_id >= 0) release_signal_raw(peer, (uint32_t)a.signal_id, a.op.amount());
      if (a.counter_id >= 0) {
        fence_toward(peer);  // the put is performed where its observers are, then counted
        atomicAdd(reinterpret_cast<unsigned long long*>(v_->counters + a.counter_id), 1ull);
      }
    }
  }

  // Proxy producer (K8): ticket, wait for the slot, write 64 bytes, publish
  // (proj/core/src/proxy_backend.cpp:19-29).  Little-endian struct image ==
  // encode_descriptor's byte layout (descriptor.hpp:13-27).
  __device__ void submit(uint8_t opcode, const Team& team, uint32_t peer, uint32_t dst_win,
                         uint64_t dst_off, uint32_t src_win, uint64_t src_or_value, uint64_t bytes,
                         const Action& a, uint8_t flags) const {
    uint64_t w[8];
    uint32_t sig_id = 0, ctr_id = 0;
    uint64_t operand = 0;
    if (a.signal_id >= 0) {
      flags |= GIN_FLAG_HAS_SIGNAL;
      sig_id = (uint32_t)a.signal_id;
      if (a.op.is_add) {
        flags |= GIN_FLAG_SIGNAL_IS_ADD;
        operand = a.op.operand;
      } else {
        operand = 1;
      }
    }
    if (a.counter_id >= 0) {
      flags |= GIN_FLAG_HAS_COUNTER;
      ctr_id = (uint32_t)a.counter_id;
    }
    // (team id, team-relative peer) as the reference's descriptor carries them;
    // the agent resolves the world rank (proxy_backend.cpp:72)
    const uint16_t team_id = (uint16_t)team.id;
    w[0] = (uint64_t)opcode | ((uint64_t)flags << 8) | ((uint64_t)team_id << 16) | ((uint64_t)peer << 32);
    w[1] = (uint64_t)dst_win | ((uint64_t)src_win << 32);
    w[2] = dst_off;
    w[3] = src_or_value;
    w[4] = bytes;
    w[5] = (uint64_t)sig_id | ((uint64_t)ctr_id << 32);
    w[6] = operand;
    w[7] = 0;
    const GinProxyView& px = v_->proxy;
    const unsigned long long ticket = atomicAdd(&px.tickets[ctx_], 1ull);
    GinRingSlot* slot = px.slots[ctx_] + (ticket & px.mask);
    // Backpressure: a full ring spins until the host agent has consumed
    // ticket - capacity (proxy_backend.cpp:24-26), read from the agent's
    // consumed counter rather than the slot's seq word (see gin_types.h).
    if (ticket > px.mask) wait_ge(px.consumed + ctx_, ticket - px.mask);
    uint64_t* dst = reinterpret_cast<uint64_t*>(slot->bytes);
#pragma unroll
    for (int i = 0; i < 8; ++i) st_relaxed_sys(dst + i, w[i]);
    st_release_sys(&slot->seq, ticket + 1);
  }

  const GinDevCommView* v_;
  uint32_t ctx_;
};

// Dissemination barrier over a team on the reserved signal cells
// (runtime.hpp:312-327, runtime.cpp:651-666).  Arrival-only semantics.
class BarrierSession {
 public:
  // `round` = barriers this rank already completed on the slot.  The world
  // team uses the NVLS multicast barrier when the comm bound one
  // (allow_nvls; every rank of a comm agrees on it, nvls.cu): one arrival
  // through the switch instead of ceil(log2 n) signal rounds.
  __device__ BarrierSession(const Gin& gin, const Team& team, uint32_t slot, uint64_t round, bool allow_nvls = true)
      : gin_(gin), team_(team), slot_(slot), round_(round) {
    my_ = 0;
    for (uint32_t i = 0; i < team.n; ++i)
      if (team.members[i] == gin.rank()) my_ = i;
    nvls_ = allow_nvls && gin.view()->nvls_mc != nullptr && team.id == 0 && team.n == gin.world();
  }
  template <class Coop>
  __device__ void sync(const Coop& c) {
    round_++;
    const uint32_t n = team_.n;
    if (n <= 1) return;
    if (nvls_) {
      c.sync();
      if (c.rank() == 0) {
        const GinDevCommView* v = gin_.view();
        asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(v->nvls_mc + slot_), "l"(1ull)
                     : "memory");
        gin_.wait_ge(v->nvls_uc + slot_, round_ * n);
      }
      c.sync();
      return;
    }
    const uint32_t base = gin_.view()->signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS + slot_ * GIN_BARRIER_STEPS;
    for (uint32_t k = 0; (1u << k) < n; ++k) {
      const uint32_t dst = (my_ + (1u << k)) % n;
      gin_.signal(c, team_, dst, base + k, SignalInc());
      gin_.wait_signal(c, base + k, round_);
    }
  }
  __device__ uint64_t round() const { return round_; }
  __device__ bool multicast() const { return nvls_; }

 private:
  const Gin& gin_;
  Team team_;
  uint32_t slot_, my_;
  uint64_t round_;
  bool nvls_;
};

// Multicast signal broadcast: one multimem.red through
// the NVLS mapping adds `amount` to broadcast cell `id` on EVERY rank of the
// comm (the switch performs the fan-out).  A separate cell namespace from the
// per-rank signal table (its cells live in the multicast granule); needs
// nvls (Comm bound a multicast object), else raises UsageError-equivalent
// GIN_DEVERR_INVALID_SIGNAL.  Release semantics: everything the calling
// thread wrote before is visible to a rank that observes the new value.
__device__ __forceinline__ bool broadcast_ok(const GinDevCommView* v, uint32_t id) {
  if (v->nvls_mc == nullptr || id >= GIN_BCAST_CELLS) {
    raise_error(v, GIN_DEVERR_INVALID_SIGNAL);
    return false;
  }
  return true;
}
template <class Coop>
__device__ void signal_broadcast(const GinDevCommView* v, const Coop& c, uint32_t id, uint64_t amount) {
  if (!broadcast_ok(v, id)) return;
  c.sync();
  if (c.rank() == 0)
    asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(v->nvls_mc + GIN_BCAST_BASE + id),
                 "l"(amount)
                 : "memory");
}
__device__ __forceinline__ uint64_t read_broadcast(const GinDevCommView* v, uint32_t id) {
  if (!broadcast_ok(v, id)) return ~0ull;
  return ld_acquire_sys(v->nvls_uc + GIN_BCAST_BASE + id);
}

}  // namespace gin
