// kernels_p2p.cu — point-to-point workloads of the reference harness, run as
// device programs over the GIN device API:
//   ping-pong   proj/core/src/harness_bench.cpp:47-90  (K14)
//   all-to-all  SURVEY.md §8(d)-2 (one-sided put+signal on windows, K15)
//   ring        proj/core/src/harness_ring.cpp:18-57   (Listing 2 of the paper)
//   moe-ht      proj/core/src/harness_moe.cpp:283-382  (circular-buffer flow control, K13)
// Every launcher takes the comms this process drives; several comms on one
// device are emulated ranks in ONE cooperative launch (blockIdx.y = rank lane).
#include <algorithm>
#include <map>
#include <cstring>
#include <vector>

#include "gin_device.cuh"
#include "runtime_internal.h"
#include "tma.cuh"

namespace ginsim_b200 {

struct LaneViews {
  const GinDevCommView* v[GIN_MAX_RANKS];
  unsigned int* ws[GIN_MAX_RANKS];
  uint64_t base[GIN_MAX_RANKS];   // per-lane signal baseline / iteration
};

// ------------------------------------------------------------------ ping-pong
struct PingArgs {
  LaneViews lv;
  uint32_t peer0, peer1, send_win, recv_win, sig, iters, warmup, ctas;
  uint64_t bytes;
  uint64_t ready[GIN_MAX_RANKS];   // handshake count (cell sig+1) each lane waits for
  uint64_t raw0[GIN_MAX_RANKS];    // raw sub-cell (this rank, other, sig) at launch: rounds are counted from it
  uint64_t arrive0[GIN_MAX_RANKS]; // multi-CTA rounds: arrivals on workspace word 0 before this call
  uint64_t* rtt;  // device, iters entries (written by peer0's lane)
};

// One put+SignalInc per direction per iteration.  With ctas > 1 the payload
// is split across CTAs and the last CTA of each round issues the release
// (arrival counter), so the signal still covers every CTA's stores.
__global__ void pingpong_kernel(PingArgs A) {
  const GinDevCommView* v = A.lv.v[blockIdx.y];
  unsigned int* ws = A.lv.ws[blockIdx.y];
  const uint64_t base = A.lv.base[blockIdx.y];
  gin::Gin gin(v, 0);
  gin::CoopCta cta;
  const uint32_t me = v->rank;
  if (me != A.peer0 && me != A.peer1) return;
  const bool initiator = me == A.peer0;
  const uint32_t other = initiator ? A.peer1 : A.peer0;
  // Handshake on cell sig+1: each side announces its launch and waits for the
  // other's, so no ping reaches a rank before its host read of the cell the
  // rounds are counted from (the race a slow responder would otherwise lose).
  if (blockIdx.x == 0 && threadIdx.x == 0) gin.release_signal_raw(other, A.sig + 1, 1);
  if (threadIdx.x == 0) gin.wait_ge_signal(A.sig + 1, A.ready[blockIdx.y]);
  __syncthreads();
  const uint32_t total = A.warmup + A.iters;
  const uint64_t chunk = ((A.bytes + A.ctas - 1) / A.ctas + 15) & ~15ull;
  const uint64_t lo = std::min<uint64_t>(A.bytes, chunk * blockIdx.x);
  const uint64_t hi = std::min<uint64_t>(A.bytes, lo + chunk);
  __shared__ int last;
  auto send = [&](uint32_t round) {
    if (hi > lo) {
      gin::coop_copy(cta, gin.window_ptr(A.recv_win, other, lo), gin.window_ptr(A.send_win, me, lo), hi - lo);
    }
    if (A.ctas == 1) {
      cta.sync();
      if (threadIdx.x == 0) gin.release_signal_raw(other, A.sig, 1);
      return;
    }
    cta.sync();
    if (threadIdx.x == 0) {
      gin::fence_acq_rel_sys();
      const unsigned prev = atomicAdd(ws, 1u);
      last = prev + 1 == (unsigned)(A.arrive0[blockIdx.y] + (uint64_t)round * A.ctas);
      if (last) {
        gin::fence_acq_rel_sys();
        gin.release_signal_raw(other, A.sig, 1);
      }
    }
  };
  // one sender per cell: poll its raw sub-cell (one acquire load, no backoff)
  auto wait = [&](uint64_t want) {
    if (threadIdx.x == 0) gin.wait_signal_from(other, A.sig, want);
    cta.sync();
  };
  // ws counts CTA arrivals across calls (whose CTA counts differ with the
  // message size): round i of this call is complete at arrive0 + i*ctas
  (void)base;
  const uint64_t sig0 = A.raw0[blockIdx.y];
  for (uint32_t i = 1; i <= total; ++i) {
    if (initiator) {
      const uint64_t t0 = gin::globaltimer();
      send(i);
      wait(sig0 + i);
      const uint64_t t1 = gin::globaltimer();
      if (blockIdx.x == 0 && threadIdx.x == 0 && i > A.warmup) A.rtt[i - 1 - A.warmup] = t1 - t0;
    } else {
      wait(sig0 + i);
      send(i);
    }
  }
}

// ------------------------------------------------------------------ raw round-trip floor
// The NVLink round trip with no API in the way: one
// thread per rank, a flag word in the peer's signal table written with a
// single store and polled with a single load.  mode 0: st.release.sys /
// ld.acquire.sys polls; mode 1: st.relaxed.sys / ld.relaxed.sys (no
// ordering at all: the fabric floor); mode 2: st.release.sys / relaxed polls
// + one fence.acq_rel.sys once the flag is seen; mode 3: red.release.sys.add
// (the signal path's release) / relaxed polls + one fence; modes 4 / 5 split
// the cost: st.release.sys with relaxed polls, st.relaxed with acquire polls
// (diagnostic only: neither orders anything end to end).
struct FloorArgs {
  const GinDevCommView* v[GIN_MAX_RANKS];
  uint32_t peer0, peer1, sig, iters, warmup, mode;
  uint64_t ready[GIN_MAX_RANKS];  // handshake arrivals expected on cell sig+1 (one per call, host-counted)
  uint64_t* rtt;
};

__global__ void rtt_floor_kernel(FloorArgs A) {
  const GinDevCommView* v = A.v[blockIdx.y];
  if (threadIdx.x != 0) return;
  gin::Gin gin(v, 0);
  const uint32_t me = v->rank;
  if (me != A.peer0 && me != A.peer1) return;
  const bool initiator = me == A.peer0;
  const uint32_t other = initiator ? A.peer1 : A.peer0;
  uint64_t* mine = gin.sub_cell(me, other, A.sig);    // written by the peer
  uint64_t* theirs = gin.sub_cell(other, me, A.sig);  // written by me
  // Launch handshake on cell sig+1: read the flag's current value, then
  // announce this launch and wait for the peer's announcement (the host
  // counts the calls) -- the peer writes the flag only after that, so
  // b_mine precedes its first write.
  const uint64_t b_mine = gin::ld_acquire_sys(mine);
  const uint64_t b_theirs = gin::ld_relaxed_sys(theirs);  // my writes continue from earlier calls
  gin::red_release_sys_add(gin.sub_cell(other, me, A.sig + 1), 1);
  gin.wait_signal_from(other, A.sig + 1, A.ready[blockIdx.y]);
  const uint64_t t_start = gin::globaltimer();
  auto wait = [&](uint64_t want) {
    for (uint32_t s = 1;; ++s) {
      const uint64_t x = (A.mode == 0 || A.mode == 5) ? gin::ld_acquire_sys(mine) : gin::ld_relaxed_sys(mine);
      if (x >= want) {
        if (A.mode == 2 || A.mode == 3) gin::fence_acq_rel_sys();  // one acquire fence after a relaxed poll
        return;
      }
      if ((s & 4095) == 0 && gin::globaltimer() - t_start > v->timeout_ns) {
        gin::raise_error(v, GIN_DEVERR_TIMEOUT);
        return;
      }
    }
  };
  auto post = [&](uint64_t x) {
    if (A.mode == 0 || A.mode == 2 || A.mode == 4) gin::st_release_sys(theirs, x);
    else if (A.mode == 3) gin::red_release_sys_add(theirs, 1);  // the signal path's release-add
    else gin::st_relaxed_sys(theirs, x);
  };
  for (uint32_t i = 1; i <= A.warmup + A.iters; ++i) {
    if (initiator) {
      const uint64_t t0 = gin::globaltimer();
      post(b_theirs + i);
      wait(b_mine + i);
      const uint64_t t1 = gin::globaltimer();
      if (i > A.warmup) A.rtt[i - 1 - A.warmup] = t1 - t0;
    } else {
      wait(b_mine + i);
      post(b_theirs + i);
    }
  }
}

// ------------------------------------------------------------------ windowed bandwidth
// bw_rank_program (harness_bench.cpp:92-129): rank peer0 issues `window` puts
// of `bytes` into peer1's recv window at w*bytes, then flushes, per timed
// iteration; peer1 is passive (one-sided).  On the GPU the puts of an
// iteration are spread over the grid's CTAs (CTA b moves its slice of every
// put), each CTA flushes (fence.acq_rel.sys = local completion) and arrives
// on a counter; the iteration ends when every CTA has arrived, timed by CTA 0.
struct BwArgs {
  LaneViews lv;
  uint32_t peer0, peer1, send_win, recv_win, window, iters, warmup;
  uint64_t bytes;
  uint64_t arrive0[GIN_MAX_RANKS];
  uint64_t* ns;  // iters entries
};

__global__ void bw_kernel(BwArgs A) {
  const GinDevCommView* v = A.lv.v[blockIdx.y];
  if (v->rank != A.peer0) return;
  unsigned int* ctr = A.lv.ws[blockIdx.y] + 1024;
  gin::Gin gin(v, 0);
  gin::CoopCta cta;
  const uint32_t G = gridDim.x;
  const uint64_t per = ((A.bytes + G - 1) / G + 15) & ~15ull;
  const uint64_t lo = std::min<uint64_t>(A.bytes, per * blockIdx.x), hi = std::min<uint64_t>(A.bytes, lo + per);
  for (uint32_t i = 0; i < A.warmup + A.iters; ++i) {
    const uint64_t t0 = gin::globaltimer();
    if (hi > lo)
      for (uint32_t w = 0; w < A.window; ++w)
        gin::coop_copy(cta, gin.window_ptr(A.recv_win, A.peer1, (uint64_t)w * A.bytes + lo),
                       gin.window_ptr(A.send_win, A.peer0, lo), hi - lo);
    gin.flush(cta);  // local completion of this CTA's puts (runtime.cpp:460-470)
    if (threadIdx.x == 0) {
      atomicAdd(ctr, 1u);
      const unsigned target = (unsigned)(A.arrive0[blockIdx.y] + (uint64_t)(i + 1) * G);
      const uint64_t tw = gin::globaltimer();
      while (*reinterpret_cast<volatile unsigned*>(ctr) - target > 0x7FFFFFFFu) {
        if (gin::globaltimer() - tw > v->timeout_ns) {
          gin::raise_error(v, GIN_DEVERR_TIMEOUT);
          break;
        }
      }
      if (blockIdx.x == 0 && i >= A.warmup) A.ns[i - A.warmup] = gin::globaltimer() - t0;
    }
    cta.sync();
  }
}

// ------------------------------------------------------------------ all-to-all
struct A2aArgs {
  LaneViews lv;
  uint32_t send_win, recv_win, sig, ctas_per_peer;
  uint64_t bytes;     // per peer
  uint64_t expected;  // wait target for the local cell
};

constexpr int kA2aThreads = 256;
constexpr int kA2aWarps = kA2aThreads / 32;
constexpr int kA2aStages = 4;
constexpr uint32_t kA2aChunk = 4096;

// CTA b serves peer index b / ctas_per_peer (staggered: peer = me+1+pi, so
// every link is busy from the start) and slice b % ctas_per_peer of its M
// bytes.  Each warp streams its 4 KiB chunks of the slice through a
// 4-stage TMA pipeline (bulk load from the local send window into shared
// memory, bulk store into the peer's recv window over NVLink).  The last CTA
// of each peer releases it with one red.release.sys (SignalInc).
__global__ void __launch_bounds__(kA2aThreads) alltoall_kernel(A2aArgs A) {
  extern __shared__ __align__(128) char smem[];
  const GinDevCommView* v = A.lv.v[blockIdx.y];
  unsigned int* ws = A.lv.ws[blockIdx.y];
  const uint64_t arrivals_before = A.lv.base[blockIdx.y];  // per-peer arrivals of earlier launches
  gin::Gin gin(v, 0);
  const uint32_t n = v->world, me = v->rank;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t pi = blockIdx.x / A.ctas_per_peer, slice = blockIdx.x % A.ctas_per_peer;
  const uint32_t peer = (me + 1 + pi) % n;
  const uint64_t per = ((A.bytes + A.ctas_per_peer - 1) / A.ctas_per_peer + 15) & ~15ull;
  const uint64_t lo = std::min<uint64_t>(A.bytes, per * slice), hi = std::min<uint64_t>(A.bytes, lo + per);
  __shared__ int last;
  const char* src = gin.window_ptr(A.send_win, me, (uint64_t)peer * A.bytes);
  char* dst = gin.window_ptr(A.recv_win, peer, (uint64_t)me * A.bytes);
  if ((((uintptr_t)src | (uintptr_t)dst | A.bytes) & 15) == 0) {
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem) + warp * kA2aStages;
    char* buf = smem + 1024 + (size_t)warp * kA2aStages * kA2aChunk;
    const uint64_t nch = (hi - lo + kA2aChunk - 1) / kA2aChunk;
    if (lane == 0) {
      for (int s = 0; s < kA2aStages; ++s) gin::tma::mbar_init(bars + s, 1);
      gin::tma::fence_mbar_init();
      auto len = [&](uint64_t c) { return (uint32_t)std::min<uint64_t>(kA2aChunk, hi - lo - c * kA2aChunk); };
      for (int s = 0; s < kA2aStages; ++s) {
        const uint64_t c = warp + (uint64_t)s * kA2aWarps;
        if (c < nch) {
          gin::tma::mbar_arrive_expect_tx(bars + s, len(c));
          gin::tma::load(buf + (size_t)s * kA2aChunk, src + lo + c * kA2aChunk, len(c), bars + s);
        }
      }
      for (uint64_t i = 0;; ++i) {
        const uint64_t c = warp + i * kA2aWarps;
        if (c >= nch) break;
        const int s = (int)(i % kA2aStages);
        gin::tma::mbar_wait(bars + s, (uint32_t)((i / kA2aStages) & 1));
        gin::tma::store(dst + lo + c * kA2aChunk, buf + (size_t)s * kA2aChunk, len(c));
        gin::tma::commit();
        gin::tma::wait_read<0>();
        const uint64_t cn = c + (uint64_t)kA2aStages * kA2aWarps;
        if (cn < nch) {
          gin::tma::mbar_arrive_expect_tx(bars + s, len(cn));
          gin::tma::load(buf + (size_t)s * kA2aChunk, src + lo + cn * kA2aChunk, len(cn), bars + s);
        }
      }
      gin::tma::wait_all();
      gin::tma::fence_proxy_async_global();
    }
  } else if (hi > lo) {
    gin::coop_copy(gin::CoopCta{}, dst + lo, src + lo, hi - lo);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    gin::fence_acq_rel_gpu();
    const unsigned prev = atomicAdd(ws + 16 + peer, 1u);
    last = prev + 1 == (unsigned)(arrivals_before + A.ctas_per_peer);
    if (last) gin.release_signal_raw(peer, A.sig, 1);  // red.release.sys: cumulative over the peer's CTAs
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) gin.wait_ge_signal(A.sig, A.expected);
}

// ------------------------------------------------------------------ ordering stress
// acceptance #1 (acceptance.cpp:63-118, fabric.cpp:63-79) on the device API:
// `channels` independent (ctx, src -> dst) channels per rank run in parallel,
// each a stream of put + SignalAdd(1) rounds into a 2-slot ring at the right
// neighbour; the receiving CTA acquires signal >= round+1 and checks EVERY
// byte of that round's put (tagged with sender, channel, round), then hands
// the slot back with a credit signal.  A put the signal did not cover shows up
// as a stale or torn slot -> VERIFY on the device error word.
struct OrderArgs {
  LaneViews lv;
  uint32_t src_win, dst_win, rounds, channels;
  uint64_t bytes;  // per put
};

__device__ __forceinline__ uint32_t order_word(uint32_t sender, uint32_t ch, uint32_t round, uint64_t i) {
  return (sender << 24) ^ (ch << 16) ^ (round * 2654435761u) ^ (uint32_t)(i * 40503u);
}

__global__ void ordering_stress_kernel(OrderArgs A) {
  const GinDevCommView* v = A.lv.v[blockIdx.y];
  const uint64_t base = A.lv.base[blockIdx.y];  // signal values reached by earlier launches
  const uint32_t n = v->world, r = v->rank, right = (r + 1) % n, left = (r + n - 1) % n;
  const uint32_t ch = blockIdx.x % A.channels;
  const bool sender = blockIdx.x < A.channels;
  gin::Gin gin(v, ch % v->n_ctx);
  gin::CoopCta cta;
  const gin::Team world = gin::WorldTeam(n);
  const uint32_t words = (uint32_t)(A.bytes / 4);
  const uint32_t data_cell = ch, credit_cell = A.channels + ch;
  __shared__ int bad;
  for (uint32_t round = 0; round < A.rounds; ++round) {
    const uint64_t slot = (uint64_t)(ch * 2 + (round & 1)) * A.bytes;
    if (sender) {
      if (round >= 2) gin.wait_signal(cta, credit_cell, base + round - 1);  // slot free again
      uint32_t* src = reinterpret_cast<uint32_t*>(gin.window_ptr(A.src_win, r, slot));
      for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) src[i] = order_word(r, ch, round, i);
      cta.sync();
      gin.put(cta, world, right, A.dst_win, slot, A.src_win, slot, A.bytes,
              gin::SignalAction(data_cell, gin::SignalAdd(1)));
    } else {
      gin.wait_signal(cta, data_cell, base + round + 1);
      if (threadIdx.x == 0) bad = 0;
      cta.sync();
      const uint32_t* dst = reinterpret_cast<const uint32_t*>(gin.window_ptr(A.dst_win, r, slot));
      for (uint32_t i = threadIdx.x; i < words; i += blockDim.x) {
        uint32_t w;
        asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(w) : "l"(dst + i) : "memory");
        if (w != order_word(left, ch, round, i)) bad = 1;
      }
      cta.sync();
      if (bad) {
        if (threadIdx.x == 0) gin::raise_error(v, GIN_DEVERR_VERIFY);
        return;
      }
      gin.signal(cta, world, left, credit_cell, gin::SignalAdd(1));  // hand the slot back
    }
  }
}

// ------------------------------------------------------------------ ring
struct RingArgs {
  LaneViews lv;
  uint32_t send_win, recv_win, rounds;
  uint32_t team_id, sig, slot;
  uint64_t bytes;
};

__device__ __forceinline__ uint8_t ring_byte(uint32_t sender, uint32_t round, uint64_t i) {
  return (uint8_t)(sender * 131u + round * 31u + i * 7u + 1u);
}

// harness_ring.cpp:18-57 over a team (world = id 0): team rank i puts to team
// rank (i+1) % |team| at recv[world_rank(i) * S] with SignalInc on `sig`,
// waits, verifies its predecessor's (world rank, round) pattern, resets,
// flushes and syncs a BarrierSession over the team (barrier slot `slot`).
// Ranks outside the team return at once.  Puts and signals name team-relative
// peers, so the Proxy backend's descriptors carry (team id, team rank) and
// the agent resolves them (proxy_backend.cpp:72).
__global__ void ring_kernel(RingArgs A) {
  const GinDevCommView* v = A.lv.v[blockIdx.y];
  gin::Gin gin(v, 0);
  gin::CoopCta cta;
  const gin::Team team = gin.team(A.team_id);
  uint32_t me = team.n;
  for (uint32_t i = 0; i < team.n; ++i)
    if (team.members[i] == v->rank) me = i;
  if (team.n == 0) {
    if (threadIdx.x == 0) gin::raise_error(v, GIN_DEVERR_RANK_OUT_OF_RANGE);
    return;
  }
  if (me == team.n) return;  // not a member
  const uint32_t n = team.n, r = v->rank, peer = (me + 1) % n, pred_w = team.world_rank((me + n - 1) % n);
  const uint32_t peer_w = team.world_rank(peer);
  const uint64_t S = A.bytes;
  gin::BarrierSession barrier(gin, team, A.slot, A.lv.base[blockIdx.y]);
  __shared__ int bad;
  for (uint32_t round = 0; round < A.rounds; ++round) {
    char* send = gin.window_ptr(A.send_win, r, (uint64_t)peer_w * S);
    for (uint64_t i = threadIdx.x; i < S; i += blockDim.x) send[i] = (char)ring_byte(r, round, i);
    cta.sync();
    gin.put(cta, team, peer, A.recv_win, (uint64_t)r * S, A.send_win, (uint64_t)peer_w * S, S,
            gin::SignalAction(A.sig, gin::SignalInc()));
    gin.wait_signal(cta, A.sig, 1);
    if (*reinterpret_cast<volatile unsigned int*>(v->error)) return;  // e.g. an invalid signal id
    if (threadIdx.x == 0) bad = 0;
    cta.sync();
    const char* recv = gin.window_ptr(A.recv_win, r, (uint64_t)pred_w * S);
    for (uint64_t i = threadIdx.x; i < S; i += blockDim.x)
      if ((uint8_t)recv[i] != ring_byte(pred_w, round, i)) bad = 1;
    cta.sync();
    if (bad) {
      if (threadIdx.x == 0) gin::raise_error(v, GIN_DEVERR_VERIFY);
      return;
    }
    if (threadIdx.x == 0) gin.reset_signal(A.sig);
    gin.flush(cta);     // sources reusable before the next round overwrites them
    barrier.sync(cta);  // no peer may signal round+1 before everyone reset
  }
}

// ------------------------------------------------------------------ moe-ht flow control
struct HtArgs {
  const GinDevCommView* pool[GIN_MAX_RANKS][8];  // [rank lane][comm index]
  uint32_t channels, slots, messages, n_pool;
  uint64_t seed;
};

__device__ __forceinline__ uint8_t ht_byte(uint32_t channel, uint32_t msg, uint64_t i, uint64_t seed) {
  return (uint8_t)(seed + channel * 37u + msg * 11u + i);
}

// One CTA per (rank lane, channel).  Producer step then consumer step per
// message, exactly as moe_ht_rank_program; windows 0 = recv, 1 = stage.
__global__ void moe_ht_kernel(HtArgs A) {
  const uint32_t channel = blockIdx.x;
  const uint32_t comm_idx = channel / 4;  // pool_select with n_ctx from the view
  const GinDevCommView* v0 = A.pool[blockIdx.y][0];
  const uint32_t n_ctx = v0->n_ctx;
  const uint32_t ci = channel / n_ctx, ctx = channel % n_ctx;
  (void)comm_idx;
  const GinDevCommView* v = A.pool[blockIdx.y][ci];
  gin::Gin gin(v, ctx);
  gin::CoopCta cta;
  const gin::Team world = gin::WorldTeam(v->world);
  const uint32_t n = v->world, r = v->rank, succ = (r + 1) % n, pred = (r + n - 1) % n;
  const uint32_t B = A.slots, M = A.messages;
  const uint32_t tail_sig = 2 * ctx, head_sig = 2 * ctx + 1, stage_ctr = ctx;
  const uint64_t lane = (uint64_t)ctx * B * 256;
  __shared__ int bad;
  for (uint32_t m = 0; m < M; ++m) {
    // -- producer step
    if (m >= B) {
      gin.wait_signal(cta, head_sig, m + 1 - B);   // remote slot consumed
      gin.wait_counter(cta, stage_ctr, m + 1 - B); // stage slot locally complete
    }
    if (threadIdx.x == 0 && gin.read_signal(head_sig) > m) gin::raise_error(v, GIN_DEVERR_FLOW_CONTROL);
    char* slot = gin.window_ptr(1, r, lane + (uint64_t)(m % B) * 256);
    const uint64_t generation = (uint64_t)m + 1;
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
      slot[i] = i < 8 ? (char)(generation >> (8 * i)) : (char)ht_byte(channel, m, i - 8, A.seed);
    cta.sync();
    gin.put(cta, world, succ, 0, lane + (uint64_t)(m % B) * 256, 1, lane + (uint64_t)(m % B) * 256, 256,
            gin::CounterAction(stage_ctr));
    gin.signal(cta, world, succ, tail_sig, gin::SignalAdd(1));
    // -- consumer step
    gin.wait_signal(cta, tail_sig, m + 1);
    if (threadIdx.x == 0) bad = 0;
    cta.sync();
    const char* got = gin.window_ptr(0, r, lane + (uint64_t)(m % B) * 256);
    for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) {
      const uint8_t want = i < 8 ? (uint8_t)(generation >> (8 * i)) : ht_byte(channel, m, i - 8, A.seed);
      if ((uint8_t)got[i] != want) bad = i < 8 ? 2 : 1;
    }
    cta.sync();
    if (bad) {
      if (threadIdx.x == 0) gin::raise_error(v, bad == 2 ? GIN_DEVERR_FLOW_CONTROL : GIN_DEVERR_VERIFY);
      return;
    }
    gin.signal(cta, world, pred, head_sig, gin::SignalAdd(1));
  }
  gin.wait_signal(cta, head_sig, M);
  gin.flush(cta);
}

// ------------------------------------------------------------------ host helpers
static LaneViews lanes(const ginsim_cuda_comm_t* comms, uint32_t n) {
  LaneViews lv{};
  for (uint32_t i = 0; i < n; ++i) {
    lv.v[i] = comms[i]->impl.dev_view;
    lv.ws[i] = comms[i]->impl.host_view.workspace;
  }
  return lv;
}

static void coop_launch(const void* kernel, dim3 grid, dim3 block, void* arg, cudaStream_t s) {
  void* args[] = {arg};
  GIN_CUDA(cudaLaunchCooperativeKernel(kernel, grid, block, args, 0, s));
}

static void sync_and_check(const ginsim_cuda_comm_t* comms, uint32_t n, cudaStream_t s) {
  GIN_CUDA(cudaStreamSynchronize(s));
  for (uint32_t i = 0; i < n; ++i) check_device_error(&comms[i]->impl);
}

// Host-side per-comm launch/round counters: the device arrival counters in
// the comm workspace are monotone, so each launch passes where they stand.
static uint64_t bump_host_counter(Comm* c, uint32_t slot, uint64_t by) {
  std::lock_guard<std::mutex> lk(c->mu);
  c->op_counter[slot] += by;
  return c->op_counter[slot];
}

}  // namespace ginsim_b200

using namespace ginsim_b200;

extern "C" {

int ginsim_cuda_pingpong(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1,
                         uint32_t send_win, uint32_t recv_win, uint64_t bytes, uint32_t iters, uint32_t warmup,
                         uint32_t signal_id, uint32_t threads, uint64_t* rtt_ns_out, void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  if (peer0 == peer1 || peer0 >= c0->world || peer1 >= c0->world) fail(GINSIM_E_INVALID_PEER, "ping-pong needs two distinct ranks");
  if (signal_id + 1 >= c0->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal out of range (uses signal_id and signal_id+1)");
  if (iters == 0) fail(GINSIM_E_USAGE, "bench iterations must be positive");
  DeviceGuard g(c0->device);
  PingArgs A{};
  A.lv = lanes(comms, n);
  A.peer0 = peer0;
  A.peer1 = peer1;
  A.send_win = send_win;
  A.recv_win = recv_win;
  A.sig = signal_id;
  A.iters = iters;
  A.warmup = warmup;
  A.bytes = bytes;
  A.rtt = rtt_ns_out;
  A.ctas = bytes >= (1u << 20) ? 16 : (bytes >= (256u << 10) ? 4 : 1);
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (c->rank != peer0 && c->rank != peer1) continue;
    for (uint32_t w : {send_win, recv_win}) {
      if (!c->window_live(w)) fail(GINSIM_E_UNKNOWN_WINDOW, "ping-pong window not registered");
    }
    if (c->windows[send_win].sizes[c->rank] < bytes) fail(GINSIM_E_OUT_OF_BOUNDS, "send window smaller than message");
    const uint32_t other = c->rank == peer0 ? peer1 : peer0;
    if (c->windows[recv_win].sizes[other] < bytes) fail(GINSIM_E_OUT_OF_BOUNDS, "peer recv window smaller than message");
    uint64_t cur = 0;
    if (int rc = ginsim_cuda_read_signal(comms[i], signal_id, &cur)) fail(rc, ginsim_cuda_last_error());
    // the arrival counter only advances on multi-CTA launches
    const uint64_t adv = A.ctas > 1 ? (uint64_t)(warmup + iters) * A.ctas : 0;
    A.arrive0[i] = bump_host_counter(c, 0, adv) - adv;
    A.lv.base[i] = cur;
    // raw sub-cell the peer's pings land in (read before the launch; the
    // handshake keeps the peer from pinging before this kernel runs)
    GIN_CUDA(cudaMemcpy(&A.raw0[i], c->host_view.signals[c->rank] + (uint64_t)other * c->cfg.signal_cells + signal_id, 8,
                        cudaMemcpyDeviceToHost));
    // handshake cell sig+1 (dedicated to ping-pong): one arrival per call
    A.ready[i] = bump_host_counter(c, 6, 1);
  }
  // small messages: one warp (the CTA barrier before the release is then a
  // warp barrier); large ones spread the copy over 512 threads per CTA
  const uint32_t thr = threads ? threads : (bytes <= 4096 ? 32 : 512);
  coop_launch((const void*)pingpong_kernel, dim3(A.ctas, n), dim3(thr), &A, (cudaStream_t)stream);
  sync_and_check(comms, n, (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_rtt_floor(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1, uint32_t mode,
                          uint32_t iters, uint32_t warmup, uint32_t signal_id, uint64_t* rtt_ns_out, void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  if (peer0 == peer1 || peer0 >= c0->world || peer1 >= c0->world) fail(GINSIM_E_INVALID_PEER, "needs two distinct ranks");
  if (signal_id + 1 >= c0->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal out of range (uses signal_id and signal_id+1)");
  if (mode > 5)
    fail(GINSIM_E_USAGE, "mode: 0 release/acquire, 1 relaxed, 2 release/relaxed poll+fence, 3 release-add/relaxed "
                         "poll+fence, 4 release/relaxed poll, 5 relaxed/acquire poll");
  if (iters == 0) fail(GINSIM_E_USAGE, "iterations must be positive");
  DeviceGuard g(c0->device);
  FloorArgs A{};
  A.peer0 = peer0;
  A.peer1 = peer1;
  A.sig = signal_id;
  A.iters = iters;
  A.warmup = warmup;
  A.mode = mode;
  A.rtt = rtt_ns_out;
  for (uint32_t i = 0; i < n; ++i) {
    A.v[i] = comms[i]->impl.dev_view;
    Comm* c = comm_impl(comms[i]);
    if (c->rank == peer0 || c->rank == peer1) A.ready[i] = bump_host_counter(c, 9, 1);
  }
  coop_launch((const void*)rtt_floor_kernel, dim3(1, n), dim3(32), &A, (cudaStream_t)stream);
  sync_and_check(comms, n, (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_bw(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t peer0, uint32_t peer1, uint32_t send_win,
                   uint32_t recv_win, uint64_t bytes, uint32_t window, uint32_t iters, uint32_t warmup, uint32_t ctas,
                   uint64_t* ns_out, void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  if (peer0 == peer1 || peer0 >= c0->world || peer1 >= c0->world) fail(GINSIM_E_INVALID_PEER, "needs two distinct ranks");
  if (iters == 0 || window == 0 || bytes == 0) fail(GINSIM_E_USAGE, "bw needs iterations, a window and a size");
  BwArgs A{};
  A.lv = lanes(comms, n);
  A.peer0 = peer0;
  A.peer1 = peer1;
  A.send_win = send_win;
  A.recv_win = recv_win;
  A.window = window;
  A.iters = iters;
  A.warmup = warmup;
  A.bytes = bytes;
  A.ns = ns_out;
  int sms = 0;
  GIN_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c0->device));
  // 256 KiB of each put per CTA, at most one CTA per SM per emulated rank
  const uint32_t G = ctas ? ctas : (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms / n, bytes >> 18));
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (c->rank != peer0) continue;
    if (!c->window_live(send_win) || !c->window_live(recv_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
    if (c->windows[send_win].sizes[peer0] < bytes || c->windows[recv_win].sizes[peer1] < (uint64_t)window * bytes)
      fail(GINSIM_E_OUT_OF_BOUNDS, "windows must hold the message (send) and window * message (peer's recv)");
    const uint64_t adv = (uint64_t)(warmup + iters) * G;
    A.arrive0[i] = bump_host_counter(c, 8, adv) - adv;
  }
  DeviceGuard g(c0->device);
  coop_launch((const void*)bw_kernel, dim3(G, n), dim3(512), &A, (cudaStream_t)stream);
  sync_and_check(comms, n, (cudaStream_t)stream);
  GIN_API_END
}

int ginsim_cuda_alltoall(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t send_win, uint32_t recv_win,
                         uint64_t bytes_per_peer, uint32_t signal_id, uint64_t expected, uint32_t ctas,
                         void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  const uint32_t world = c0->world;
  if (world < 2) fail(GINSIM_E_USAGE, "all-to-all needs at least 2 ranks");
  if (signal_id >= c0->cfg.signal_cells) fail(GINSIM_E_INVALID_SIGNAL, "signal out of range");
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (!c->window_live(send_win) || !c->window_live(recv_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
    for (uint32_t r = 0; r < world; ++r) {
      if (c->windows[recv_win].sizes[r] < (uint64_t)world * bytes_per_peer ||
          c->windows[send_win].sizes[r] < (uint64_t)world * bytes_per_peer)
        fail(GINSIM_E_OUT_OF_BOUNDS, "windows must hold world * bytes_per_peer");
    }
  }
  DeviceGuard g(c0->device);
  A2aArgs A{};
  A.lv = lanes(comms, n);
  A.send_win = send_win;
  A.recv_win = recv_win;
  A.sig = signal_id;
  A.bytes = bytes_per_peer;
  A.expected = expected;
  // occupancy is queried once per device (it is a driver round trip)
  static int sms_of[64] = {0}, cap_of[64] = {0};
  const size_t smem = 1024 + (size_t)kA2aWarps * kA2aStages * kA2aChunk;
  const int dv = c0->device & 63;
  if (!sms_of[dv]) {
    GIN_CUDA(cudaFuncSetAttribute((const void*)alltoall_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    GIN_CUDA(cudaDeviceGetAttribute(&sms_of[dv], cudaDevAttrMultiProcessorCount, c0->device));
    cap_of[dv] = max_coresident_ctas((const void*)alltoall_kernel, kA2aThreads, smem, c0->device);
  }
  const int sms = sms_of[dv], cap_per_dev = cap_of[dv];
  const uint32_t want = ctas ? ctas : (uint32_t)sms;
  uint32_t per_peer = std::max<uint32_t>(1, want / (world - 1));
  const uint64_t max_useful = std::max<uint64_t>(1, bytes_per_peer / (16u << 10));
  per_peer = (uint32_t)std::min<uint64_t>(per_peer, max_useful);
  const int cap = cap_per_dev / (int)n;  // emulated ranks share one device's co-residency
  while (per_peer > 1 && (int)(per_peer * (world - 1)) > cap) --per_peer;
  A.ctas_per_peer = per_peer;
  // the per-peer arrival counters are monotone across launches whose CTA
  // split differs (it follows the message size): pass where they stand
  for (uint32_t i = 0; i < n; ++i) A.lv.base[i] = bump_host_counter(&comms[i]->impl, 1, per_peer) - per_peer;
  const dim3 grid(per_peer * (world - 1), n);
  if (n == 1) {  // one rank per process: CTAs never wait on one another
    alltoall_kernel<<<grid, kA2aThreads, smem, (cudaStream_t)stream>>>(A);
    GIN_CUDA(cudaGetLastError());
  } else {
    void* args[] = {&A};
    GIN_CUDA(cudaLaunchCooperativeKernel((const void*)alltoall_kernel, grid, dim3(kA2aThreads), args, smem,
                                         (cudaStream_t)stream));
  }
  GIN_API_END
}

int ginsim_cuda_ordering_stress(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t src_win, uint32_t dst_win,
                                uint64_t bytes, uint32_t channels, uint32_t rounds, void* stream) {
  GIN_API_BEGIN
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  if (c0->world < 2) fail(GINSIM_E_USAGE, "ordering stress needs at least 2 ranks");
  if (bytes == 0 || bytes % 4 || channels == 0 || 2 * channels > c0->cfg.signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS)
    fail(GINSIM_E_USAGE, "bytes must be a positive multiple of 4; 2*channels signal cells needed");
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (!c->window_live(src_win) || !c->window_live(dst_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
    for (uint32_t r = 0; r < c->world; ++r)
      if (c->windows[src_win].sizes[r] < 2ull * channels * bytes || c->windows[dst_win].sizes[r] < 2ull * channels * bytes)
        fail(GINSIM_E_OUT_OF_BOUNDS, "windows must hold 2 * channels * bytes");
  }
  DeviceGuard g(c0->device);
  OrderArgs A{};
  A.lv = lanes(comms, n);
  A.src_win = src_win;
  A.dst_win = dst_win;
  A.rounds = rounds;
  A.channels = channels;
  A.bytes = bytes;
  // every launch adds `rounds` to each data and credit cell (credits: rounds on
  // the sender side as well), so the base advances by rounds per launch
  for (uint32_t i = 0; i < n; ++i) A.lv.base[i] = bump_host_counter(&comms[i]->impl, 5, rounds) - rounds;
  coop_launch((const void*)ordering_stress_kernel, dim3(2 * channels, n), dim3(256), &A, (cudaStream_t)stream);
  sync_and_check(comms, n, (cudaStream_t)stream);
  GIN_API_END
}

static void ring_launch(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t team_id, uint32_t send_win,
                        uint32_t recv_win, uint64_t bytes, uint32_t rounds, uint32_t sig, void* stream) {
  check_same_device(comms, n);
  Comm* c0 = &comms[0]->impl;
  if (c0->world < 2) fail(GINSIM_E_USAGE, "ring exchange needs at least 2 ranks");
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    if (!c->window_live(send_win) || !c->window_live(recv_win)) fail(GINSIM_E_UNKNOWN_WINDOW, "window not registered");
    for (uint32_t r = 0; r < c->world; ++r)
      if (c->windows[send_win].sizes[r] < c->world * bytes || c->windows[recv_win].sizes[r] < c->world * bytes)
        fail(GINSIM_E_OUT_OF_BOUNDS, "ring windows must hold world * bytes");
  }
  DeviceGuard g(c0->device);
  RingArgs A{};
  A.lv = lanes(comms, n);
  A.send_win = send_win;
  A.recv_win = recv_win;
  A.rounds = rounds;
  A.bytes = bytes;
  A.team_id = team_id;
  A.sig = sig;
  // World rings sync on barrier slot 0, sub-team rings on slot 1.  The round
  // count a BarrierSession continues from is read from the slot's first cell
  // (one signal per completed round; quiescent between launches), so a
  // launch that failed part-way (e.g. a device-side validation error) does
  // not desynchronise later ones.
  A.slot = team_id == 0 ? 0 : 1;
  for (uint32_t i = 0; i < n; ++i) {
    Comm* c = comm_impl(comms[i]);
    uint64_t done = 0;
    if (team_id == 0 && c->nvls.on) {  // the world team's BarrierSession runs on the NVLS cells
      DeviceGuard dg(c->device);
      GIN_CUDA(cudaMemcpy(&done, reinterpret_cast<uint64_t*>(c->nvls.uc_va) + A.slot, 8, cudaMemcpyDeviceToHost));
      done /= c->world;
    } else {
      const uint32_t cell = c->cfg.signal_cells - GIN_BARRIER_SLOTS * GIN_BARRIER_STEPS + A.slot * GIN_BARRIER_STEPS;
      if (int rc = ginsim_cuda_read_signal(comms[i], cell, &done)) fail(rc, ginsim_cuda_last_error());
    }
    A.lv.base[i] = done;
  }
  coop_launch((const void*)ring_kernel, dim3(1, n), dim3(512), &A, (cudaStream_t)stream);
  sync_and_check(comms, n, (cudaStream_t)stream);
}

int ginsim_cuda_ring(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t send_win, uint32_t recv_win, uint64_t bytes,
                     uint32_t rounds, void* stream) {
  GIN_API_BEGIN
  ring_launch(comms, n, 0, send_win, recv_win, bytes, rounds, 0, stream);
  GIN_API_END
}

int ginsim_cuda_team_ring(const ginsim_cuda_comm_t* comms, uint32_t n, uint32_t team_id, uint32_t send_win,
                          uint32_t recv_win, uint64_t bytes, uint32_t rounds, uint32_t signal_id, void* stream) {
  GIN_API_BEGIN
  ring_launch(comms, n, team_id, send_win, recv_win, bytes, rounds, signal_id, stream);
  GIN_API_END
}

int ginsim_cuda_moe_ht_ring(const ginsim_cuda_comm_t* pool, uint32_t n, uint32_t n_pool, uint32_t channels,
                            uint32_t slots, uint32_t messages, uint64_t seed, void* stream) {
  GIN_API_BEGIN
  if (n == 0 || n > GIN_MAX_RANKS || n_pool == 0 || n_pool > 8) fail(GINSIM_E_USAGE, "bad pool shape");
  if (slots == 0 || channels == 0 || messages == 0) fail(GINSIM_E_USAGE, "moe-ht needs slots, channels, and messages");
  if (!pool) fail(GINSIM_E_USAGE, "null communicator pool");
  for (uint32_t i = 0; i < n * n_pool; ++i) comm_impl(pool[i]);
  Comm* c0 = &pool[0]->impl;
  if (c0->world < 2) fail(GINSIM_E_USAGE, "moe-ht needs at least 2 ranks");
  const uint32_t n_ctx = c0->cfg.n_contexts;
  if ((channels + n_ctx - 1) / n_ctx > n_pool) fail(GINSIM_E_USAGE, "comm pool too small for the channel count");
  HtArgs A{};
  for (uint32_t r = 0; r < n; ++r) {
    for (uint32_t p = 0; p < n_pool; ++p) {
      Comm* c = &pool[r * n_pool + p]->impl;
      if (c->device != c0->device) fail(GINSIM_E_USAGE, "emulated ranks must share a device");
      if (!c->window_live(0) || !c->window_live(1)) fail(GINSIM_E_UNKNOWN_WINDOW, "each pool comm needs recv and stage windows");
      if (c->windows[0].sizes[c->rank] < (uint64_t)n_ctx * slots * 256) fail(GINSIM_E_OUT_OF_BOUNDS, "recv window too small");
      A.pool[r][p] = c->dev_view;
    }
  }
  A.channels = channels;
  A.slots = slots;
  A.messages = messages;
  A.n_pool = n_pool;
  A.seed = seed;
  DeviceGuard g(c0->device);
  coop_launch((const void*)moe_ht_kernel, dim3(channels, n), dim3(256), &A, (cudaStream_t)stream);
  std::vector<ginsim_cuda_comm_t> all(pool, pool + n * n_pool);
  sync_and_check(all.data(), n * n_pool, (cudaStream_t)stream);
  GIN_API_END
}

}  // extern "C"
