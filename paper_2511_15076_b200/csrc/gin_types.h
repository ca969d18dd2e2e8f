// gin_types.h — POD types shared by the host runtime and the sm_100a device API.
//
// The device-side communicator view is the B200 analogue of the state a
// reference DevComm owns (proj/core/include/ginsim/runtime.hpp:123-246): rank,
// world, the signal/counter tables (runtime.hpp:230-232), and the window
// registry (runtime.hpp:141).  It lives in device memory; kernels receive a
// pointer to it.  Peer windows and peer signal tables are VMM mappings of the
// peers' physical allocations (cuMemCreate/cuMemMap), so a device put is a
// plain NVLink store.
#pragma once
#include <stdint.h>

#define GIN_MAX_RANKS 8
#define GIN_MAX_WINDOWS 64
#define GIN_MAX_CONTEXTS 16
#define GIN_MAX_TEAMS 16
// proj/core/include/ginsim/runtime.hpp:62-63: top 8 slots x 8 steps of the
// signal table are reserved for BarrierSession.
#define GIN_BARRIER_SLOTS 8
#define GIN_BARRIER_STEPS 8
// NVLS region (one multicast granule): words [0, 8) = barrier slots,
// [GIN_BCAST_BASE, GIN_BCAST_BASE + GIN_BCAST_CELLS) = broadcast signal cells.
#define GIN_BCAST_BASE 64
#define GIN_BCAST_CELLS 256

// proj/core/include/ginsim/descriptor.hpp:34-45
#define GIN_OP_PUT 0x01
#define GIN_OP_PUT_INLINE 0x02
#define GIN_OP_SIGNAL_ONLY 0x03
#define GIN_FLAG_HAS_SIGNAL 0x01
#define GIN_FLAG_SIGNAL_IS_ADD 0x02
#define GIN_FLAG_HAS_COUNTER 0x04
#define GIN_INLINE_WINDOW 0xFFFFFFFFu

#define GIN_BACKEND_DIRECT 0
#define GIN_BACKEND_PROXY 1

// Device error codes written to DevCommView::error (first error wins).
#define GIN_DEVERR_NONE 0
#define GIN_DEVERR_TIMEOUT 19        // ginsim::Timeout
#define GIN_DEVERR_OUT_OF_BOUNDS 3   // ginsim::OutOfBounds
#define GIN_DEVERR_INVALID_PEER 15   // ginsim::InvalidPeer
#define GIN_DEVERR_RANK_OUT_OF_RANGE 5  // ginsim::RankOutOfRange (team_translate, types.cpp:14-20)
#define GIN_DEVERR_INVALID_SIGNAL 16
#define GIN_DEVERR_INVALID_COUNTER 17
#define GIN_DEVERR_UNKNOWN_WINDOW 4
#define GIN_DEVERR_INVALID_CONTEXT 11
#define GIN_DEVERR_FLOW_CONTROL 21
#define GIN_DEVERR_VERIFY 20

typedef struct GinWindowView {
  char* base[GIN_MAX_RANKS];      // every rank's region, mapped into this rank
  uint64_t size[GIN_MAX_RANKS];   // per-rank capacity (asymmetric allowed)
} GinWindowView;

// A registered team (proj/core/include/ginsim/types.hpp:75-84,
// runtime.cpp:329-343): team-relative rank i is world rank members[i].
// Slot 0 is the world team (id 0); n == 0 marks a free slot.
typedef struct GinTeamView {
  uint32_t id;
  uint32_t n;
  uint8_t members[GIN_MAX_RANKS];
} GinTeamView;

// One proxy descriptor ring per context (proj/core/include/ginsim/
// proxy_backend.hpp:23-53): slots live in pinned host memory mapped into the
// device; the ticket counter lives in device memory (GPU producers only).
typedef struct GinRingSlot {
  uint64_t seq;
  uint8_t bytes[64];
} GinRingSlot;  // 72-byte stride, as the reference's static_assert demands

typedef struct GinProxyView {
  GinRingSlot* slots[GIN_MAX_CONTEXTS];        // host-pinned, device-mapped
  unsigned long long* tickets;                 // device: [ctx] next ticket
  uint64_t* completed;                         // device: [ctx] tickets locally complete
  // host-pinned, written only by the agent: [ctx] tickets consumed.  Producers
  // wait on this (never on the slot's own seq word) before reusing a slot: a
  // slot line the GPU has itself written can be served stale from its L2 after
  // the CPU rewrites it, while a line the GPU only ever reads is re-fetched.
  const uint64_t* consumed;
  uint32_t mask;                               // capacity - 1
  uint32_t pad;
} GinProxyView;

typedef struct GinDevCommView {
  uint32_t rank, world, n_ctx, signal_cells, counter_cells, backend, n_windows, device;
  uint64_t timeout_ns;
  // signals of rank d: sub-cells [src][cell] written only by src, plus a
  // per-cell reset baseline owned by d.  value(cell) = sum_src sub - base.
  uint64_t* signals[GIN_MAX_RANKS];
  uint64_t* signal_base;     // local [cell]
  uint64_t* counters;        // local [cell]
  uint64_t* counter_base;    // local [cell]
  unsigned int* error;       // local device error word
  unsigned int* workspace;   // local scratch for kernels (zeroed at init), 64 KiB
  // NVLS barrier region (null when multicast is unavailable): the multicast
  // mapping (multimem.* reaches every rank's copy through the NVSwitch) and
  // this rank's own copy of the same cells.
  uint64_t* nvls_mc;
  uint64_t* nvls_uc;
  uint32_t same_gpu;              // bit r: rank r's memory is on this rank's GPU (emulated ranks): GPU-scope
                                  // fences order this rank's writes for its observers, no .sys needed
  uint32_t pad0;
  uint64_t win_live;              // bit w: window id w is registered (ids are reused after deregister)
  GinWindowView win[GIN_MAX_WINDOWS];
  GinTeamView teams[GIN_MAX_TEAMS];
  GinProxyView proxy;
} GinDevCommView;
