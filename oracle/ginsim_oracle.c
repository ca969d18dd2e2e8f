/*
 * ginsim_oracle.c — CPU ORACLE (test infrastructure only).
 *
 * Plain-C restatement of the reference's hot-path arithmetic, used ONLY by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as the
 * checker.  Nothing in paper_2511_15076_b200/ links, loads or calls this file.
 *
 * Parity status: PINNED.  Every function here is cross-checked against the
 * reference itself (oracle/_ref, compiled from /root/reference/proj/core/src by
 * oracle/build_ref.sh) through the golden fixtures in tests/golden/ that
 * oracle/make_golden.py generates from it.
 *
 * Citations are /root/reference-relative.
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------ */
/* proj/core/src/harness_moe.cpp:17-22 (mix64 = splitmix64 finaliser)        */
uint64_t gso_mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

/* std::mt19937_64 as fully specified by [rand.predef] (C++11 26.5.5):       */
/* w=64 n=312 m=156 r=31 a=0xB5026F5AA96619E9 u=29 d=0x5555555555555555       */
/* s=17 b=0x71D67FFFEDA60000 t=37 c=0xFFF7EEE000000000 l=43 f=6364136223846793005 */
typedef struct {
  uint64_t mt[312];
  int idx;
} gso_mt64;

void gso_mt64_seed(gso_mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i) {
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

uint64_t gso_mt64_next(gso_mt64* g) {
  if (g->idx >= 312) {
    const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    for (int i = 0; i < 312; ++i) {
      uint64_t y = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
      uint64_t v = g->mt[(i + 156) % 312] ^ (y >> 1);
      if (y & 1) v ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = v;
    }
    g->idx = 0;
  }
  uint64_t x = g->mt[g->idx++];
  x ^= (x >> 29) & 0x5555555555555555ull;
  x ^= (x << 17) & 0x71D67FFFEDA60000ull;
  x ^= (x << 37) & 0xFFF7EEE000000000ull;
  x ^= x >> 43;
  return x;
}

/* proj/core/src/harness_moe.cpp:25-30 (route_token): top_k distinct experts,
 * drawn as rng() % E into a std::set, returned ascending. */
void gso_route_token(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t src,
                     uint32_t token, uint32_t* out) {
  gso_mt64 g;
  gso_mt64_seed(&g, gso_mix64(seed ^ gso_mix64((uint64_t)src * 100003ull + token)));
  uint32_t n = 0;
  while (n < top_k) {
    uint32_t e = (uint32_t)(gso_mt64_next(&g) % experts);
    uint32_t pos = 0;
    while (pos < n && out[pos] < e) ++pos;
    if (pos < n && out[pos] == e) continue;
    for (uint32_t j = n; j > pos; --j) out[j] = out[j - 1];
    out[pos] = e;
    ++n;
  }
}

/* Routing table for every token of one source rank: out[t*top_k + k]. */
void gso_route_table(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t src,
                     uint32_t tokens, uint32_t* out) {
  for (uint32_t t = 0; t < tokens; ++t) gso_route_token(seed, experts, top_k, src, t, out + (size_t)t * top_k);
}

/* proj/core/src/harness_moe.cpp:32-34 */
uint16_t gso_token_element(uint64_t seed, uint32_t src, uint32_t token, uint32_t i) {
  return (uint16_t)(seed + src * 7919u + token * 131u + i * 13u);
}
/* proj/core/src/harness_moe.cpp:36-38 */
uint16_t gso_expert_transform(uint16_t in, uint32_t expert) {
  return (uint16_t)(in * 3u + expert * 17u + 1u);
}
/* proj/core/src/harness_moe.cpp:40-42 */
uint16_t gso_combine_weight(uint32_t src, uint32_t token, uint32_t k) {
  return (uint16_t)(1u + (src + 3u * token + 5u * k) % 7u);
}

/* proj/core/src/harness_moe.cpp:46-57 (oracle_combine) */
void gso_oracle_combine(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden,
                        uint32_t src, uint32_t token, uint16_t* out) {
  uint32_t ex[256];
  gso_route_token(seed, experts, top_k, src, token, ex);
  for (uint32_t i = 0; i < hidden; ++i) out[i] = 0;
  for (uint32_t k = 0; k < top_k; ++k) {
    uint16_t w = gso_combine_weight(src, token, k);
    for (uint32_t i = 0; i < hidden; ++i) {
      uint16_t y = gso_expert_transform(gso_token_element(seed, src, token, i), ex[k]);
      out[i] = (uint16_t)(out[i] + w * y);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* moe-ll final state (proj/core/src/harness_moe.cpp:105-250).
 * Fills, for rank r of an n-rank run, exactly what moe_ll_rank_program
 * snapshots (:244-249): dispatch_recv (window 0, worst-case layout
 * ((e_loc*n+src)*T+slot)*dmsg, :122,:135-137), combine_recv (window 2,
 * (token*K+k)*cmsg, :203-205) and the signal cells (per-expert
 * (n<<32)+count, :163-167; combine flag e_local = T*K, :217-223).
 * Buffers must be zero-initialised by the caller with sizes
 *   dispatch: e_local*n*T*(2*hidden+16), combine: T*K*2*hidden, cells: n_cells u64. */
static void st16(uint8_t* p, uint16_t v) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); }
static void st32(uint8_t* p, uint32_t v) { for (int i = 0; i < 4; ++i) p[i] = (uint8_t)(v >> (8 * i)); }

int gso_moe_ll_rank_state(uint64_t seed, uint32_t n, uint32_t experts, uint32_t top_k,
                          uint32_t T, uint32_t hidden, uint32_t r, uint8_t* dispatch_recv,
                          uint8_t* combine_recv, uint64_t* cells, uint32_t n_cells) {
  if (n == 0 || experts % n || top_k > 256 || top_k > experts) return -1;
  const uint32_t e_local = experts / n;
  if (e_local + 1 > n_cells) return -2;
  const uint64_t dmsg = 2ull * hidden + 16, cmsg = 2ull * hidden;
  uint32_t* route = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T * top_k);
  uint32_t* sent = (uint32_t*)calloc(experts, sizeof(uint32_t));
  /* dispatch: every source's messages to the experts this rank owns */
  for (uint32_t src = 0; src < n; ++src) {
    memset(sent, 0, sizeof(uint32_t) * experts);
    gso_route_table(seed, experts, top_k, src, T, route);
    for (uint32_t t = 0; t < T; ++t) {
      for (uint32_t k = 0; k < top_k; ++k) {
        const uint32_t e = route[(size_t)t * top_k + k];
        const uint32_t slot = sent[e]++;
        if (e / e_local != r) continue;
        const uint32_t e_loc = e % e_local;
        uint8_t* msg = dispatch_recv + (((uint64_t)e_loc * n + src) * T + slot) * dmsg;
        for (uint32_t i = 0; i < hidden; ++i) st16(msg + 2ull * i, gso_token_element(seed, src, t, i));
        st32(msg + 2ull * hidden + 0, src);
        st32(msg + 2ull * hidden + 4, t);
        st32(msg + 2ull * hidden + 8, k);
        st32(msg + 2ull * hidden + 12, k + 1);
      }
    }
    for (uint32_t e = r * e_local; e < (r + 1) * e_local; ++e) {
      cells[e % e_local] += (1ull << 32) + sent[e];
    }
  }
  /* combine: this rank's own tokens come back transformed by their experts */
  gso_route_table(seed, experts, top_k, r, T, route);
  for (uint32_t t = 0; t < T; ++t) {
    for (uint32_t k = 0; k < top_k; ++k) {
      const uint32_t e = route[(size_t)t * top_k + k];
      uint8_t* out = combine_recv + ((uint64_t)t * top_k + k) * cmsg;
      for (uint32_t i = 0; i < hidden; ++i) {
        st16(out + 2ull * i, gso_expert_transform(gso_token_element(seed, r, t, i), e));
      }
    }
  }
  cells[e_local] += (uint64_t)T * top_k;
  free(route);
  free(sent);
  return 0;
}

/* Per-(expert, source) message counts as seen by the owner: cnt[e*n + src]. */
void gso_moe_counts(uint64_t seed, uint32_t n, uint32_t experts, uint32_t top_k, uint32_t T,
                    uint32_t* cnt) {
  uint32_t* route = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T * top_k);
  memset(cnt, 0, sizeof(uint32_t) * (size_t)experts * n);
  for (uint32_t src = 0; src < n; ++src) {
    gso_route_table(seed, experts, top_k, src, T, route);
    for (size_t j = 0; j < (size_t)T * top_k; ++j) cnt[(size_t)route[j] * n + src]++;
  }
  free(route);
}

/* ------------------------------------------------------------------------ */
/* bf16 mode (outside the reference; parity unpinned by it).
 * All fp32 arithmetic below is single rounded per operation (compiled with
 * -ffp-contract=off); the device code uses __fmul_rn/__fadd_rn in the same
 * order, so results are bit-identical, and within 1 bf16 ulp of an fp64 sum. */
static uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7F800000u) == 0x7F800000u) return (uint16_t)((u >> 16) | ((u & 0xFFFF) ? 0x40 : 0));
  u += 0x7FFFu + ((u >> 16) & 1u);
  return (uint16_t)(u >> 16);
}
static float bf2f(uint16_t b) {
  uint32_t u = (uint32_t)b << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}
uint16_t gso_bf16_round(float f) { return f2bf(f); }
float gso_bf16_to_float(uint16_t b) { return bf2f(b); }

/* token value: sign/exponent/mantissa drawn from mix64 so every mantissa bit
 * is exercised; exponent in [120,131] keeps |x| in [2^-7, 2^5). */
uint16_t gso_bf16_token(uint64_t seed, uint32_t src, uint32_t token, uint32_t i) {
  uint64_t h = gso_mix64(seed ^ gso_mix64(((uint64_t)src << 40) ^ ((uint64_t)token << 20) ^ i));
  uint16_t sign = (uint16_t)((h >> 63) << 15);
  uint16_t expo = (uint16_t)(120u + (uint32_t)((h >> 8) % 12u));
  uint16_t mant = (uint16_t)(h & 0x7Fu);
  return (uint16_t)(sign | (expo << 7) | mant);
}
/* y = bf16(fp32(x) * s_e + c_e), s_e = 1 + (e%7)/8, c_e = ((e%9)-4)/16 */
uint16_t gso_bf16_transform(uint16_t x, uint32_t expert) {
  volatile float s = 1.0f + (float)(expert % 7u) / 8.0f;
  volatile float c = ((float)(expert % 9u) - 4.0f) / 16.0f;
  volatile float p = bf2f(x) * s;
  volatile float q = p + c;
  return f2bf(q);
}
float gso_bf16_weight(uint32_t src, uint32_t token, uint32_t k) {
  return (float)gso_combine_weight(src, token, k) / 8.0f;
}
/* out[i] = bf16( sum_k w_k * y_k[i] ) with fp32 accumulation in k order. */
void gso_bf16_combine(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden,
                      uint32_t src, uint32_t token, uint16_t* out, double* out_f64) {
  uint32_t ex[256];
  gso_route_token(seed, experts, top_k, src, token, ex);
  for (uint32_t i = 0; i < hidden; ++i) {
    volatile float acc = 0.0f;
    double acc64 = 0.0;
    uint16_t x = gso_bf16_token(seed, src, token, i);
    for (uint32_t k = 0; k < top_k; ++k) {
      float w = gso_bf16_weight(src, token, k);
      float y = bf2f(gso_bf16_transform(x, ex[k]));
      volatile float prod = w * y;
      acc = acc + prod;
      acc64 += (double)w * (double)y;
    }
    out[i] = f2bf(acc);
    if (out_f64) out_f64[i] = acc64;
  }
}

/* ------------------------------------------------------------------------ */
/* 64-byte descriptor codec (proj/core/include/ginsim/descriptor.hpp:13-27,
 * proj/core/src/descriptor.cpp:32-199).  Returns 0 when valid, else a
 * nonzero reason code (the reference's reason strings are not part of the
 * wire contract). */
typedef struct {
  uint8_t opcode, flags;
  uint16_t team;
  uint32_t peer, dst_window, src_window;
  uint64_t dst_offset, src_offset_or_value, bytes;
  uint32_t signal_id, counter_id;
  uint64_t signal_operand;
} gso_descriptor;

enum { GSO_HAS_SIGNAL = 1, GSO_SIGNAL_IS_ADD = 2, GSO_HAS_COUNTER = 4 };

int gso_descriptor_check(const gso_descriptor* d) {
  const int is_inline = d->src_window == 0xFFFFFFFFu;
  switch (d->opcode) {
    case 1:
      if (is_inline) return 1;
      break;
    case 2:
      if (!is_inline) return 2;
      if (d->bytes > 8) return 3;
      break;
    case 3:
      if (d->bytes != 0) return 4;
      if (!(d->flags & GSO_HAS_SIGNAL)) return 5;
      if (!is_inline) return 6;
      if (d->dst_window || d->dst_offset || d->src_offset_or_value) return 7;
      break;
    default:
      return 8;
  }
  if (d->flags & ~7u) return 9;
  if (d->flags & GSO_HAS_SIGNAL) {
    if (!(d->flags & GSO_SIGNAL_IS_ADD) && d->signal_operand != 1) return 10;
  } else {
    if (d->flags & GSO_SIGNAL_IS_ADD) return 11;
    if (d->signal_id || d->signal_operand) return 12;
  }
  if (!(d->flags & GSO_HAS_COUNTER) && d->counter_id) return 13;
  return 0;
}

static void stle(uint8_t* b, int off, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) b[off + i] = (uint8_t)(v >> (8 * i));
}
static uint64_t ldle(const uint8_t* b, int off, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= (uint64_t)b[off + i] << (8 * i);
  return v;
}

int gso_descriptor_encode(const gso_descriptor* d, uint8_t* out64) {
  int why = gso_descriptor_check(d);
  if (why) return why;
  memset(out64, 0, 64);
  stle(out64, 0, d->opcode, 1);
  stle(out64, 1, d->flags, 1);
  stle(out64, 2, d->team, 2);
  stle(out64, 4, d->peer, 4);
  stle(out64, 8, d->dst_window, 4);
  stle(out64, 12, d->src_window, 4);
  stle(out64, 16, d->dst_offset, 8);
  stle(out64, 24, d->src_offset_or_value, 8);
  stle(out64, 32, d->bytes, 8);
  stle(out64, 40, d->signal_id, 4);
  stle(out64, 44, d->counter_id, 4);
  stle(out64, 48, d->signal_operand, 8);
  return 0;
}

int gso_descriptor_decode(const uint8_t* b, gso_descriptor* d) {
  uint8_t op = (uint8_t)ldle(b, 0, 1);
  if (op < 1 || op > 3) return 8;
  d->opcode = op;
  d->flags = (uint8_t)ldle(b, 1, 1);
  d->team = (uint16_t)ldle(b, 2, 2);
  d->peer = (uint32_t)ldle(b, 4, 4);
  d->dst_window = (uint32_t)ldle(b, 8, 4);
  d->src_window = (uint32_t)ldle(b, 12, 4);
  d->dst_offset = ldle(b, 16, 8);
  d->src_offset_or_value = ldle(b, 24, 8);
  d->bytes = ldle(b, 32, 8);
  d->signal_id = (uint32_t)ldle(b, 40, 4);
  d->counter_id = (uint32_t)ldle(b, 44, 4);
  d->signal_operand = ldle(b, 48, 8);
  if (ldle(b, 56, 8) != 0) return 14;
  return gso_descriptor_check(d);
}

/* ------------------------------------------------------------------------ */
/* ping-pong payload (proj/core/src/harness_bench.cpp:63) */
uint8_t gso_pingpong_byte(uint32_t rank, uint64_t i) { return (uint8_t)(i * 31u + rank); }
/* ring payload (proj/core/src/harness_ring.cpp:12-14) */
uint8_t gso_ring_byte(uint32_t sender, uint32_t round, uint64_t i) {
  return (uint8_t)(sender * 131u + round * 31u + i * 7u + 1u);
}
/* moe-ht slot payload (proj/core/src/harness_moe.cpp:263-268) */
uint8_t gso_ht_byte(uint32_t channel, uint32_t msg, uint64_t i, uint64_t seed) {
  return (uint8_t)(seed + channel * 37u + msg * 11u + i);
}

/* moe-ht final receive planes (proj/core/src/harness_moe.cpp:283-382): for a
 * rank, plane c (= channel / n_ctx) receive window of n_ctx*B*256 bytes holds,
 * in lane ctx = channel % n_ctx, slot m%B, the LAST message m written there by
 * the predecessor: 8-byte LE generation m+1 then ht_byte(channel, m, i). The
 * payload is rank-independent, so every rank's planes are identical. */
void gso_moe_ht_plane(uint64_t seed, uint32_t channels, uint32_t n_ctx, uint32_t slots,
                      uint32_t messages, uint32_t plane, uint8_t* recv) {
  memset(recv, 0, (size_t)n_ctx * slots * 256);
  for (uint32_t ctx = 0; ctx < n_ctx; ++ctx) {
    uint32_t channel = plane * n_ctx + ctx;
    if (channel >= channels) break;
    for (uint32_t m = 0; m < messages; ++m) {
      uint8_t* slot = recv + ((size_t)ctx * slots + m % slots) * 256;
      uint64_t gen = (uint64_t)m + 1;
      for (int i = 0; i < 8; ++i) slot[i] = (uint8_t)(gen >> (8 * i));
      for (uint64_t i = 0; i < 248; ++i) slot[8 + i] = gso_ht_byte(channel, m, i, seed);
    }
  }
}

/* ------------------------------------------------------------------------ */
/* Bulk helpers for the Python test harness (same arithmetic as above). */
void gso_tokens_u16(uint64_t seed, uint32_t src, uint32_t T, uint32_t H, uint16_t* out) {
  for (uint32_t t = 0; t < T; ++t)
    for (uint32_t i = 0; i < H; ++i) out[(size_t)t * H + i] = gso_token_element(seed, src, t, i);
}
void gso_tokens_bf16(uint64_t seed, uint32_t src, uint32_t T, uint32_t H, uint16_t* out) {
  for (uint32_t t = 0; t < T; ++t)
    for (uint32_t i = 0; i < H; ++i) out[(size_t)t * H + i] = gso_bf16_token(seed, src, t, i);
}
void gso_weights(uint32_t src, uint32_t T, uint32_t K, int bf16, void* out) {
  for (uint32_t t = 0; t < T; ++t)
    for (uint32_t k = 0; k < K; ++k) {
      if (bf16) ((float*)out)[(size_t)t * K + k] = gso_bf16_weight(src, t, k);
      else ((uint16_t*)out)[(size_t)t * K + k] = gso_combine_weight(src, t, k);
    }
}
void gso_oracle_combine_all(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden, uint32_t src,
                            uint32_t T, uint16_t* out) {
  for (uint32_t t = 0; t < T; ++t) gso_oracle_combine(seed, experts, top_k, hidden, src, t, out + (size_t)t * hidden);
}
void gso_bf16_combine_all(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden, uint32_t src,
                          uint32_t T, uint16_t* out, double* out_f64) {
  for (uint32_t t = 0; t < T; ++t)
    gso_bf16_combine(seed, experts, top_k, hidden, src, t, out + (size_t)t * hidden,
                     out_f64 ? out_f64 + (size_t)t * hidden : 0);
}
/* bf16-mode dispatch payload / combine rows follow the same layout as
 * gso_moe_ll_rank_state with the bf16 generator and transform. */
int gso_moe_bf16_rank_state(uint64_t seed, uint32_t n, uint32_t experts, uint32_t top_k, uint32_t T,
                            uint32_t hidden, uint32_t r, uint8_t* dispatch_recv, uint8_t* combine_recv) {
  if (n == 0 || experts % n || top_k > 256 || top_k > experts) return -1;
  const uint32_t e_local = experts / n;
  const uint64_t dmsg = 2ull * hidden + 16, cmsg = 2ull * hidden;
  uint32_t* route = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T * top_k);
  uint32_t* sent = (uint32_t*)calloc(experts, sizeof(uint32_t));
  for (uint32_t src = 0; src < n; ++src) {
    memset(sent, 0, sizeof(uint32_t) * experts);
    gso_route_table(seed, experts, top_k, src, T, route);
    for (uint32_t t = 0; t < T; ++t)
      for (uint32_t k = 0; k < top_k; ++k) {
        const uint32_t e = route[(size_t)t * top_k + k];
        const uint32_t slot = sent[e]++;
        if (e / e_local != r) continue;
        uint8_t* msg = dispatch_recv + (((uint64_t)(e % e_local) * n + src) * T + slot) * dmsg;
        for (uint32_t i = 0; i < hidden; ++i) st16(msg + 2ull * i, gso_bf16_token(seed, src, t, i));
        st32(msg + 2ull * hidden + 0, src);
        st32(msg + 2ull * hidden + 4, t);
        st32(msg + 2ull * hidden + 8, k);
        st32(msg + 2ull * hidden + 12, k + 1);
      }
  }
  gso_route_table(seed, experts, top_k, r, T, route);
  for (uint32_t t = 0; t < T; ++t)
    for (uint32_t k = 0; k < top_k; ++k) {
      const uint32_t e = route[(size_t)t * top_k + k];
      uint8_t* out = combine_recv + ((uint64_t)t * top_k + k) * cmsg;
      for (uint32_t i = 0; i < hidden; ++i) st16(out + 2ull * i, gso_bf16_transform(gso_bf16_token(seed, r, t, i), e));
    }
  free(route);
  free(sent);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* fp8 mode (mode 2; a labelled variant outside the reference, SURVEY.md §8f
 * f3, the paper's LL dispatch format PAPER.md:878-896): each 128-element
 * block of a bf16 token row is sent as e4m3 codes plus one fp32 scale.
 *   amax  = max |x_i| over the block (exact)
 *   scale = amax / 448,  inv = 448 / amax   (fp32, single rounded; 1 if amax = 0)
 *   q_i   = e4m3(x_i * inv)  round-to-nearest-even, saturating at +-448
 *   deq_i = float(q_i) * scale
 * The expert transform then runs on deq (y = bf16(deq * s_e + c_e)); the
 * combine is the bf16 one.  Message = [q: H bytes][scales: H/128 x f32][meta]. */
static float e4m3_value(uint8_t c) {  /* positive codes 0x00..0x7E */
  const uint32_t e = (c >> 3) & 0xF, m = c & 7;
  if (e == 0) return (float)m / 512.0f;                 /* subnormal: m * 2^-9 */
  return ldexpf(1.0f + (float)m / 8.0f, (int)e - 7);
}
uint8_t gso_fp8_e4m3(float v) {
  const uint8_t sign = (v < 0.0f || (v == 0.0f && signbit(v))) ? 0x80 : 0x00;
  float a = fabsf(v);
  if (a >= 448.0f) return (uint8_t)(sign | 0x7E);       /* satfinite */
  uint8_t lo = 0, hi = 0x7E;                             /* largest code with value <= a */
  while (lo < hi) {
    const uint8_t mid = (uint8_t)((lo + hi + 1) / 2);
    if (e4m3_value(mid) <= a) lo = mid; else hi = (uint8_t)(mid - 1);
  }
  uint8_t c = lo;
  if (e4m3_value(c) != a) {
    const float below = e4m3_value(c), above = e4m3_value((uint8_t)(c + 1));
    const double db = (double)a - below, da = (double)above - a;
    if (da < db || (da == db && ((c + 1) & 1) == 0)) c = (uint8_t)(c + 1);
  }
  return (uint8_t)(sign | c);
}
float gso_fp8_to_float(uint8_t c) {
  const float v = e4m3_value((uint8_t)(c & 0x7F));
  return (c & 0x80) ? -v : v;
}
/* one token row: q [H], scales [H/128] */
void gso_fp8_quant_row(uint64_t seed, uint32_t src, uint32_t token, uint32_t hidden, uint8_t* q, float* scales) {
  for (uint32_t b = 0; b < hidden / 128; ++b) {
    float amax = 0.0f;
    for (uint32_t i = 0; i < 128; ++i) {
      const float x = fabsf(bf2f(gso_bf16_token(seed, src, token, b * 128 + i)));
      if (x > amax) amax = x;
    }
    volatile float scale = amax > 0.0f ? amax / 448.0f : 1.0f;
    volatile float inv = amax > 0.0f ? 448.0f / amax : 1.0f;
    scales[b] = scale;
    for (uint32_t i = 0; i < 128; ++i) {
      volatile float p = bf2f(gso_bf16_token(seed, src, token, b * 128 + i)) * inv;
      q[b * 128 + i] = gso_fp8_e4m3(p);
    }
  }
}
/* expert transform of the dequantized value */
uint16_t gso_fp8_transform(uint8_t q, float scale, uint32_t expert) {
  volatile float s = 1.0f + (float)(expert % 7u) / 8.0f;
  volatile float c = ((float)(expert % 9u) - 4.0f) / 16.0f;
  volatile float deq = gso_fp8_to_float(q) * scale;
  volatile float p = deq * s;
  volatile float r = p + c;
  return f2bf(r);
}
/* out[t][i] = bf16(sum_k w_k * y_k[i]) over the dequantized transform, fp32 in k order */
void gso_fp8_combine_all(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden, uint32_t src, uint32_t T,
                         uint16_t* out) {
  uint32_t ex[256];
  uint8_t* q = (uint8_t*)malloc(hidden);
  float* sc = (float*)malloc(sizeof(float) * (hidden / 128));
  for (uint32_t t = 0; t < T; ++t) {
    gso_route_token(seed, experts, top_k, src, t, ex);
    gso_fp8_quant_row(seed, src, t, hidden, q, sc);
    for (uint32_t i = 0; i < hidden; ++i) {
      volatile float acc = 0.0f;
      for (uint32_t k = 0; k < top_k; ++k) {
        const float w = gso_bf16_weight(src, t, k);
        const float y = bf2f(gso_fp8_transform(q[i], sc[i / 128], ex[k]));
        volatile float prod = w * y;
        acc = acc + prod;
      }
      out[(size_t)t * hidden + i] = f2bf(acc);
    }
  }
  free(q);
  free(sc);
}
/* fp8-mode final state, reference layout: dmsg = H + H/32 + 16, cmsg = 2H */
int gso_moe_fp8_rank_state(uint64_t seed, uint32_t n, uint32_t experts, uint32_t top_k, uint32_t T,
                           uint32_t hidden, uint32_t r, uint8_t* dispatch_recv, uint8_t* combine_recv) {
  if (n == 0 || experts % n || top_k > 256 || top_k > experts || hidden % 128) return -1;
  const uint32_t e_local = experts / n;
  const uint64_t pay = (uint64_t)hidden + hidden / 32, dmsg = pay + 16, cmsg = 2ull * hidden;
  uint32_t* route = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T * top_k);
  uint32_t* sent = (uint32_t*)calloc(experts, sizeof(uint32_t));
  uint8_t* q = (uint8_t*)malloc(hidden);
  float* sc = (float*)malloc(sizeof(float) * (hidden / 128));
  for (uint32_t src = 0; src < n; ++src) {
    memset(sent, 0, sizeof(uint32_t) * experts);
    gso_route_table(seed, experts, top_k, src, T, route);
    for (uint32_t t = 0; t < T; ++t) {
      int quantized = 0;
      for (uint32_t k = 0; k < top_k; ++k) {
        const uint32_t e = route[(size_t)t * top_k + k];
        const uint32_t slot = sent[e]++;
        if (e / e_local != r) continue;
        if (!quantized) {
          gso_fp8_quant_row(seed, src, t, hidden, q, sc);
          quantized = 1;
        }
        uint8_t* msg = dispatch_recv + (((uint64_t)(e % e_local) * n + src) * T + slot) * dmsg;
        memcpy(msg, q, hidden);
        for (uint32_t b = 0; b < hidden / 128; ++b) {
          uint32_t u;
          memcpy(&u, &sc[b], 4);
          st32(msg + hidden + 4ull * b, u);
        }
        st32(msg + pay + 0, src);
        st32(msg + pay + 4, t);
        st32(msg + pay + 8, k);
        st32(msg + pay + 12, k + 1);
      }
    }
  }
  gso_route_table(seed, experts, top_k, r, T, route);
  for (uint32_t t = 0; t < T; ++t) {
    gso_fp8_quant_row(seed, r, t, hidden, q, sc);
    for (uint32_t k = 0; k < top_k; ++k) {
      const uint32_t e = route[(size_t)t * top_k + k];
      uint8_t* out = combine_recv + ((uint64_t)t * top_k + k) * cmsg;
      for (uint32_t i = 0; i < hidden; ++i) st16(out + 2ull * i, gso_fp8_transform(q[i], sc[i / 128], e));
    }
  }
  free(route);
  free(sent);
  free(q);
  free(sc);
  return 0;
}

/* fp8 combine (mode 3 = mode 2 dispatch + fp8 combine messages): each expert
 * output row y (bf16, the mode-2 transform) is quantized like the dispatch
 * rows -- [e4m3: H bytes][scales: H/128 f32] per (t, k) -- and the source
 * reduces out = bf16(sum_k w_k * (fp32(q_k) * scale_k)), fp32 in k order. */
void gso_fp8_quant_bf16(const uint16_t* row, uint32_t hidden, uint8_t* q, float* scales) {
  for (uint32_t b = 0; b < hidden / 128; ++b) {
    float amax = 0.0f;
    for (uint32_t i = 0; i < 128; ++i) {
      const float x = fabsf(bf2f(row[b * 128 + i]));
      if (x > amax) amax = x;
    }
    volatile float scale = amax > 0.0f ? amax / 448.0f : 1.0f;
    volatile float inv = amax > 0.0f ? 448.0f / amax : 1.0f;
    scales[b] = scale;
    for (uint32_t i = 0; i < 128; ++i) {
      volatile float p = bf2f(row[b * 128 + i]) * inv;
      q[b * 128 + i] = gso_fp8_e4m3(p);
    }
  }
}
/* the combine message of (src token t, expert e): y quantized */
static void fp8c_message(uint64_t seed, uint32_t src, uint32_t t, uint32_t hidden, uint32_t e, const uint8_t* xq,
                         const float* xs, uint16_t* y, uint8_t* q, float* sc) {
  for (uint32_t i = 0; i < hidden; ++i) y[i] = gso_fp8_transform(xq[i], xs[i / 128], e);
  gso_fp8_quant_bf16(y, hidden, q, sc);
  (void)seed;
  (void)src;
  (void)t;
}
void gso_fp8c_combine_all(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden, uint32_t src, uint32_t T,
                          uint16_t* out) {
  uint32_t ex[256];
  uint8_t* xq = (uint8_t*)malloc(hidden);
  float* xs = (float*)malloc(sizeof(float) * (hidden / 128));
  uint16_t* y = (uint16_t*)malloc(2ull * hidden);
  uint8_t* q = (uint8_t*)malloc((size_t)top_k * hidden);
  float* sc = (float*)malloc(sizeof(float) * top_k * (hidden / 128));
  for (uint32_t t = 0; t < T; ++t) {
    gso_route_token(seed, experts, top_k, src, t, ex);
    gso_fp8_quant_row(seed, src, t, hidden, xq, xs);
    for (uint32_t k = 0; k < top_k; ++k)
      fp8c_message(seed, src, t, hidden, ex[k], xq, xs, y, q + (size_t)k * hidden, sc + (size_t)k * (hidden / 128));
    for (uint32_t i = 0; i < hidden; ++i) {
      volatile float acc = 0.0f;
      for (uint32_t k = 0; k < top_k; ++k) {
        const float w = gso_bf16_weight(src, t, k);
        volatile float deq = gso_fp8_to_float(q[(size_t)k * hidden + i]) * sc[(size_t)k * (hidden / 128) + i / 128];
        volatile float prod = w * deq;
        acc = acc + prod;
      }
      out[(size_t)t * hidden + i] = f2bf(acc);
    }
  }
  free(xq);
  free(xs);
  free(y);
  free(q);
  free(sc);
}
/* mode-3 combine window of rank r: (t*K+k) * (H + H/32) */
void gso_fp8c_combine_window(uint64_t seed, uint32_t experts, uint32_t top_k, uint32_t hidden, uint32_t r, uint32_t T,
                             uint8_t* combine_recv) {
  uint32_t ex[256];
  const uint64_t cm = (uint64_t)hidden + hidden / 32;
  uint8_t* xq = (uint8_t*)malloc(hidden);
  float* xs = (float*)malloc(sizeof(float) * (hidden / 128));
  uint16_t* y = (uint16_t*)malloc(2ull * hidden);
  uint8_t* q = (uint8_t*)malloc(hidden);
  float* sc = (float*)malloc(sizeof(float) * (hidden / 128));
  for (uint32_t t = 0; t < T; ++t) {
    gso_route_token(seed, experts, top_k, r, t, ex);
    gso_fp8_quant_row(seed, r, t, hidden, xq, xs);
    for (uint32_t k = 0; k < top_k; ++k) {
      fp8c_message(seed, r, t, hidden, ex[k], xq, xs, y, q, sc);
      uint8_t* m = combine_recv + ((uint64_t)t * top_k + k) * cm;
      memcpy(m, q, hidden);
      for (uint32_t b = 0; b < hidden / 128; ++b) {
        uint32_t u;
        memcpy(&u, &sc[b], 4);
        st32(m + hidden + 4ull * b, u);
      }
    }
  }
  free(xq);
  free(xs);
  free(y);
  free(q);
  free(sc);
}

/* ------------------------------------------------------------------------ */
/* Record digests for the large-shape checks (bench self-check, the 8-rank
 * T=4096 GPU test).  Same definition as the device utility
 * (paper_2511_15076_b200/csrc/verify.cu, include/ginsim_cuda.h
 * ginsim_cuda_digest):  digest = sum_i mix64(w_i + i*0xD1B54A32D192ED03)
 * over the record's little-endian u64 words, tail zero-padded. */
static uint64_t dg_word(uint64_t w, uint64_t i) { return gso_mix64(w + i * 0xD1B54A32D192ED03ull); }

uint64_t gso_digest(const uint8_t* p, uint64_t bytes) {
  uint64_t acc = 0, j = 0;
  for (; 8 * j + 8 <= bytes; ++j) {
    uint64_t w;
    memcpy(&w, p + 8 * j, 8);  /* little-endian host */
    acc += dg_word(w, j);
  }
  if (8 * j < bytes) {
    uint64_t w = 0;
    for (uint32_t b = 0; 8 * j + b < bytes; ++b) w |= (uint64_t)p[8 * j + b] << (8 * b);
    acc += dg_word(w, j);
  }
  return acc;
}

/* Digests of every record rank r holds after one moe-ll step
 * (proj/core/src/harness_moe.cpp:105-250), mode 0 (u16, the reference's
 * arithmetic) or 1 (bf16):
 *   disp[s], valid[s]: dispatch window slot s (layout 0: ((e_loc*n+src)*T+slot),
 *     harness_moe.cpp:135-137; layout 1: src*T*K + prefix(e_loc) + slot, the
 *     compact per-source layout); valid[s] = 1 where a message lands.  Slots:
 *     layout 0 e_local*n*T, layout 1 n*T*K.
 *   comb[t*K+k]: combine window record (token*K+k)*cmsg of rank r
 *     (harness_moe.cpp:203-205), the expert transform of r's own token.
 * Payload digests are computed once per token (its K messages share the row;
 * only the 16-byte meta differs) when 2*hidden is a multiple of 8. */
int gso_moe_window_digests(uint64_t seed, uint32_t n, uint32_t experts, uint32_t top_k, uint32_t T,
                           uint32_t hidden, uint32_t mode, uint32_t layout, uint32_t r, uint64_t* disp,
                           uint8_t* valid, uint64_t* comb) {
  if (n == 0 || experts % n || top_k > 256 || top_k > experts || mode > 1 || layout > 1) return -1;
  const uint32_t e_local = experts / n;
  const uint64_t dmsg = 2ull * hidden + 16, cmsg = 2ull * hidden;
  const uint64_t slots = layout == 0 ? (uint64_t)e_local * n * T : (uint64_t)n * T * top_k;
  const int split = (2ull * hidden) % 8 == 0;
  const uint64_t pw = 2ull * hidden / 8;  /* payload words when split */
  uint32_t* route = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)T * top_k);
  uint32_t* sent = (uint32_t*)calloc(e_local, sizeof(uint32_t));
  uint32_t* pre = (uint32_t*)calloc(e_local + 1, sizeof(uint32_t));
  uint16_t* row = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)hidden + 16);
  uint8_t* msg = (uint8_t*)malloc(dmsg);
  memset(valid, 0, slots);
  memset(disp, 0, slots * sizeof(uint64_t));
  for (uint32_t src = 0; src < n; ++src) {
    gso_route_table(seed, experts, top_k, src, T, route);
    memset(sent, 0, sizeof(uint32_t) * e_local);
    for (size_t j = 0; j < (size_t)T * top_k; ++j)
      if (route[j] / e_local == r) sent[route[j] % e_local]++;
    pre[0] = 0;
    for (uint32_t e = 0; e < e_local; ++e) pre[e + 1] = pre[e] + sent[e];
    memset(sent, 0, sizeof(uint32_t) * e_local);
    for (uint32_t t = 0; t < T; ++t) {
      const uint32_t* ex = route + (size_t)t * top_k;
      int mine = 0;
      for (uint32_t k = 0; k < top_k; ++k) mine |= ex[k] / e_local == r;
      if (!mine) continue;
      for (uint32_t i = 0; i < hidden; ++i)
        row[i] = mode == 0 ? gso_token_element(seed, src, t, i) : gso_bf16_token(seed, src, t, i);
      uint64_t pd = 0;
      if (split)
        for (uint64_t j = 0; j < pw; ++j) {
          uint64_t w;
          memcpy(&w, (const uint8_t*)row + 8 * j, 8);
          pd += dg_word(w, j);
        }
      for (uint32_t k = 0; k < top_k; ++k) {
        const uint32_t e = ex[k];
        if (e / e_local != r) continue;
        const uint32_t e_loc = e % e_local, slot = sent[e_loc]++;
        const uint64_t s = layout == 0 ? ((uint64_t)e_loc * n + src) * T + slot
                                       : (uint64_t)src * T * top_k + pre[e_loc] + slot;
        uint64_t d;
        if (split) {
          d = pd + dg_word((uint64_t)src | ((uint64_t)t << 32), pw) + dg_word((uint64_t)k | ((uint64_t)(k + 1) << 32), pw + 1);
        } else {
          for (uint32_t i = 0; i < hidden; ++i) st16(msg + 2ull * i, row[i]);
          st32(msg + 2ull * hidden + 0, src);
          st32(msg + 2ull * hidden + 4, t);
          st32(msg + 2ull * hidden + 8, k);
          st32(msg + 2ull * hidden + 12, k + 1);
          d = gso_digest(msg, dmsg);
        }
        disp[s] = d;
        valid[s] = 1;
      }
    }
  }
  /* combine records: r's own tokens, transformed by the expert each went to */
  gso_route_table(seed, experts, top_k, r, T, route);
  for (uint32_t t = 0; t < T; ++t) {
    uint16_t* x = row;
    for (uint32_t i = 0; i < hidden; ++i)
      x[i] = mode == 0 ? gso_token_element(seed, r, t, i) : gso_bf16_token(seed, r, t, i);
    for (uint32_t k = 0; k < top_k; ++k) {
      const uint32_t e = route[(size_t)t * top_k + k];
      for (uint32_t i = 0; i < hidden; ++i)
        st16(msg + 2ull * i, mode == 0 ? gso_expert_transform(x[i], e) : gso_bf16_transform(x[i], e));
      comb[(size_t)t * top_k + k] = gso_digest(msg, cmsg);
    }
  }
  free(route);
  free(sent);
  free(pre);
  free(row);
  free(msg);
  return 0;
}
