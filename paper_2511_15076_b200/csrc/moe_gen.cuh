// moe_gen.cuh -- on-device generators of the reference workload (harness_moe.cpp:25-42).
// A fragment of kernels_moe.cu's single translation unit (included once, in order).
#pragma once

namespace ginsim_b200 {

// ------------------------------------------------------------------ synthetic inputs
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// route_token (harness_moe.cpp:25-30): std::mt19937_64 seeded with
// mix64(seed ^ mix64(src*100003 + token)), draws % E until K distinct, sorted.
__global__ void moe_route_kernel(int32_t* idx, uint64_t seed, uint32_t src, uint32_t T, uint32_t E, uint32_t K) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  uint64_t mt[312];
  mt[0] = mix64(seed ^ mix64((uint64_t)src * 100003ull + t));
  for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + (uint64_t)i;
  int pos = 312;
  int32_t picked[32];
  uint32_t got = 0;
  while (got < K) {
    if (pos >= 312) {
      for (int i = 0; i < 312; ++i) {
        const uint64_t y = (mt[i] & 0xFFFFFFFF80000000ull) | (mt[(i + 1) % 312] & 0x7FFFFFFFull);
        uint64_t nv = mt[(i + 156) % 312] ^ (y >> 1);
        if (y & 1) nv ^= 0xB5026F5AA96619E9ull;
        mt[i] = nv;
      }
      pos = 0;
    }
    uint64_t x = mt[pos++];
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    const int32_t e = (int32_t)(x % E);
    uint32_t p = 0;
    while (p < got && picked[p] < e) ++p;
    if (p < got && picked[p] == e) continue;
    for (uint32_t j = got; j > p; --j) picked[j] = picked[j - 1];
    picked[p] = e;
    ++got;
  }
  for (uint32_t k = 0; k < K; ++k) idx[(uint64_t)t * K + k] = picked[k];
}

// token_element (harness_moe.cpp:32-34) or the bf16 generator.
__global__ void moe_tokens_kernel(uint16_t* x, uint64_t seed, uint32_t src, uint32_t T, uint32_t H, uint32_t mode) {
  const uint64_t total = (uint64_t)T * H;
  for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < total; j += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(j / H), i = (uint32_t)(j % H);
    if (mode == 0) {
      x[j] = (uint16_t)(seed + src * 7919u + t * 131u + i * 13u);
    } else {
      const uint64_t h = mix64(seed ^ mix64(((uint64_t)src << 40) ^ ((uint64_t)t << 20) ^ i));
      const uint16_t sign = (uint16_t)((h >> 63) << 15);
      const uint16_t expo = (uint16_t)(120u + (uint32_t)((h >> 8) % 12u));
      x[j] = (uint16_t)(sign | (expo << 7) | (uint16_t)(h & 0x7Fu));
    }
  }
}

// combine_weight (harness_moe.cpp:40-42); bf16 mode uses w/8 as fp32.
__global__ void moe_weights_kernel(void* w, uint32_t src, uint32_t T, uint32_t K, uint32_t mode) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T * K) return;
  const uint32_t t = j / K, k = j % K;
  const uint16_t cw = (uint16_t)(1u + (src + 3u * t + 5u * k) % 7u);
  if (mode == 0) reinterpret_cast<uint16_t*>(w)[j] = cw;
  else reinterpret_cast<float*>(w)[j] = (float)cw / 8.0f;
}

}  // namespace ginsim_b200
