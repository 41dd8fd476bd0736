// philox.cuh — counter-based Philox4x32-10 generator and the integer-exact
// uniform mappings used to build the BASELINE.json inputs on device.
//
// Element i of stream `sid` under key `seed` is philox(ctr = (lo(i), hi(i),
// lo(sid), hi(sid)), key = (lo(seed), hi(seed))).  Because the counter is the
// global element index, a rank that owns elements [o, o+n) of a stream
// generates exactly the slice a single GPU would (contiguous sharding,
// SURVEY.md §8(e)).  The uniform mappings are integer-exact, so the oracle's
// host twin (oracle/twofold_oracle.c) reproduces them bit-for-bit; the
// reference's LCG mapping (lcg.py:49-60) can round to 1.0 and is not used.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace tfb {

struct U4 { uint32_t x, y, z, w; };

__host__ __device__ __forceinline__ void mulhilo32(uint32_t a, uint32_t b, uint32_t& hi, uint32_t& lo) {
  uint64_t p = static_cast<uint64_t>(a) * static_cast<uint64_t>(b);
  hi = static_cast<uint32_t>(p >> 32);
  lo = static_cast<uint32_t>(p);
}

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
  constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0, lo0, hi1, lo1;
    mulhilo32(M0, c.x, hi0, lo0);
    mulhilo32(M1, c.z, hi1, lo1);
    c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    k0 += W0;
    k1 += W1;
  }
  return c;
}

__host__ __device__ __forceinline__ U4 philox_at(uint64_t seed, uint64_t sid, uint64_t i) {
  return philox4x32_10(U4{static_cast<uint32_t>(i), static_cast<uint32_t>(i >> 32),
                          static_cast<uint32_t>(sid), static_cast<uint32_t>(sid >> 32)},
                       static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

// [0,1) in binary32: top 24 bits of word 0.
__host__ __device__ __forceinline__ float u01_f32(U4 r) {
  return static_cast<float>(r.x >> 8) * 0x1p-24f;
}
// [0,1) in binary64: top 53 bits of (word0:word1).
__host__ __device__ __forceinline__ double u01_f64(U4 r) {
  uint64_t u = (static_cast<uint64_t>(r.x) << 32) | r.y;
  return static_cast<double>(u >> 11) * 0x1p-53;
}
// Second independent binary64 uniform of the same draw (words 2:3).
__host__ __device__ __forceinline__ double u01_f64_hi(U4 r) {
  uint64_t u = (static_cast<uint64_t>(r.z) << 32) | r.w;
  return static_cast<double>(u >> 11) * 0x1p-53;
}

// Keyed bijection on [0, total) (cfg3's "random-permuted" layout): a 4-round
// balanced Feistel network on the smallest even bit width w with 2^w >= total,
// cycle-walked back into range.  Round keys come from the seed.
__host__ __device__ __forceinline__ uint32_t feistel_f(uint32_t r, uint32_t k) {
  uint32_t x = r * 0x9E3779B1u ^ k;
  x ^= x >> 15; x *= 0x85EBCA77u;
  x ^= x >> 13; x *= 0xC2B2AE3Du;
  x ^= x >> 16;
  return x;
}
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ int feistel_half_bits(uint64_t total) {
  int w = 2;
  while (w < 62 && (1ull << w) < total) w += 2;
  return w / 2;
}
__host__ __device__ __forceinline__ uint64_t feistel_permute(uint64_t p, uint64_t total, uint64_t seed) {
  const int hb = feistel_half_bits(total);
  const uint64_t mask = (1ull << hb) - 1ull;
  uint32_t keys[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) keys[k] = static_cast<uint32_t>(splitmix64(seed * 4ull + k));
  uint64_t x = p;
  do {
    uint64_t L = x >> hb, R = x & mask;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint64_t nL = R;
      R = L ^ (static_cast<uint64_t>(feistel_f(static_cast<uint32_t>(R), keys[k])) & mask);
      L = nL;
    }
    x = (L << hb) | R;
  } while (x >= total);
  return x;
}

}  // namespace tfb
