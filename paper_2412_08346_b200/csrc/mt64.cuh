// Device-side std::mt19937_64 (the engine behind graspmatch::Rng,
// rng.hpp:16-70) and Lemire's multiply-shift reduction (rng.hpp:32-44).
//
// Each particle owns one stream seeded with seed + j (grasp.cpp:149-151).
// The 312-word state lives in global memory between iterations; a CTA
// regenerates it cooperatively: the in-place twist splits into two
// dependency-free halves (positions [0,156) read only old words; positions
// [156,312) read new words of the first half), so 128 threads do a twist in
// two barrier-separated passes.
#pragma once

#include <cstdint>

namespace asicp {
namespace mt {

constexpr int kN = 312;
constexpr int kM = 156;
constexpr uint64_t kMatrixA = 0xB5026F5AA96619E9ull;
constexpr uint64_t kUpper = 0xFFFFFFFF80000000ull;
constexpr uint64_t kLower = 0x000000007FFFFFFFull;

__host__ __device__ __forceinline__ uint64_t temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= (y >> 43);
  return y;
}

__host__ __device__ __forceinline__ uint64_t mix(uint64_t a, uint64_t b) {
  const uint64_t y = (a & kUpper) | (b & kLower);
  return (y >> 1) ^ ((y & 1ull) ? kMatrixA : 0ull);
}

// std::mt19937_64(seed) initialisation.
__host__ __device__ inline void seed_state(uint64_t* s, uint64_t seed) {
  s[0] = seed;
  for (int i = 1; i < kN; ++i) s[i] = 6364136223846793005ull * (s[i - 1] ^ (s[i - 1] >> 62)) + static_cast<uint64_t>(i);
}

// Cooperative in-place twist of a shared-memory state by the whole CTA.
// Must be called by all threads of the block.
__device__ __forceinline__ void twist_block(uint64_t* s) {
  const int tid = threadIdx.x, nt = blockDim.x;
  // Phase 1: k in [0, 156) reads only old words.
  uint64_t v[3];
  int cnt = 0;
  for (int k = tid; k < kM; k += nt) v[cnt++] = s[k + kM] ^ mix(s[k], s[k + 1]);
  __syncthreads();
  cnt = 0;
  for (int k = tid; k < kM; k += nt) s[k] = v[cnt++];
  __syncthreads();
  // Phase 2: k in [156, 312) reads new s[k-156] and old s[k], s[k+1]
  // (k = 311 reads the new s[0]).
  cnt = 0;
  for (int k = kM + tid; k < kN; k += nt) {
    const uint64_t next = (k + 1 < kN) ? s[k + 1] : s[0];
    v[cnt++] = s[k - kM] ^ mix(s[k], next);
  }
  __syncthreads();
  cnt = 0;
  for (int k = kM + tid; k < kN; k += nt) s[k] = v[cnt++];
  __syncthreads();
}

// Serial twist (single thread), used by the rare rejection fallback.
__device__ __forceinline__ void twist_serial(uint64_t* s) {
  int k = 0;
  for (; k < kN - kM; ++k) s[k] = s[k + kM] ^ mix(s[k], s[k + 1]);
  for (; k < kN - 1; ++k) s[k] = s[k - (kN - kM)] ^ mix(s[k], s[k + 1]);
  s[kN - 1] = s[kM - 1] ^ mix(s[kN - 1], s[0]);
}

// Lemire reduction of one raw output x into [0, n): returns true when the
// draw is accepted (rng.hpp:35-43: lo >= n, or lo >= (2^64 - n) mod n).
__device__ __forceinline__ bool lemire(uint64_t x, uint64_t n, uint64_t* out) {
  const uint64_t lo = x * n;
  *out = __umul64hi(x, n);
  if (lo < n) {
    const uint64_t threshold = (0ull - n) % n;
    if (lo < threshold) return false;
  }
  return true;
}

}  // namespace mt
}  // namespace asicp
