// Counter-based generators of the sampler.
//  * Philox4x64-10 (Random123 constants), bit-compatible with numpy.random.Philox:
//    the reference's stream (sampling.py:39-66), RSR_RNG_SHARED.
//  * Philox4x32-10 (Random123 constants): the independent device stream,
//    RSR_RNG_DEVICE -- 32x32-bit multiplies (one IMAD.WIDE.U32 each) instead of
//    64x64-bit ones, four 32-bit draws per block, blocks aligned to sample rows.
#pragma once
#include <stdint.h>

namespace rsr {

__device__ __forceinline__ void philox4x64_10(uint64_t ctr0, uint64_t key0, uint64_t key1,
                                              uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      key0 += W0;
      key1 += W1;
    }
    const uint64_t hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
    const uint64_t hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
    const uint64_t n0 = hi1 ^ c1 ^ key0, n2 = hi0 ^ c3 ^ key1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

__device__ __forceinline__ void mul_wide_u32(uint32_t a, uint32_t b, uint32_t& lo, uint32_t& hi) {
  // one IMAD.WIDE.U32; written out because the C++ (uint64_t)a * b form leaves a
  // stray add of a zero high word per product in the generated SASS
  uint64_t p;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(p) : "r"(a), "r"(b));
  asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(p));
}

// Round keys of Philox4x32-10 for key (k0, k1): round r uses (k0 + r W0, k1 + r W1).
struct Philox32Keys {
  uint32_t k0[10], k1[10];
};

__host__ __device__ inline Philox32Keys philox32_keys(uint32_t k0, uint32_t k1) {
  Philox32Keys K;
  for (int r = 0; r < 10; ++r) {
    K.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    K.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return K;
}

// Philox4x32-10 of counter (c0..c3) under a precomputed key schedule (a kernel
// parameter: the XORs then take the round key straight from the constant bank).
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              const Philox32Keys& K, uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0, hi0, lo1, hi1;
    mul_wide_u32(M0, c0, lo0, hi0);
    mul_wide_u32(M1, c2, lo1, hi1);
    c0 = hi1 ^ c1 ^ K.k0[r];
    c1 = lo1;
    c2 = hi0 ^ c3 ^ K.k1[r];
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Philox4x32-10: counter (c0..c3), key (k0, k1).
__device__ __forceinline__ void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                              uint32_t k0, uint32_t k1, uint32_t out[4]) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += W0;
      k1 += W1;
    }
    uint32_t lo0, hi0, lo1, hi1;
    mul_wide_u32(M0, c0, lo0, hi0);
    mul_wide_u32(M1, c2, lo1, hi1);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Device stream, row-aligned: draw (row R, component n) of generation `gen` is word
// n % 4 of the Philox4x32-10 block with counter [n / 4, R lo, R hi, gen lo] and key
// [seed lo ^ gen hi, seed hi].  A row's draws come in whole blocks (N = 295: 74 blocks,
// the last one partly used), so a lane can produce the FP4 words of its own row segment
// without staging the draws through shared memory the way the flat-indexed reference
// stream needs.
__device__ __forceinline__ void device_row_block(uint64_t row, uint32_t q, uint64_t seed,
                                                 uint64_t gen, uint32_t out[4]) {
  philox4x32_10(q, (uint32_t)row, (uint32_t)(row >> 32), (uint32_t)gen,
                (uint32_t)seed ^ (uint32_t)(gen >> 32), (uint32_t)(seed >> 32), out);
}

__host__ __device__ inline Philox32Keys device_keys(uint64_t seed, uint64_t gen) {
  return philox32_keys((uint32_t)seed ^ (uint32_t)(gen >> 32), (uint32_t)(seed >> 32));
}

// The same block with the key schedule of device_keys(seed, gen) precomputed.
__device__ __forceinline__ void device_row_block(uint64_t row, uint32_t q, uint64_t gen,
                                                 const Philox32Keys& K, uint32_t out[4]) {
  philox4x32_10(q, (uint32_t)row, (uint32_t)(row >> 32), (uint32_t)gen, K, out);
}

// The four draws of flat block b of the reference stream as 53-bit fixed-point values
// r (u = r * 2^-53, numpy's random() mantissa raw >> 11) compared against the
// thresholds T = ceil(cum * 2^53).  (The device stream compares raw32 << 21 with the
// same table: r >= T <=> raw32 >= ceil(cum * 2^32), the inverse CDF at 2^-32.)
template <bool C32>
__device__ __forceinline__ void draw_block(int64_t b, uint64_t seed, uint64_t gen,
                                           unsigned long long r[4]) {
  uint64_t w[4];
  if (C32)
    philox4x64_10((uint64_t)(uint32_t)(b + 1), seed, gen, w);
  else
    philox4x64_10((uint64_t)b + 1ull, seed, gen, w);
#pragma unroll
  for (int j = 0; j < 4; ++j) r[j] = w[j] >> 11;
}

}  // namespace rsr
