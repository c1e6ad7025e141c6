// Counter-based generators of the sampler.
//  * Philox4x64-10 (Random123 constants), bit-compatible with numpy.random.Philox:
//    the reference's stream (sampling.py:39-66), RSR_RNG_SHARED.
//  * Philox4x32-10 (Random123 constants): the independent device stream,
//    RSR_RNG_DEVICE -- 32x32-bit multiplies (one IMAD.WIDE.U32 each) instead of
//    64x64-bit ones, four 32-bit draws per block.
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
    const uint64_t p0 = (uint64_t)M0 * c0, p1 = (uint64_t)M1 * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0, n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

// Device stream, block b of generation `gen`: counter (b, gen), key seed (64-bit
// halves).  Flat draw f of a generation is word f % 4 of block f / 4, as for the
// shared stream.
__device__ __forceinline__ void device_block(uint64_t b, uint64_t seed, uint64_t gen,
                                             uint32_t out[4]) {
  philox4x32_10((uint32_t)b, (uint32_t)(b >> 32), (uint32_t)gen, (uint32_t)(gen >> 32),
                (uint32_t)seed, (uint32_t)(seed >> 32), out);
}

// The four draws of flat block b as 53-bit fixed-point values r (u = r * 2^-53)
// compared against the thresholds T = ceil(cum * 2^53).  Shared stream: r = raw >> 11
// (numpy's random() mantissa).  Device stream: r = raw32 << 21, so r >= T <=> raw32 >=
// ceil(cum * 2^32) -- the inverse CDF at 2^-32 resolution.
template <int RNG, bool C32>
__device__ __forceinline__ void draw_block(int64_t b, uint64_t seed, uint64_t gen,
                                           unsigned long long r[4]) {
  if (RNG == 0) {
    uint64_t w[4];
    if (C32)
      philox4x64_10((uint64_t)(uint32_t)(b + 1), seed, gen, w);
    else
      philox4x64_10((uint64_t)b + 1ull, seed, gen, w);
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = w[j] >> 11;
  } else {
    uint32_t w[4];
    device_block((uint64_t)b, seed, gen, w);
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = (unsigned long long)w[j] << 21;
  }
}

}  // namespace rsr
