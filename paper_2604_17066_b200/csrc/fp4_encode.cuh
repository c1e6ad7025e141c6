// FP4 sample-operand words (include/rsr_b200.h "FP4 layout"), shared by the
// fused sampler (sample.cu) and the standalone encoder (classify_fp4.cu).
#pragma once
#include <stdint.h>

namespace rsr {

// Word w of a sample row = elements c0 = 8w .. 8w+7 (low nibble first, e2m1
// 1.0 = 0x2): A_up[c] = [x_n < k], A_lo[c] = [x_n >= k] for c < kdim,
// c = n(M-1) + k-1; both 1 at the bias column c = kdim; 0 beyond.  `x` is the
// row's states (byte addressable, e.g. shared memory).
__device__ __forceinline__ void fp4_sample_word(const uint8_t* x, int w, int M, int kdim,
                                                uint32_t& up, uint32_t& lo) {
  const int c0 = 8 * w;
  if (M == 2 && c0 + 8 <= kdim) {
    // 8 states (0/1) -> 8 nibbles: byte j's bit 0 moves to bit 4j+1
    uint32_t a = 0, b = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      a |= (uint32_t)x[c0 + j] << (8 * j);
      b |= (uint32_t)x[c0 + 4 + j] << (8 * j);
    }
    const uint32_t na = (a & 1u) | ((a >> 4) & 0x10u) | ((a >> 8) & 0x100u) | ((a >> 12) & 0x1000u);
    const uint32_t nb = (b & 1u) | ((b >> 4) & 0x10u) | ((b >> 8) & 0x100u) | ((b >> 12) & 0x1000u);
    lo = (na | (nb << 16)) << 1;  // [x >= 1]
    up = lo ^ 0x22222222u;        // [x < 1]
    return;
  }
  if (M == 3 && c0 + 8 <= kdim) {
    // 4 states (0..2) -> 4 bytes, one per component: nibbles [x<1], [x<2] (A_up)
    // and [x>=1], [x>=2] (A_lo), by byte permutes over 3-entry tables
    const int n0 = c0 / 2;
    uint32_t a = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) a |= (uint32_t)x[n0 + j] << (8 * j);
    const uint32_t sel = (a & 0xFu) | ((a >> 4) & 0xF0u) | ((a >> 8) & 0xF00u) | ((a >> 12) & 0xF000u);
    up = __byte_perm(0x00002022u, 0u, sel);  // x = 0, 1, 2 -> 0x22, 0x20, 0x00
    lo = __byte_perm(0x00220200u, 0u, sel);  // x = 0, 1, 2 -> 0x00, 0x02, 0x22
    return;
  }
  up = lo = 0;
  int n = c0 / (M - 1), k = c0 - n * (M - 1) + 1;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int c = c0 + j;
    uint32_t u, l;
    if (c < kdim) {
      u = x[n] < k;
      l = 1 - u;
    } else {
      u = l = (c == kdim);
    }
    up |= (u ? 0x2u : 0u) << (4 * j);
    lo |= (l ? 0x2u : 0u) << (4 * j);
    if (++k == M) {
      k = 1;
      ++n;
    }
  }
}

}  // namespace rsr
