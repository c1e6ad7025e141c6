// (1) On-device sampling and (2) thermometer encodings.
//
// Replaces sampling.py:39-90 (numpy Philox4x64-10 stream keyed by
// [seed, generation_index], flat draw index (start+i)*N + n, inverse CDF by
// searchsorted(side="right") on cumsum(probs)) and encoding.py:138-153.
//
// Bit-exactness: numpy's Philox pre-increments its 256-bit counter, so flat
// draw f is word f%4 of the block generated from counter f/4 + 1.  The
// inverse CDF is done in integers: with r = raw >> 11 and u = r * 2^-53
// (exact), u >= cum  <=>  r >= ceil(cum * 2^53) (scaling by 2^53 is exact), so
// state = #{m < M-1 : r >= T_m} with T_m = ceil(cumsum(probs[n])[m] * 2^53).
// The clip to M-1 (sampling.py:89) is implied by counting only m < M-1.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "fp4_encode.cuh"
#include "philox.cuh"

namespace {

constexpr int kThreads = 256;

// Per-block prologue: thresholds T[n*(M-1)+m] from a sequential fp64 cumsum
// (np.cumsum order), stored in shared memory.
__device__ void load_thresholds(const double* __restrict__ probs, int N, int M,
                                unsigned long long* T) {
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    double cum = 0.0;
    for (int m = 0; m < M - 1; ++m) {
      cum = __dadd_rn(cum, probs[(int64_t)n * M + m]);
      double scaled = __dmul_rn(cum, 9007199254740992.0);  // * 2^53, exact
      T[n * (M - 1) + m] = (unsigned long long)ceil(scaled);
    }
  }
  __syncthreads();
}

// Row-end padding of one thermometer row: nbias ones then zeros up to ld.
__device__ __forceinline__ void thermo_tail(int8_t* arow, int kdim, int nbias, int ld) {
  for (int c = kdim; c < ld; ++c) arow[c] = (int8_t)(c < kdim + nbias);
}

// One Philox block (4 consecutive flat draws) per thread.  M2 specialises the
// binary case (state = [r >= T_n], thermometer byte = 1 - state).  The row of
// flat index fb is fb / N computed as a multiply-high by magic = floor(2^64/N)
// plus one correction step.
template <bool M2, int RNG>
__global__ void __launch_bounds__(kThreads)
sample_kernel(const double* __restrict__ probs, int N, int M, uint64_t seed, uint64_t gen,
              int64_t f0, int64_t f1, int64_t b_lo, int64_t nblk, uint8_t* __restrict__ states,
              int8_t* __restrict__ thermo, int ld, int kdim, int nbias, uint64_t magic,
              int64_t start_row) {
  extern __shared__ unsigned long long T[];
  load_thresholds(probs, N, M, T);
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblk) return;
  const int64_t b = b_lo + t;
  const uint64_t fb = 4ull * (uint64_t)b;
  uint64_t row = __umul64hi(fb, magic);
  int n = (int)(fb - row * (uint64_t)N);
  if (n >= N) {
    n -= N;
    ++row;
  }
  unsigned long long rr[4];
  if (RNG == 0) {
    rsr::draw_block<false>(b, seed, gen, rr);
  } else {
    // device stream: draw (row, n) from that row's block n / 4 (rows are block-aligned,
    // so the four flat draws may come from two blocks)
    uint64_t r = row;
    int nn = n;
    uint32_t w[4];
    int q = -1;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if ((nn >> 2) != q) {
        q = nn >> 2;
        rsr::device_row_block(r, (uint32_t)q, seed, gen, w);
      }
      rr[j] = (unsigned long long)w[nn & 3] << 21;
      if (++nn == N) {
        nn = 0;
        ++r;
        q = -1;
      }
    }
  }
  uint8_t st[4];
  int ns[4];
  int64_t rows[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const unsigned long long r = rr[j];
    int s;
    if (M2) {
      s = r >= T[n] ? 1 : 0;
    } else {
      s = 0;
      const unsigned long long* Tn = T + n * (M - 1);
      for (int m = 0; m < M - 1; ++m) s += (r >= Tn[m]) ? 1 : 0;
    }
    st[j] = (uint8_t)s;
    ns[j] = n;
    rows[j] = (int64_t)row - start_row;
    if (++n == N) {
      n = 0;
      ++row;
    }
  }
  const bool full = (int64_t)fb >= f0 && (int64_t)fb + 3 < f1;
  if (states) {
    if (full && ((f0 & 3) == 0)) {
      const uint32_t packed = (uint32_t)st[0] | ((uint32_t)st[1] << 8) | ((uint32_t)st[2] << 16) |
                              ((uint32_t)st[3] << 24);
      *reinterpret_cast<uint32_t*>(states + ((int64_t)fb - f0)) = packed;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t f = (int64_t)fb + j;
        if (f >= f0 && f < f1) states[f - f0] = st[j];
      }
    }
  }
  if (thermo) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t f = (int64_t)fb + j;
      if (full || (f >= f0 && f < f1)) {
        int8_t* arow = thermo + rows[j] * (int64_t)ld;
        if (M2) {
          arow[ns[j]] = (int8_t)(1 - st[j]);
        } else {
          for (int k = 1; k < M; ++k) arow[ns[j] * (M - 1) + (k - 1)] = (int8_t)(st[j] < k);
        }
        if (ns[j] == N - 1) thermo_tail(arow, kdim, nbias, ld);
      }
    }
  }
}

// Row-blocked sampler with the FP4 operand fused (the default path).  A CTA
// owns kRowsPerCta whole rows: its threads compute every Philox block that
// overlaps the rows' flat draw range (blocks straddling two CTAs are computed
// by both, each keeping its own draws), drop the states into shared memory,
// then write the uint8 state rows (16-byte stores: the chunk is 32-row
// aligned) and the FP4 rows [A_up | A_lo] (16-byte stores, 4 words a thread).
//
// The generator is bound by the 64-bit multiplies of Philox4x64-10 on the FMA
// pipe (tools/philox_rate.cu: 0.79 ms per 2^20 x 295 draws for the bare
// generator), so the rest is kept off that pipe and branch-free: the
// threshold table has N + 3 rows (row n >= N repeats row n - N) so a block's
// four draws index T without a wrap test, interior blocks store their four
// states as one 32-bit word, and the FP4 pass reads each row segment with
// aligned 32-bit loads + funnel shifts and converts 8 states per word with a
// few shifts and one byte permute.
constexpr int kRowsPerCta = 64;
constexpr int kRowThreads = 256;
constexpr int kChunksPerCta = 2;
constexpr int kTExtra = 3;  // extra threshold rows (no wrap within a block)
#ifndef RSR_SAMPLE_MINB
#define RSR_SAMPLE_MINB 3
#endif

__device__ void load_thresholds_ext(const double* __restrict__ probs, int N, int M,
                                    unsigned long long* T) {
  for (int n = threadIdx.x; n < N + kTExtra; n += blockDim.x) {
    const int src = n % N;
    double cum = 0.0;
    for (int m = 0; m < M - 1; ++m) {
      cum = __dadd_rn(cum, probs[(int64_t)src * M + m]);
      T[n * (M - 1) + m] = (unsigned long long)ceil(__dmul_rn(cum, 9007199254740992.0));
    }
  }
  __syncthreads();
}

// 8 consecutive state bytes starting at shared byte offset `base` (any
// alignment) as two 32-bit words, from aligned loads + funnel shifts.
template <int W>
__device__ __forceinline__ void load_state_words(const uint8_t* st, uint32_t base, uint32_t* x) {
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(st + (base & ~3u));
  const uint32_t sh = (base & 3u) * 8u;
  uint32_t raw[W + 1];
#pragma unroll
  for (int k = 0; k <= W; ++k) raw[k] = wp[k];
#pragma unroll
  for (int k = 0; k < W; ++k) x[k] = __funnelshift_r(raw[k], raw[k + 1], sh);
}

// FP4 words of one quad (4 words = 32 elements) of a state row, fast paths
// for quads wholly below kdim (M = 2: 8 states per word; M = 3: 4 states).
template <int MT>
__device__ __forceinline__ void fp4_quad_fast(const uint8_t* st, uint32_t base, uint32_t* u,
                                              uint32_t* l) {
  if (MT == 2) {
    uint32_t x[8];
    load_state_words<8>(st, base, x);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      // bytes (e0..e3), (e4..e7) of 0/1 -> nibble j = e_j at bit 4j+1
      const uint32_t ta = x[2 * t] | (x[2 * t] >> 4), tb = x[2 * t + 1] | (x[2 * t + 1] >> 4);
      l[t] = __byte_perm(ta, tb, 0x6420) << 1;  // [x >= 1]
      u[t] = l[t] ^ 0x22222222u;               // [x <  1]
    }
  } else {
    uint32_t x[4];
    load_state_words<4>(st, base, x);
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t a = x[t];
      const uint32_t sel =
          (a & 0xFu) | ((a >> 4) & 0xF0u) | ((a >> 8) & 0xF00u) | ((a >> 12) & 0xF000u);
      u[t] = __byte_perm(0x00002022u, 0u, sel);  // x = 0, 1, 2 -> 0x22, 0x20, 0x00
      l[t] = __byte_perm(0x00220200u, 0u, sel);  // x = 0, 1, 2 -> 0x00, 0x02, 0x22
    }
  }
}

// Each CTA computes the threshold table once, then walks kChunksPerCta chunks
// of kRowsPerCta rows (chunk c = blockIdx.x + k * gridDim.x) with the state
// staging buffer double-buffered, so one barrier per chunk separates the
// generator phase from the store phase (the next chunk's generator writes the
// other buffer).
// C32: every Philox counter of the launch fits 32 bits (flat draws < 2^34), so
// the first round's 64x64 multiply is a 64x32 one (two IMAD.WIDE fewer per block
// on the FMA pipe, which bounds this kernel).
// RPC: rows per chunk (64; 16 for the widest rows, whose 64-row staging buffers would not
// fit shared memory)
template <int MT, bool C32, int RPC = kRowsPerCta>  // MT 2, 3: specialised state count; 0: any M
__global__ void __launch_bounds__(kRowThreads, RSR_SAMPLE_MINB)
sample_rows_kernel(const double* __restrict__ probs, int N, int M, uint64_t seed, uint64_t gen,
                   int64_t start_row, int64_t count, uint8_t* __restrict__ states,
                   uint8_t* __restrict__ fp4, int row_bytes, int st_bytes, int64_t fp4_row_stride,
                   int64_t fp4_plane) {
  extern __shared__ __align__(16) unsigned long long T[];
  load_thresholds_ext(probs, N, M, T);
  const int Mm1 = MT ? MT - 1 : M - 1;
  // two [rows][N] state buffers (+16 B slack each for the funnel loads)
  uint8_t* st_base =
      reinterpret_cast<uint8_t*>(T) + ((size_t)(N + kTExtra) * Mm1 * 8 + 15) / 16 * 16;
  const int kdim = N * Mm1, words = row_bytes / 4, quads = words / 4;
  const int fastq = MT ? kdim / 32 : 0;  // quads per row on the specialised path
  const int64_t n_chunks = (count + RPC - 1) / RPC;
  int buf = 0;
  for (int64_t chunk = blockIdx.x; chunk < n_chunks; chunk += gridDim.x, buf ^= 1) {
    uint8_t* st = st_base + buf * st_bytes;
    const int64_t r0 = chunk * RPC;
    const int rows = (int)(count - r0 < RPC ? count - r0 : RPC);
    const int span = rows * N;                                     // draws of this chunk
    const int64_t f0 = (start_row + r0) * (int64_t)N;              // first flat draw
    const int64_t b0 = f0 >> 2, b1 = (f0 + span - 1) >> 2;         // Philox blocks
    const bool aligned = (f0 & 3) == 0;                            // o0 % 4 == 0 for all blocks
    // local draw offset of word 0 of this thread's first block, and its column;
    // each further block of the thread is 4 * blockDim.x draws later
    int o0 = (int)(4 * (b0 + threadIdx.x) - f0);
    int n0 = (o0 + N) % N;
    const int ostep = 4 * (int)blockDim.x, nstep = ostep % N;
    for (int64_t b = b0 + threadIdx.x; b <= b1; b += blockDim.x, o0 += ostep) {
      unsigned long long rr[4];
      rsr::draw_block<C32>(b, seed, gen, rr);
      const unsigned long long* Tn = T + n0 * Mm1;
      n0 += nstep;
      if (n0 >= N) n0 -= N;
      uint32_t s[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned long long r = rr[j];
        const unsigned long long* Tj = Tn + j * Mm1;
        if (MT == 2) {
          s[j] = r >= Tj[0];
        } else if (MT == 3) {
          s[j] = (uint32_t)(r >= Tj[0]) + (uint32_t)(r >= Tj[1]);
        } else {
          uint32_t c = 0;
          for (int m = 0; m < Mm1; ++m) c += r >= Tj[m];
          s[j] = c;
        }
      }
      if (o0 >= 0 && o0 + 4 <= span) {
        if (aligned) {
          *reinterpret_cast<uint32_t*>(st + o0) = s[0] | (s[1] << 8) | (s[2] << 16) | (s[3] << 24);
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) st[o0 + j] = (uint8_t)s[j];
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (o0 + j >= 0 && o0 + j < span) st[o0 + j] = (uint8_t)s[j];
      }
    }
    __syncthreads();
    if (states) {
      uint8_t* dst = states + r0 * (int64_t)N;
      if (rows == RPC) {  // RPC * N bytes, 16-byte aligned chunk
        const int vecs = span / 16;
        for (int i = threadIdx.x; i < vecs; i += blockDim.x)
          reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(st)[i];
      } else {
        for (int i = threadIdx.x; i < span; i += blockDim.x) dst[i] = st[i];
      }
    }
    if (fp4) {
      // items (row, quad): the specialised quads first, then the quads holding
      // the bias column / zero padding (generic per-word encoder), in separate
      // loops so a warp does not diverge between the two
      const int nfast = rows * fastq, slowq = quads - fastq;
      for (int i = threadIdx.x; MT != 0 && i < nfast; i += blockDim.x) {
        const int r = i / (MT ? fastq : 1), q = i - r * fastq;
        uint4 up, lo;
        fp4_quad_fast<MT>(st, (uint32_t)(r * N + (MT == 2 ? 32 : 16) * q), &up.x, &lo.x);
        uint8_t* row = fp4 + (r0 + r) * fp4_row_stride;
        reinterpret_cast<uint4*>(row)[q] = up;
        reinterpret_cast<uint4*>(row + fp4_plane)[q] = lo;
      }
      for (int i = threadIdx.x; i < rows * slowq; i += blockDim.x) {
        const int r = i / slowq, q = fastq + (i - r * slowq);
        uint4 up, lo;
        uint32_t* u = &up.x;
        uint32_t* l = &lo.x;
#pragma unroll
        for (int t = 0; t < 4; ++t) rsr::fp4_sample_word(st + r * N, 4 * q + t, M, kdim, u[t], l[t]);
        uint8_t* row = fp4 + (r0 + r) * fp4_row_stride;
        reinterpret_cast<uint4*>(row)[q] = up;
        reinterpret_cast<uint4*>(row + fp4_plane)[q] = lo;
      }
    }
  }
}

__global__ void philox_raw_kernel(uint64_t seed, uint64_t gen, int64_t first, int64_t count,
                                  int64_t b_lo, int64_t nblk, uint64_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblk) return;
  const int64_t b = b_lo + t;
  uint64_t w[4];
  rsr::philox4x64_10((uint64_t)b + 1ull, seed, gen, w);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t f = 4 * b + j;
    if (f >= first && f < first + count) out[f - first] = w[j];
  }
}

// Raw draws of rows [start, start + count) of the device stream, one thread per block.
__global__ void device_raw_kernel(uint64_t seed, uint64_t gen, int64_t start, int64_t count,
                                  int N, uint32_t* __restrict__ out) {
  const int qb = (N + 3) / 4;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * qb) return;
  const int64_t i = t / qb;
  const int q = (int)(t - i * qb);
  uint32_t w[4];
  rsr::device_row_block((uint64_t)(start + i), (uint32_t)q, seed, gen, w);
#pragma unroll
  for (int j = 0; j < 4; ++j)
    if (4 * q + j < N) out[i * N + 4 * q + j] = w[j];
}

// Row-aligned sampler of the device stream with the FP4 operand fused.  Thread
// (rr, w) of a CTA owns FP4 word w (columns 8w .. 8w+7 of both halves) of rows
// rr, rr + R, rr + 2R, ... of the CTA's row chunk, and the states of the components
// those columns belong to -- M = 2: components 8w .. 8w+7 (two Philox blocks), M = 3:
// 4w .. 4w+3 (one block), other M generic.  Each thread derives its 8 column
// thresholds once, into registers: no shared memory, no barriers, no per-item division
// (the flat-indexed reference stream needs shared-memory staging of its draws).
//
// Column c = n (M-1) + k - 1 of the operand is [x_n >= k] in the lower half and its
// complement in the upper one, and x_n >= k <=> raw32_n >= T32 = ceil(cum_{n,k-1} 2^32)
// (T53 = ceil(cum 2^53) from the sampler's sequential fp64 cumsum, T32 = ceil(T53 / 2^21)).
// A threshold of 2^32 is out of 32-bit range; such a column never counts (its value v
// is 0), which also covers the columns past kdim.
__device__ __forceinline__ void column_threshold(const double* __restrict__ probs, int M, int Mm1,
                                                 int c, uint32_t& t, bool& valid) {
  const int n = c / Mm1, m = c - n * Mm1;
  double cum = 0.0;
  for (int i = 0; i <= m; ++i) cum = __dadd_rn(cum, probs[(int64_t)n * M + i]);
  const unsigned long long t53 = (unsigned long long)ceil(__dmul_rn(cum, 9007199254740992.0));
  const unsigned long long t32 = (t53 + ((1ull << 21) - 1)) >> 21;
  valid = !(t32 >> 32);
  t = valid ? (uint32_t)t32 : ~0u;
}

template <int MT>
__global__ void __launch_bounds__(1024) sample_dev_rows_kernel(
    const double* __restrict__ probs, int N, int M, const rsr::Philox32Keys K, uint64_t gen,
    int64_t start, int64_t count, uint8_t* __restrict__ states, uint8_t* __restrict__ fp4,
    int words, int R, int passes, int64_t row_stride, int64_t plane) {
  // U rows per thread per pass (M = 2, 3): their Philox chains are independent, so the
  // scheduler interleaves them (a chain is 10 dependent multiply-xor rounds)
  constexpr int U = MT ? 2 : 1;
  const int PR = U * R;  // rows per pass
  // state rows of a pass, staged (double-buffered) so they leave as aligned 16-byte
  // stores: rows of N bytes are not word aligned, and a lane's 8 state bytes would
  // otherwise need up to four differently sized stores
  extern __shared__ __align__(16) uint8_t stage[];
  const int stage_bytes = (PR * N + 16 + 15) & ~15;
  const int w = threadIdx.x % words, rr = threadIdx.x / words;
  const bool lane_on = rr < R;
  const int Mm1 = MT ? MT - 1 : M - 1;
  const int kdim = N * Mm1;
  // per-thread column constants
  uint32_t T[8], v[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const int c = 8 * w + s;
    T[s] = ~0u;
    v[s] = 0;
    if (lane_on && c < kdim) {
      bool ok;
      column_threshold(probs, M, Mm1, c, T[s], ok);
      if (ok) v[s] = MT == 2 ? 1u << (8 * (s & 3)) : MT == 3 ? 1u << (8 * (s >> 1)) : 2u << (4 * s);
    }
  }
  const int rem = kdim - 8 * w;  // columns of this word below kdim
  const uint32_t flip = rem >= 8 ? 0x22222222u : rem > 0 ? (0x22222222u & ((1u << (4 * rem)) - 1u)) : 0u;
  const uint32_t bias = rem >= 0 && rem < 8 ? 2u << (4 * rem) : 0u;
  const bool has_cols = lane_on && rem > 0;
  const int nst = MT == 2 ? min(8, N - 8 * w) : MT == 3 ? min(4, N - 4 * w) : 0;
  const int64_t c0 = (int64_t)blockIdx.x * PR * passes;  // first row of this CTA
  const int64_t left = (count - c0 + PR - 1) / PR;
  const int np = left < passes ? (int)left : passes;
  for (int p = 0; p < np; ++p) {
    const int64_t pr = c0 + (int64_t)p * PR;  // first row of the pass
    const int prows = count - pr < PR ? (int)(count - pr) : PR;
    uint8_t* buf = stage + (p & 1) * stage_bytes;
    const int sb = states ? (int)(reinterpret_cast<uintptr_t>(states + pr * N) & 15u) : 0;
    uint32_t lo[U];
#pragma unroll
    for (int u = 0; u < U; ++u) lo[u] = 0;
    if (has_cols) {
      if (MT == 2) {
        // both blocks of every row, unconditionally (a word past N/8 + 1/2 has v = 0 on
        // its upper half), so the U x 2 chains form one straight-line block
        uint32_t d[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t row = (uint64_t)(start + pr + u * R + rr);
          rsr::device_row_block(row, (uint32_t)(2 * w), gen, K, d[u]);
          rsr::device_row_block(row, (uint32_t)(2 * w + 1), gen, K, d[u] + 4);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t s0 = 0, s1 = 0;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            s0 += d[u][s] >= T[s] ? v[s] : 0u;
            s1 += d[u][s + 4] >= T[s + 4] ? v[s + 4] : 0u;
          }
          // state bytes (0/1) -> nibbles at bit 4j + 1 (cf. fp4_quad_fast)
          lo[u] = __byte_perm(s0 | (s0 >> 4), s1 | (s1 >> 4), 0x6420) << 1;
          if (states && u * R + rr < prows) {
            uint8_t* srow = buf + sb + (u * R + rr) * N;
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (j < nst) srow[8 * w + j] = (uint8_t)((j < 4 ? s0 : s1) >> (8 * (j & 3)));
          }
        }
      } else if (MT == 3) {
        uint32_t d[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u)
          rsr::device_row_block((uint64_t)(start + pr + u * R + rr), (uint32_t)w, gen, K, d[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) {
          uint32_t s0 = 0;
#pragma unroll
          for (int s = 0; s < 8; ++s) s0 += d[u][s >> 1] >= T[s] ? v[s] : 0u;
          const uint32_t sel = (s0 & 0xFu) | ((s0 >> 4) & 0xF0u) | ((s0 >> 8) & 0xF00u) |
                               ((s0 >> 12) & 0xF000u);
          lo[u] = __byte_perm(0x00220200u, 0u, sel);  // x = 0, 1, 2 -> 0x00, 0x02, 0x22
          if (states && u * R + rr < prows) {
            uint8_t* srow = buf + sb + (u * R + rr) * N;
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (j < nst) srow[4 * w + j] = (uint8_t)(s0 >> (8 * j));
          }
        }
      } else if (rr < prows) {
        const uint64_t row = (uint64_t)(start + pr + rr);
        uint32_t d[4];
        int q = -1;
        for (int s = 0; s < 8; ++s) {
          const int n = (8 * w + s) / Mm1;
          if (n >= N) break;
          if ((n >> 2) != q) {
            q = n >> 2;
            rsr::device_row_block(row, (uint32_t)q, gen, K, d);
          }
          lo[0] |= d[n & 3] >= T[s] ? v[s] : 0u;
        }
        if (states) {
          // component n is written by the word holding its first column; x_n counts its
          // columns set (columns in later words are compared here directly)
          uint8_t* srow = buf + sb + rr * N;
          for (int s = 0; s < 8; ++s) {
            const int c = 8 * w + s;
            if (c >= kdim) break;
            if (c % Mm1) continue;
            const int n = c / Mm1;
            uint32_t dd[4];
            rsr::device_row_block(row, (uint32_t)(n >> 2), gen, K, dd);
            int x = 0;
            for (int k = 0; k < Mm1; ++k) {
              const int cc = c + k;
              if ((cc >> 3) == w) {
                x += (lo[0] >> (4 * (cc & 7) + 1)) & 1u;
              } else {
                uint32_t t;
                bool ok;
                column_threshold(probs, M, Mm1, cc, t, ok);
                x += ok && dd[n & 3] >= t;
              }
            }
            srow[n] = (uint8_t)x;
          }
        }
      }
    }
    if (fp4 && lane_on) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (u * R + rr >= prows) break;
        const uint32_t l = lo[u] | bias;
        uint8_t* prow = fp4 + (pr + u * R + rr) * row_stride;
        reinterpret_cast<uint32_t*>(prow)[w] = l ^ flip;
        reinterpret_cast<uint32_t*>(prow + plane)[w] = l;
      }
    }
    if (states) {
      __syncthreads();  // the pass's rows are staged (the other buffer is free again)
      // buf[sb + i] = global byte pr * N + i, with the same alignment mod 16
      uint8_t* g = states + pr * N;
      const int L = prows * N;
      const int head = min(L, (16 - sb) & 15);
      const int nvec = (L - head) >> 4;
      for (int i = threadIdx.x; i < nvec; i += blockDim.x)
        reinterpret_cast<uint4*>(g + head)[i] = reinterpret_cast<const uint4*>(buf + sb + head)[i];
      const int tail0 = head + (nvec << 4);
      const int t = threadIdx.x;
      if (t < head) g[t] = buf[sb + t];
      else if (t < head + (L - tail0)) g[tail0 + t - head] = buf[sb + tail0 + t - head];
    }
  }
}




__global__ void uniform_kernel(uint64_t seed, uint64_t gen, int64_t first, int64_t count,
                               int64_t b_lo, int64_t nblk, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nblk) return;
  const int64_t b = b_lo + t;
  uint64_t w[4];
  rsr::philox4x64_10((uint64_t)b + 1ull, seed, gen, w);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int64_t f = 4 * b + j;
    if (f >= first && f < first + count)
      out[f - first] = __dmul_rn((double)(w[j] >> 11), 1.1102230246251565e-16);  // 2^-53
  }
}

// A rows from states: A[i, n(M-1)+k-1] = [x_n < k]; bias columns = 1; zero pad.
__global__ void encode_samples_kernel(const uint8_t* __restrict__ states, int64_t count, int N,
                                      int M, int8_t* __restrict__ out, int ld, int kdim,
                                      int nbias) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * ld) return;
  const int64_t i = t / ld;
  const int c = (int)(t - i * ld);
  int8_t v;
  if (c < kdim) {
    const int n = c / (M - 1), k = c % (M - 1) + 1;
    v = (int8_t)(states[i * N + n] < k);
  } else {
    v = (int8_t)(c < kdim + nbias);
  }
  out[t] = v;
}

// B rows from reference states (see include/rsr_b200.h for the layout).
__global__ void encode_refs_kernel(const uint8_t* __restrict__ states, int64_t count,
                                   int64_t rows_total, int N, int M, int side,
                                   int8_t* __restrict__ out, int ld, int kdim, int nbias) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows_total) return;
  int8_t* row = out + r * (int64_t)ld;
  if (r >= count) {  // never-hit pad row: A.B = bias column 0 = 1
    for (int c = lane; c < ld; c += 32) row[c] = (int8_t)(c == kdim);
    return;
  }
  const uint8_t* x = states + r * (int64_t)N;
  int below = 0;  // c_r = #{(n,k) : r_n < k}
  for (int c = lane; c < kdim; c += 32) {
    const int n = c / (M - 1), k = c % (M - 1) + 1;
    const int lt = x[n] < k;
    if (side == RSR_SIDE_UPPER) {
      row[c] = (int8_t)(!lt);
    } else {
      row[c] = (int8_t)(-lt);
      below += lt;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) below += __shfl_xor_sync(0xffffffffu, below, o);
  for (int c = kdim + lane; c < ld; c += 32) {
    int v = 0;
    if (side == RSR_SIDE_LOWER && c < kdim + nbias) {
      const int j = c - kdim;
      const int rem = below - 127 * j;
      v = rem <= 0 ? 0 : (rem > 127 ? 127 : rem);
    }
    row[c] = (int8_t)v;
  }
}

// encoding.py:138-153 row layout: row-major N x M per item.
__global__ void encode_rows_kernel(const uint8_t* __restrict__ states, int64_t count, int N, int M,
                                   int kind, uint8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t L = (int64_t)N * M;
  if (t >= count * L) return;
  const int64_t i = t / L;
  const int j = (int)(t - i * L);
  const int n = j / M, m = j - n * M;
  const int x = states[i * N + n];
  out[t] = (uint8_t)(kind == 0 ? (m == x) : kind == 1 ? (m <= x) : (m >= x));
}

// np.packbits(axis=1): byte b holds bits 8b..8b+7, MSB first, zero padded.
__global__ void packbits_kernel(const uint8_t* __restrict__ rows, int64_t count, int L, int comp,
                                uint8_t* __restrict__ out) {
  const int nbytes = (L + 7) / 8;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * nbytes) return;
  const int64_t i = t / nbytes;
  const int b = (int)(t - i * nbytes);
  const uint8_t* r = rows + i * L;
  unsigned v = 0;
  for (int q = 0; q < 8; ++q) {
    const int j = 8 * b + q;
    unsigned bit = 0;
    if (j < L) bit = comp ? (r[j] == 0) : (r[j] != 0);
    v |= bit << (7 - q);
  }
  out[t] = (uint8_t)v;
}

}  // namespace

extern "C" int rsr_encode_rows(const uint8_t* states, int64_t count, int n_components,
                               int n_states, int kind, uint8_t* out, void* stream) {
  RSR_REQUIRE(n_components >= 1 && n_states >= 1 && count >= 0, "rsr_encode_rows: bad shape");
  RSR_REQUIRE(kind >= 0 && kind <= 2, "rsr_encode_rows: kind must be 0, 1 or 2");
  const int64_t total = count * n_components * n_states;
  if (total == 0) return RSR_OK;
  encode_rows_kernel<<<(unsigned)rsr::ceil_div(total, kThreads), kThreads, 0,
                       rsr::as_stream(stream)>>>(states, count, n_components, n_states, kind, out);
  return rsr::check_launch("encode_rows_kernel");
}

extern "C" int rsr_packbits_rows(const uint8_t* rows, int64_t count, int row_len, int complement,
                                 uint8_t* out, void* stream) {
  RSR_REQUIRE(row_len >= 0 && count >= 0, "rsr_packbits_rows: bad shape");
  const int64_t total = count * ((row_len + 7) / 8);
  if (total == 0) return RSR_OK;
  packbits_kernel<<<(unsigned)rsr::ceil_div(total, kThreads), kThreads, 0,
                    rsr::as_stream(stream)>>>(rows, count, row_len, complement, out);
  return rsr::check_launch("packbits_kernel");
}

extern "C" int rsr_philox_raw(uint64_t seed, uint64_t gen, int64_t first, int64_t count,
                              uint64_t* out, void* stream) {
  RSR_REQUIRE(first >= 0 && count >= 0, "rsr_philox_raw: negative range");
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(out != nullptr, "rsr_philox_raw: null output");
  const int64_t b_lo = first / 4, b_hi = (first + count - 1) / 4, nblk = b_hi - b_lo + 1;
  philox_raw_kernel<<<(unsigned)rsr::ceil_div(nblk, kThreads), kThreads, 0,
                      rsr::as_stream(stream)>>>(seed, gen, first, count, b_lo, nblk, out);
  return rsr::check_launch("philox_raw_kernel");
}

extern "C" int rsr_device_raw(uint64_t seed, uint64_t gen, int64_t start, int64_t count,
                              int n_components, uint32_t* out, void* stream) {
  RSR_REQUIRE(start >= 0 && count >= 0 && n_components >= 1, "rsr_device_raw: bad shape");
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(out != nullptr, "rsr_device_raw: null output");
  const int64_t total = count * ((n_components + 3) / 4);
  device_raw_kernel<<<(unsigned)rsr::ceil_div(total, kThreads), kThreads, 0,
                      rsr::as_stream(stream)>>>(seed, gen, start, count, n_components, out);
  return rsr::check_launch("device_raw_kernel");
}

extern "C" int rsr_uniform_field(uint64_t seed, uint64_t gen, int64_t start, int64_t count,
                                 int n_components, double* out, void* stream) {
  RSR_REQUIRE(start >= 0 && count >= 0 && n_components >= 1, "rsr_uniform_field: bad shape");
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(out != nullptr, "rsr_uniform_field: null output");
  const int64_t first = start * n_components, total = count * n_components;
  const int64_t b_lo = first / 4, b_hi = (first + total - 1) / 4, nblk = b_hi - b_lo + 1;
  uniform_kernel<<<(unsigned)rsr::ceil_div(nblk, kThreads), kThreads, 0,
                   rsr::as_stream(stream)>>>(seed, gen, first, total, b_lo, nblk, out);
  return rsr::check_launch("uniform_kernel");
}

extern "C" int rsr_sample_ex(const double* probs, int n_components, int n_states, uint64_t seed,
                             uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                             int8_t* out_thermo, int ld_thermo, int rng, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(rng == RSR_RNG_SHARED || rng == RSR_RNG_DEVICE, "rsr_sample: bad rng %d", rng);
  RSR_REQUIRE(N >= 1 && M >= 2 && M <= 255, "rsr_sample: need N >= 1 and 2 <= M <= 255");
  RSR_REQUIRE(start >= 0 && count >= 1, "rsr_sample: n_samples must be >= 1");
  RSR_REQUIRE(probs != nullptr, "rsr_sample: null probs");
  RSR_REQUIRE(out_states || out_thermo, "rsr_sample: no output requested");
  const int kdim = rsr::thermo_kdim(N, M), nbias = rsr::thermo_bias_cols(N, M);
  if (out_thermo)
    RSR_REQUIRE(ld_thermo >= rsr::thermo_kpad(N, M), "rsr_sample: ld_thermo < Kpad (%d)",
                rsr::thermo_kpad(N, M));
  const size_t smem = (size_t)N * (M - 1) * sizeof(unsigned long long);
  RSR_REQUIRE(smem <= 200 * 1024, "rsr_sample: N*(M-1) too large for the threshold table");
  auto kern = rng == RSR_RNG_DEVICE ? (M == 2 ? sample_kernel<true, 1> : sample_kernel<false, 1>)
                                    : (M == 2 ? sample_kernel<true, 0> : sample_kernel<false, 0>);
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t f0 = start * N, f1 = (start + count) * N;
  const int64_t b_lo = f0 / 4, b_hi = (f1 - 1) / 4, nblk = b_hi - b_lo + 1;
  const uint64_t magic = ~0ull / (uint64_t)N;  // floor((2^64 - 1) / N)
  kern<<<(unsigned)rsr::ceil_div(nblk, kThreads), kThreads, smem, rsr::as_stream(stream)>>>(
      probs, N, M, seed, gen, f0, f1, b_lo, nblk, out_states, out_thermo, ld_thermo, kdim, nbias,
      magic, start);
  return rsr::check_launch("sample_kernel");
}

extern "C" int rsr_sample(const double* probs, int n_components, int n_states, uint64_t seed,
                          uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                          int8_t* out_thermo, int ld_thermo, void* stream) {
  return rsr_sample_ex(probs, n_components, n_states, seed, gen, start, count, out_states,
                       out_thermo, ld_thermo, RSR_RNG_SHARED, stream);
}

extern "C" int rsr_encode_samples(const uint8_t* states, int64_t count, int n_components,
                                  int n_states, int8_t* out, int ld, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(N >= 1 && M >= 2 && count >= 0, "rsr_encode_samples: bad shape");
  RSR_REQUIRE(ld >= rsr::thermo_kpad(N, M) && ld % 16 == 0, "rsr_encode_samples: bad ld");
  if (count == 0) return RSR_OK;
  const int64_t total = count * ld;
  encode_samples_kernel<<<(unsigned)rsr::ceil_div(total, kThreads), kThreads, 0,
                          rsr::as_stream(stream)>>>(states, count, N, M, out, ld,
                                                    rsr::thermo_kdim(N, M),
                                                    rsr::thermo_bias_cols(N, M));
  return rsr::check_launch("encode_samples_kernel");
}

extern "C" int rsr_encode_refs(const uint8_t* states, int64_t count, int64_t rows_total,
                               int n_components, int n_states, int side, int8_t* out, int ld,
                               void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(N >= 1 && M >= 2 && count >= 0 && rows_total >= count, "rsr_encode_refs: bad shape");
  RSR_REQUIRE(side == RSR_SIDE_LOWER || side == RSR_SIDE_UPPER, "rsr_encode_refs: bad side");
  RSR_REQUIRE(ld >= rsr::thermo_kpad(N, M) && ld % 16 == 0, "rsr_encode_refs: bad ld");
  if (rows_total == 0) return RSR_OK;
  const int warps = kThreads / 32;
  encode_refs_kernel<<<(unsigned)rsr::ceil_div(rows_total, warps), kThreads, 0,
                       rsr::as_stream(stream)>>>(states, count, rows_total, N, M, side, out, ld,
                                                 rsr::thermo_kdim(N, M),
                                                 rsr::thermo_bias_cols(N, M));
  return rsr::check_launch("encode_refs_kernel");
}

namespace {
template <int RPC>
const void* rows_kernel_rpc(int M, bool c32) {
  if (c32)
    return M == 2   ? reinterpret_cast<const void*>(sample_rows_kernel<2, true, RPC>)
           : M == 3 ? reinterpret_cast<const void*>(sample_rows_kernel<3, true, RPC>)
                    : reinterpret_cast<const void*>(sample_rows_kernel<0, true, RPC>);
  return M == 2   ? reinterpret_cast<const void*>(sample_rows_kernel<2, false, RPC>)
         : M == 3 ? reinterpret_cast<const void*>(sample_rows_kernel<3, false, RPC>)
                  : reinterpret_cast<const void*>(sample_rows_kernel<0, false, RPC>);
}

const void* rows_kernel(int M, bool c32, int rpc) {
  return rpc == kRowsPerCta ? rows_kernel_rpc<kRowsPerCta>(M, c32) : rows_kernel_rpc<16>(M, c32);
}

int launch_dev_rows(const double* probs, int N, int M, uint64_t seed, uint64_t gen, int64_t start,
                    int64_t count, uint8_t* states, uint8_t* fp4, int row_bytes,
                    int64_t row_stride, int64_t plane, cudaStream_t st) {
  const void* kern = M == 2   ? reinterpret_cast<const void*>(sample_dev_rows_kernel<2>)
                     : M == 3 ? reinterpret_cast<const void*>(sample_dev_rows_kernel<3>)
                              : reinterpret_cast<const void*>(sample_dev_rows_kernel<0>);
  // FP4 words per row (both halves share them): all row_bytes / 4 when the operand is
  // written (padding words are zero), else just those holding components
  int words = fp4 ? row_bytes / 4 : (N * (M - 1) + 7) / 8;
  RSR_REQUIRE(words <= 1024, "rsr_sample_fp4: N*(M-1) too large for the device-stream sampler");
  // R rows per pass: the thread count words * R rounded up to whole warps wastes the
  // fewest lanes (ties: the larger CTA up to 512 threads)
  // (measured, N = 295: 160-thread CTAs beat 480-thread ones by 15-30%)
  int R = 1;
  double best = -1e9;
  for (int r = 1; r * words <= 1024; ++r) {
    const int th = (r * words + 31) / 32 * 32;
    const double score = (double)(r * words) / th - 0.0005 * th - (th < 128 ? 0.2 : 0.0);
    if (score > best) {
      best = score;
      R = r;
    }
  }
  const int threads = (R * words + 31) / 32 * 32;
  // 32 rows per CTA: short-lived CTAs, so the Stage-1 loop's high-priority kernels
  // (searches, insertion) find SM space within a few microseconds while a prefetched
  // batch is drawn on the low-priority stream (cfg3 loop on this stream: 0.117 s with
  // 128-row CTAs, 0.0965 s with 32; the sampler alone is 10 % slower: every CTA derives
  // its column constants once).  M = 2, 3 threads take two rows per pass.
  // RSR_DEVROWS_CTA_ROWS overrides (experiments).
  const int U = (M == 2 || M == 3) ? 2 : 1;
  static const int cta_rows = [] {
    const char* e = getenv("RSR_DEVROWS_CTA_ROWS");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  const int passes = std::max(1, cta_rows / (U * R));
  const int64_t grid = rsr::ceil_div(count, (int64_t)U * R * passes);
  const rsr::Philox32Keys keys = rsr::device_keys(seed, gen);
  void* args[] = {(void*)&probs, (void*)&N,      (void*)&M,     (void*)&keys,
                  (void*)&gen,   (void*)&start,  (void*)&count, (void*)&states,
                  (void*)&fp4,   (void*)&words,  (void*)&R,     (void*)&passes,
                  (void*)&row_stride, (void*)&plane};
  const size_t smem = states ? 2 * (size_t)((U * R * N + 16 + 15) & ~15) : 0;
  if (smem > 48 * 1024) {
    const int rc = rsr::ensure_dynamic_smem(kern, smem);
    if (rc) return rc;
  }
  RSR_CUDA(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(threads), args, smem, st));
  return rsr::check_launch("sample_dev_rows_kernel");
}
}  // namespace

extern "C" int rsr_sample_fp4_ex(const double* probs, int n_components, int n_states,
                                 uint64_t seed, uint64_t gen, int64_t start, int64_t count,
                                 uint8_t* out_states, uint8_t* out_fp4, int row_bytes,
                                 int64_t fp4_plane_stride, int rng, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(rng == RSR_RNG_SHARED || rng == RSR_RNG_DEVICE, "rsr_sample_fp4: bad rng %d", rng);
  RSR_REQUIRE(N >= 1 && M >= 2 && M <= 255, "rsr_sample_fp4: need N >= 1 and 2 <= M <= 255");
  RSR_REQUIRE(start >= 0 && count >= 1, "rsr_sample_fp4: n_samples must be >= 1");
  RSR_REQUIRE(probs != nullptr, "rsr_sample_fp4: null probs");
  RSR_REQUIRE(out_states || out_fp4, "rsr_sample_fp4: no output requested");
  if (out_fp4)
    RSR_REQUIRE(row_bytes == rsr_fp4_row_bytes(N, M), "rsr_sample_fp4: row_bytes must be %d",
                rsr_fp4_row_bytes(N, M));
  if (out_states)
    RSR_REQUIRE((reinterpret_cast<uintptr_t>(out_states) & 15) == 0,
                "rsr_sample_fp4: out_states must be 16-byte aligned");
  if (out_fp4)
    RSR_REQUIRE((reinterpret_cast<uintptr_t>(out_fp4) & 15) == 0,
                "rsr_sample_fp4: out_fp4 must be 16-byte aligned");
  // FP4 operand layout: interleaved rows [A_up | A_lo] (plane stride 0), or planar --
  // A_up rows of row_bytes, the A_lo plane fp4_plane_stride bytes further
  RSR_REQUIRE(fp4_plane_stride == 0 ||
                  (fp4_plane_stride % 16 == 0 && fp4_plane_stride >= count * (int64_t)row_bytes),
              "rsr_sample_fp4: fp4_plane_stride must be 0 or a multiple of 16 >= count*row_bytes");
  const int64_t fp4_row_stride = fp4_plane_stride ? row_bytes : 2 * (int64_t)row_bytes;
  const int64_t fp4_plane = fp4_plane_stride ? fp4_plane_stride : row_bytes;
  if (rng == RSR_RNG_DEVICE)
    return launch_dev_rows(probs, N, M, seed, gen, start, count, out_states, out_fp4, row_bytes,
                           fp4_row_stride, fp4_plane, rsr::as_stream(stream));
  // 64-row chunks, or 16-row ones when two 64-row staging buffers do not fit
  const size_t t_bytes = ((size_t)(N + kTExtra) * (M - 1) * sizeof(unsigned long long) + 15) / 16 * 16;
  int rpc = kRowsPerCta;
  if (t_bytes + 2 * (size_t)((kRowsPerCta * N + 16 + 15) / 16 * 16) > 200 * 1024) rpc = 16;
  const int st_bytes = (rpc * N + 16 + 15) / 16 * 16;  // + funnel-load slack
  const size_t smem = t_bytes + 2 * (size_t)st_bytes;
  RSR_REQUIRE(smem <= 200 * 1024, "rsr_sample_fp4: N*(M-1) too large for shared memory");
  const bool c32 = ((start + count) * (int64_t)N + 3) / 4 + 1 < ((int64_t)1 << 32);
  const void* kern = rows_kernel(M, c32, rpc);
  if (smem > 48 * 1024) {
    const int rc = rsr::ensure_dynamic_smem(kern, smem);
    if (rc) return rc;
  }
  int dev = 0, sms = 0, per_sm = 0;
  RSR_CUDA(cudaGetDevice(&dev));
  RSR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RSR_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRowThreads, smem));
  // CTAs walk a bounded number of chunks: short-lived CTAs let the Stage-1
  // loop's high-priority kernels take SMs while a prefetched batch is drawn
  // on the low-priority stream (a persistent grid would hold every SM)
  static const int cpc = [] {
    const char* e = getenv("RSR_SAMPLE_CPC");
    return e ? std::max(1, atoi(e)) : kChunksPerCta;
  }();
  const int64_t chunks = rsr::ceil_div(count, rpc);
  const int64_t grid = std::max<int64_t>(std::min<int64_t>(chunks, (int64_t)sms * std::max(per_sm, 1)),
                                         rsr::ceil_div(chunks, cpc));
  void* args[] = {(void*)&probs,     (void*)&N,         (void*)&M,
                  (void*)&seed,      (void*)&gen,       (void*)&start,
                  (void*)&count,     (void*)&out_states, (void*)&out_fp4,
                  (void*)&row_bytes, (void*)&st_bytes,  (void*)&fp4_row_stride,
                  (void*)&fp4_plane};
  RSR_CUDA(cudaLaunchKernel(kern, dim3((unsigned)grid), dim3(kRowThreads), args, smem,
                            rsr::as_stream(stream)));
  return rsr::check_launch("sample_rows_kernel");
}

extern "C" int rsr_sample_fp4(const double* probs, int n_components, int n_states, uint64_t seed,
                              uint64_t gen, int64_t start, int64_t count, uint8_t* out_states,
                              uint8_t* out_fp4, int row_bytes, void* stream) {
  return rsr_sample_fp4_ex(probs, n_components, n_states, seed, gen, start, count, out_states,
                           out_fp4, row_bytes, 0, RSR_RNG_SHARED, stream);
}
