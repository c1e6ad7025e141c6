// (2) Bit-packed CUDA-core dominance classifier (comparison variant), label
// finalisation, order-preserving compaction and the full violation matrix.
//
// Replaces classify.py:42-44 (_violation_block_packed), 57-96
// (violation_counts), 99-148 (_chunk_hits/_hits_for incl. first match) and
// 240-245 (precedence + np.flatnonzero).
//
// Thermometer bits: sample a_c = [x_n < k]; upper ref u_c = [r_n >= k];
// lower ref l_c = [r_n < k].  Violations exist iff OR_c(a_c & u_c) != 0
// (upper) or OR_c(~a_c & l_c) != 0 (lower): one LOP3 per 32 positions, no
// popcount needed for the any-zero test.
#include "common.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kSPT = 4;       // samples per thread (amortises the shared-memory broadcast)
constexpr int kTileRefs = 256;

__global__ void pack_bits_kernel(const uint8_t* __restrict__ states, int64_t count, int N, int M,
                                 int invert, uint32_t* __restrict__ out, int words) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * words) return;
  const int64_t i = t / words;
  const int w = (int)(t - i * words);
  const int kdim = N * (M - 1);
  const uint8_t* x = states + i * N;
  uint32_t v = 0;
  for (int b = 0; b < 32; ++b) {
    const int c = w * 32 + b;
    if (c >= kdim) break;
    const int n = c / (M - 1), k = c % (M - 1) + 1;
    const int lt = x[n] < k;
    v |= (uint32_t)(invert ? !lt : lt) << b;
  }
  out[t] = v;
}

template <int W, bool FIRST>
__global__ void __launch_bounds__(kThreads)
classify_bits_kernel(const uint32_t* __restrict__ sbits, int64_t S,
                     const uint32_t* __restrict__ lbits, int64_t nl,
                     const uint32_t* __restrict__ ubits, int64_t nu, uint8_t* __restrict__ flags,
                     int64_t* __restrict__ first_l, int64_t* __restrict__ first_u, int acc) {
  __shared__ uint32_t tile[kTileRefs * W];
  const int64_t s0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * kSPT;
  uint32_t a[kSPT][W];
#pragma unroll
  for (int q = 0; q < kSPT; ++q)
#pragma unroll
    for (int w = 0; w < W; ++w) a[q][w] = (s0 + q < S) ? sbits[(s0 + q) * W + w] : 0u;
  uint32_t hit[kSPT];
  int64_t fst[2][kSPT];
#pragma unroll
  for (int q = 0; q < kSPT; ++q) {
    hit[q] = 0;
    fst[0][q] = fst[1][q] = -1;
  }
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    const uint32_t* refs = side ? ubits : lbits;
    const int64_t n = side ? nu : nl;
    for (int64_t r0 = 0; r0 < n; r0 += kTileRefs) {
      const int cnt = (int)(n - r0 < kTileRefs ? n - r0 : kTileRefs);
      __syncthreads();
      for (int i = threadIdx.x; i < cnt * W; i += blockDim.x) tile[i] = refs[r0 * W + i];
      __syncthreads();
      for (int r = 0; r < cnt; ++r) {
        uint32_t b[W];
#pragma unroll
        for (int w = 0; w < W; ++w) b[w] = tile[r * W + w];
#pragma unroll
        for (int q = 0; q < kSPT; ++q) {
          uint32_t v = 0;
#pragma unroll
          for (int w = 0; w < W; ++w) v |= (side ? a[q][w] : ~a[q][w]) & b[w];
          if (v == 0) {
            hit[q] |= side ? RSR_HIT_UPPER : RSR_HIT_LOWER;
            if (FIRST && fst[side][q] < 0) fst[side][q] = r0 + r;
          }
        }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kSPT; ++q) {
    const int64_t s = s0 + q;
    if (s < S) {
      flags[s] = (uint8_t)((acc ? flags[s] : 0) | hit[q]);
      if (FIRST) {
        if (first_l) first_l[s] = fst[0][q];
        if (first_u) first_u[s] = fst[1][q];
      }
    }
  }
}

// Any row width: one thread per sample, words streamed from global memory (L1
// caches the sample row; reference rows are read by every thread of the warp
// at the same address, i.e. broadcast).
__global__ void classify_bits_wide_kernel(const uint32_t* __restrict__ sbits, int64_t S,
                                          const uint32_t* __restrict__ lbits, int64_t nl,
                                          const uint32_t* __restrict__ ubits, int64_t nu,
                                          int W, uint8_t* __restrict__ flags,
                                          int64_t* __restrict__ first_l,
                                          int64_t* __restrict__ first_u, int acc) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= S) return;
  const uint32_t* a = sbits + s * W;
  uint32_t hit = 0;
  int64_t fst[2] = {-1, -1};
  for (int side = 0; side < 2; ++side) {
    const uint32_t* refs = side ? ubits : lbits;
    const int64_t n = side ? nu : nl;
    for (int64_t r = 0; r < n; ++r) {
      const uint32_t* b = refs + r * W;
      uint32_t v = 0;
      for (int w = 0; w < W && !v; ++w) v |= (side ? a[w] : ~a[w]) & b[w];
      if (v == 0) {
        hit |= side ? RSR_HIT_UPPER : RSR_HIT_LOWER;
        if (fst[side] < 0) fst[side] = r;
      }
    }
  }
  flags[s] = (uint8_t)((acc ? flags[s] : 0) | hit);
  if (first_l) first_l[s] = fst[0];
  if (first_u) first_u[s] = fst[1];
}

__global__ void finalize_kernel(const uint8_t* __restrict__ flags, int64_t S,
                                uint8_t* __restrict__ labels, unsigned long long* counts) {
  __shared__ unsigned long long bc[4];
  if (threadIdx.x < 4) bc[threadIdx.x] = 0;
  __syncthreads();
  unsigned long long c[4] = {0, 0, 0, 0};
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < S;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint8_t f = flags[i];
    const uint8_t lab = (f & RSR_HIT_LOWER) ? RSR_LABEL_LOWER
                        : (f & RSR_HIT_UPPER) ? RSR_LABEL_UPPER
                                              : RSR_LABEL_UNCLASSIFIED;
    if (labels) labels[i] = lab;
    c[lab] += 1;
    c[3] += (f == (RSR_HIT_LOWER | RSR_HIT_UPPER));
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    unsigned long long v = c[j];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&bc[j], v);
  }
  __syncthreads();
  if (threadIdx.x < 4 && bc[threadIdx.x]) atomicAdd(&counts[threadIdx.x], bc[threadIdx.x]);
}

// ---- order-preserving compaction (3 passes over tiles of kCTile elements)
constexpr int kCPer = 16;
constexpr int kCTile = kThreads * kCPer;

__global__ void compact_count_kernel(const uint8_t* __restrict__ labels, int64_t S, int label,
                                     int64_t* __restrict__ tile_counts) {
  const int64_t base = (int64_t)blockIdx.x * kCTile;
  int c = 0;
  for (int j = 0; j < kCPer; ++j) {
    const int64_t i = base + (int64_t)j * kThreads + threadIdx.x;
    c += (i < S && labels[i] == label);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  __shared__ int ws[kThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
    tile_counts[blockIdx.x] = t;
  }
}

__global__ void compact_scan_kernel(int64_t* __restrict__ tile_counts, int64_t ntiles,
                                    int64_t* __restrict__ out_count) {
  // single block, 1024 threads: exclusive scan in chunks
  __shared__ int64_t carry;
  __shared__ int64_t ws[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t b0 = 0; b0 < ntiles; b0 += blockDim.x) {
    const int64_t i = b0 + threadIdx.x;
    int64_t v = i < ntiles ? tile_counts[i] : 0;
    int64_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t z = lane < (int)(blockDim.x >> 5) ? ws[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(0xffffffffu, z, o);
        if (lane >= o) z += y;
      }
      ws[lane] = z;
    }
    __syncthreads();
    const int64_t incl = x + (w ? ws[w - 1] : 0) + carry;
    if (i < ntiles) tile_counts[i] = incl - v;
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) *out_count = carry;
}

__global__ void compact_write_kernel(const uint8_t* __restrict__ labels, int64_t S, int label,
                                     const int64_t* __restrict__ tile_offsets,
                                     int64_t* __restrict__ out_idx) {
  // thread t owns elements base + t*kCPer .. +kCPer-1 (contiguous) to keep order
  const int64_t base = (int64_t)blockIdx.x * kCTile + (int64_t)threadIdx.x * kCPer;
  int c = 0;
  for (int j = 0; j < kCPer; ++j) {
    const int64_t i = base + j;
    c += (i < S && labels[i] == label);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  __shared__ int ws[kThreads / 32];
  if (lane == 31) ws[w] = x;
  __syncthreads();
  int pre = 0;
  for (int k = 0; k < w; ++k) pre += ws[k];
  int64_t pos = tile_offsets[blockIdx.x] + pre + x - c;
  for (int j = 0; j < kCPer; ++j) {
    const int64_t i = base + j;
    if (i < S && labels[i] == label) out_idx[pos++] = i;
  }
}

__global__ void violation_kernel(const uint8_t* __restrict__ xs, int64_t H,
                                 const uint8_t* __restrict__ rs, int64_t R, int N, int side,
                                 int32_t* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t h = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (r >= R || h >= H) return;
  const uint8_t* x = xs + h * N;
  const uint8_t* ref = rs + r * N;
  int v = 0;
  for (int n = 0; n < N; ++n) v += side == RSR_SIDE_LOWER ? (x[n] > ref[n]) : (x[n] < ref[n]);
  out[h * R + r] = v;
}

__global__ void violation_rows_kernel(const uint8_t* __restrict__ xs, int64_t H,
                                      const uint8_t* __restrict__ rs, int64_t R, int L,
                                      int32_t* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t h = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (r >= R || h >= H) return;
  const uint8_t* x = xs + h * L;
  const uint8_t* ref = rs + r * L;
  int v = 0;
  for (int j = 0; j < L; ++j) v += (x[j] != 0) & (ref[j] == 0);
  out[h * R + r] = v;
}

template <int W>
int launch_bits(const uint32_t* sb, int64_t S, const uint32_t* lb, int64_t nl, const uint32_t* ub,
                int64_t nu, uint8_t* flags, int64_t* fl, int64_t* fu, int acc, cudaStream_t st) {
  const unsigned grid = (unsigned)rsr::ceil_div(S, (int64_t)kThreads * kSPT);
  if (fl || fu)
    classify_bits_kernel<W, true><<<grid, kThreads, 0, st>>>(sb, S, lb, nl, ub, nu, flags, fl, fu,
                                                             acc);
  else
    classify_bits_kernel<W, false><<<grid, kThreads, 0, st>>>(sb, S, lb, nl, ub, nu, flags,
                                                              nullptr, nullptr, acc);
  return rsr::check_launch("classify_bits_kernel");
}

}  // namespace

extern "C" int rsr_pack_thermo_bits(const uint8_t* states, int64_t count, int n_components,
                                    int n_states, int invert, uint32_t* out, int words,
                                    void* stream) {
  RSR_REQUIRE(n_components >= 1 && n_states >= 2 && count >= 0, "rsr_pack_thermo_bits: bad shape");
  RSR_REQUIRE((int64_t)words * 32 >= (int64_t)n_components * (n_states - 1),
              "rsr_pack_thermo_bits: words too small");
  if (count == 0) return RSR_OK;
  const int64_t total = count * words;
  pack_bits_kernel<<<(unsigned)rsr::ceil_div(total, kThreads), kThreads, 0,
                     rsr::as_stream(stream)>>>(states, count, n_components, n_states, invert, out,
                                               words);
  return rsr::check_launch("pack_bits_kernel");
}

extern "C" int rsr_classify_bits(const uint32_t* sample_bits, int64_t S,
                                 const uint32_t* lower_bits, int64_t n_lower,
                                 const uint32_t* upper_bits, int64_t n_upper, int words,
                                 uint8_t* flags, int64_t* first_lower, int64_t* first_upper,
                                 int accumulate, void* stream) {
  RSR_REQUIRE(S >= 0 && n_lower >= 0 && n_upper >= 0, "rsr_classify_bits: negative size");
  RSR_REQUIRE(words >= 1, "rsr_classify_bits: words >= 1");
  if (S == 0) return RSR_OK;
  cudaStream_t st = rsr::as_stream(stream);
  if (words > 32) {  // wide rows (N(M-1) > 1024): generic-width kernel
    const unsigned grid = (unsigned)rsr::ceil_div(S, 128);
    classify_bits_wide_kernel<<<grid, 128, 0, st>>>(sample_bits, S, lower_bits, n_lower, upper_bits,
                                                    n_upper, words, flags, first_lower,
                                                    first_upper, accumulate);
    return rsr::check_launch("classify_bits_wide_kernel");
  }
  switch (words) {
#define RSR_W(w) \
  case w:        \
    return launch_bits<w>(sample_bits, S, lower_bits, n_lower, upper_bits, n_upper, flags, \
                          first_lower, first_upper, accumulate, st);
    RSR_W(1) RSR_W(2) RSR_W(3) RSR_W(4) RSR_W(5) RSR_W(6) RSR_W(7) RSR_W(8)
    RSR_W(9) RSR_W(10) RSR_W(11) RSR_W(12) RSR_W(13) RSR_W(14) RSR_W(15) RSR_W(16)
    RSR_W(17) RSR_W(18) RSR_W(19) RSR_W(20) RSR_W(21) RSR_W(22) RSR_W(23) RSR_W(24)
    RSR_W(25) RSR_W(26) RSR_W(27) RSR_W(28) RSR_W(29) RSR_W(30) RSR_W(31) RSR_W(32)
#undef RSR_W
  }
  return RSR_EINVAL;
}

extern "C" int rsr_finalize(const uint8_t* flags, int64_t S, uint8_t* labels, int64_t* counts,
                            void* stream) {
  RSR_REQUIRE(S >= 0 && counts != nullptr, "rsr_finalize: bad arguments");
  cudaStream_t st = rsr::as_stream(stream);
  RSR_CUDA(cudaMemsetAsync(counts, 0, 4 * sizeof(int64_t), st));
  if (S == 0) return RSR_OK;
  int64_t blocks = rsr::ceil_div(S, kThreads);
  if (blocks > 148 * 8) blocks = 148 * 8;
  finalize_kernel<<<(unsigned)blocks, kThreads, 0, st>>>(
      flags, S, labels, reinterpret_cast<unsigned long long*>(counts));
  return rsr::check_launch("finalize_kernel");
}

extern "C" int64_t rsr_compact_scratch(int64_t S) { return rsr::ceil_div(S, kCTile) + 1; }

extern "C" int rsr_compact(const uint8_t* labels, int64_t S, int label, int64_t* out_idx,
                           int64_t* out_count, int64_t* scratch, void* stream) {
  RSR_REQUIRE(S >= 0 && out_count && scratch, "rsr_compact: bad arguments");
  cudaStream_t st = rsr::as_stream(stream);
  if (S == 0) {
    RSR_CUDA(cudaMemsetAsync(out_count, 0, sizeof(int64_t), st));
    return RSR_OK;
  }
  const int64_t ntiles = rsr::ceil_div(S, kCTile);
  compact_count_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(labels, S, label, scratch);
  int rc = rsr::check_launch("compact_count_kernel");
  if (rc) return rc;
  compact_scan_kernel<<<1, 1024, 0, st>>>(scratch, ntiles, out_count);
  rc = rsr::check_launch("compact_scan_kernel");
  if (rc) return rc;
  if (!out_idx) return RSR_OK;
  compact_write_kernel<<<(unsigned)ntiles, kThreads, 0, st>>>(labels, S, label, scratch, out_idx);
  return rsr::check_launch("compact_write_kernel");
}

extern "C" int rsr_violation_counts(const uint8_t* samples, int64_t H, const uint8_t* refs,
                                    int64_t R, int n_components, int side, int32_t* out,
                                    void* stream) {
  RSR_REQUIRE(H >= 0 && R >= 0 && n_components >= 1, "rsr_violation_counts: bad shape");
  RSR_REQUIRE(side == RSR_SIDE_LOWER || side == RSR_SIDE_UPPER, "rsr_violation_counts: bad side");
  if (H == 0 || R == 0) return RSR_OK;
  dim3 grid((unsigned)rsr::ceil_div(R, 128), (unsigned)(H < 65535 ? H : 65535),
            (unsigned)rsr::ceil_div(H, 65535));
  violation_kernel<<<grid, 128, 0, rsr::as_stream(stream)>>>(samples, H, refs, R, n_components,
                                                             side, out);
  return rsr::check_launch("violation_kernel");
}

extern "C" int rsr_violation_counts_rows(const uint8_t* sample_rows, int64_t H,
                                         const uint8_t* ref_rows, int64_t R, int row_len,
                                         int32_t* out, void* stream) {
  RSR_REQUIRE(H >= 0 && R >= 0 && row_len >= 0, "rsr_violation_counts_rows: bad shape");
  if (H == 0 || R == 0) return RSR_OK;
  dim3 grid((unsigned)rsr::ceil_div(R, 128), (unsigned)(H < 65535 ? H : 65535),
            (unsigned)rsr::ceil_div(H, 65535));
  violation_rows_kernel<<<grid, 128, 0, rsr::as_stream(stream)>>>(sample_rows, H, ref_rows, R,
                                                                  row_len, out);
  return rsr::check_launch("violation_rows_kernel");
}
