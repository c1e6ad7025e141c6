// Support compaction of the FP4 thermometer contraction.
//
// D[s, r] = sum_c A[s, c] * B[r, c] counts the thermometer columns c where
// reference r requires a level sample s does not reach (upper side, classify.py:42-44
// on the encodings of encoding.py:138-153; the lower side symmetrically).  A column
// in which no reference row of a side is 1 adds 0 to every D of that side, so
// dropping it leaves every count -- hence every label, first match and violation
// count -- unchanged.  The s-t path references of BASELINE configs[3] touch only
// ~213 of the 295 edges (an edge on no shortest s-t path never appears), so the
// contraction shrinks from 5 to 4 K-steps of 64 columns (row_bytes 160 -> 128).
//
//   rsr_fp4_or_rows        OR of the reference rows of a side (the column support),
//                          one row of 32-bit words; the host turns it into a column map.
//   rsr_fp4_gather_columns dst column j = src column cols[j] (j < n_cols), 0 past it:
//                          the same map applies to the reference rows and to either
//                          sample plane, with the bias column kdim as its last entry
//                          (1 in every sample row, 0 in real reference rows, 1 in pad
//                          rows -- so pad rows stay never-hit).
#include "common.cuh"

namespace {

// One block ORs a strided slice of the rows in registers (one 32-bit word per thread
// and row-column), then one atomicOr per word.
__global__ void __launch_bounds__(256) or_rows_kernel(const uint32_t* __restrict__ B,
                                                      int64_t rows, int words,
                                                      uint32_t* __restrict__ out) {
  const int rows_per_pass = blockDim.x / words;
  if (rows_per_pass == 0) return;
  const int w = threadIdx.x % words, rr = threadIdx.x / words;
  if (rr >= rows_per_pass) return;
  uint32_t acc = 0;
  for (int64_t r = (int64_t)blockIdx.x * rows_per_pass + rr; r < rows;
       r += (int64_t)gridDim.x * rows_per_pass)
    acc |= B[r * words + w];
  if (acc) atomicOr(out + w, acc);
}

// A block converts kGatherRows rows.  The source rows are staged in shared memory with
// a stride of row_bytes + 4 (an odd number of 32-bit words, so the 32 lanes of a warp --
// 32 rows at the same column -- hit 32 different banks); the extra word is 0 and the
// map's pad entries point at it.  The global loads are issued in batches of kBatch
// 16-byte vectors per thread before any is stored (a load -> store loop keeps one
// vector in flight per thread: 1.2 TB/s).  A warp owns one 16-byte output chunk (32
// columns) at a time: its 32 map entries (word, shift) sit in registers while the lanes
// walk the rows, one 32-bit shared load, shift and mask per column.  Output rows are
// assembled in shared memory (stride row_bytes + 16: conflict-free 16-byte stores) and
// leave with coalesced 16-byte stores.
constexpr int kGatherRows = 128;
constexpr int kBatch = 8;

__global__ void __launch_bounds__(256, 3) gather_columns_kernel(
    const uint8_t* __restrict__ src, int64_t src_stride, int64_t count, int src_row_bytes,
    const int32_t* __restrict__ cols, int n_cols, uint8_t* __restrict__ dst, int64_t dst_stride,
    int dst_row_bytes) {
  extern __shared__ __align__(16) uint32_t sm32[];
  const int sw = src_row_bytes / 4 + 1;   // staged source row stride in words (odd)
  const int dw = dst_row_bytes / 4 + 4;   // staged output row stride in words
  uint32_t* outs = sm32;                                         // [kGatherRows * dw]
  int32_t* map = reinterpret_cast<int32_t*>(sm32 + kGatherRows * dw);  // [2 * dst_row_bytes]
  uint32_t* rows = sm32 + kGatherRows * dw + 2 * dst_row_bytes;  // [kGatherRows * sw]
  const int dst_cols = 2 * dst_row_bytes;
  for (int j = threadIdx.x; j < dst_cols; j += blockDim.x) {
    const int c = j < n_cols ? cols[j] : -1;
    map[j] = c < 0 ? (sw - 1) << 8 : ((c >> 3) << 8) | ((c & 7) * 4);
  }
  const int64_t r0 = (int64_t)blockIdx.x * kGatherRows;
  const int nr = (int)(count - r0 < kGatherRows ? count - r0 : kGatherRows);
  const int vec_per_row = src_row_bytes / 16;
  const int nvec = nr * vec_per_row;
  for (int base = 0; base < nvec; base += kBatch * blockDim.x) {
    uint4 x[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int v = base + b * blockDim.x + threadIdx.x;
      if (v < nvec) {
        const int r = v / vec_per_row, q = v - r * vec_per_row;
        x[b] = __ldcs(reinterpret_cast<const uint4*>(src + (r0 + r) * src_stride) + q);
      }
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int v = base + b * blockDim.x + threadIdx.x;
      if (v < nvec) {
        const int r = v / vec_per_row, q = v - r * vec_per_row;
        uint32_t* d = rows + r * sw + 4 * q;
        d[0] = x[b].x;
        d[1] = x[b].y;
        d[2] = x[b].z;
        d[3] = x[b].w;
      }
    }
  }
  for (int r = threadIdx.x; r < nr; r += blockDim.x) rows[r * sw + sw - 1] = 0u;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int chunks = dst_row_bytes / 16;
  for (int q = warp; q < chunks; q += blockDim.x / 32) {
    int32_t m[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) m[e] = map[32 * q + e];
    for (int r = lane; r < nr; r += 32) {
      const uint32_t* row = rows + r * sw;
      uint32_t w[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t v = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int me = m[8 * k + e];
          v |= ((row[me >> 8] >> (me & 31)) & 0xFu) << (4 * e);
        }
        w[k] = v;
      }
      *reinterpret_cast<uint4*>(outs + r * dw + 4 * q) = make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  __syncthreads();
  for (int v = threadIdx.x; v < nr * chunks; v += blockDim.x) {
    const int r = v / chunks, q = v - r * chunks;
    *reinterpret_cast<uint4*>(dst + (r0 + r) * dst_stride + 16 * q) =
        *reinterpret_cast<const uint4*>(outs + r * dw + 4 * q);
  }
}

}  // namespace

extern "C" int rsr_fp4_or_rows(const uint8_t* B, int64_t rows, int row_bytes, uint32_t* out,
                               void* stream) {
  RSR_REQUIRE(rows >= 0 && row_bytes >= 4 && row_bytes % 4 == 0 && row_bytes <= 1024,
              "rsr_fp4_or_rows: bad shape");
  RSR_REQUIRE(out != nullptr && (rows == 0 || B != nullptr), "rsr_fp4_or_rows: null pointer");
  RSR_REQUIRE((reinterpret_cast<uintptr_t>(B) & 3) == 0 && (reinterpret_cast<uintptr_t>(out) & 3) == 0,
              "rsr_fp4_or_rows: pointers must be 4-byte aligned");
  cudaStream_t st = rsr::as_stream(stream);
  RSR_CUDA(cudaMemsetAsync(out, 0, row_bytes, st));
  if (rows == 0) return RSR_OK;
  const int words = row_bytes / 4;
  const int rows_per_pass = 256 / words;
  int64_t grid = rsr::ceil_div(rows, (int64_t)rows_per_pass * 16);
  if (grid > 148 * 8) grid = 148 * 8;
  or_rows_kernel<<<(unsigned)grid, 256, 0, st>>>(reinterpret_cast<const uint32_t*>(B), rows,
                                                  words, out);
  return rsr::check_launch("or_rows_kernel");
}

extern "C" int rsr_fp4_gather_columns(const uint8_t* src, int64_t src_stride, int64_t count,
                                      int src_row_bytes, const int32_t* cols, int n_cols,
                                      uint8_t* dst, int64_t dst_stride, int dst_row_bytes,
                                      void* stream) {
  RSR_REQUIRE(count >= 0, "rsr_fp4_gather_columns: negative count");
  RSR_REQUIRE(src_row_bytes >= 16 && src_row_bytes % 16 == 0 && src_row_bytes <= RSR_FP4_MAX_ROW_BYTES &&
                  dst_row_bytes >= 16 && dst_row_bytes % 16 == 0 && dst_row_bytes <= RSR_FP4_MAX_ROW_BYTES,
              "rsr_fp4_gather_columns: row bytes must be multiples of 16 in [16, 768]");
  RSR_REQUIRE(n_cols >= 0 && n_cols <= 2 * dst_row_bytes,
              "rsr_fp4_gather_columns: n_cols must lie in [0, 2*dst_row_bytes]");
  RSR_REQUIRE(src_stride >= src_row_bytes && src_stride % 16 == 0 && dst_stride >= dst_row_bytes &&
                  dst_stride % 16 == 0,
              "rsr_fp4_gather_columns: strides must be multiples of 16 >= the row bytes");
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(src && dst && (n_cols == 0 || cols), "rsr_fp4_gather_columns: null pointer");
  RSR_REQUIRE((reinterpret_cast<uintptr_t>(src) & 15) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0,
              "rsr_fp4_gather_columns: src and dst must be 16-byte aligned");
  const size_t smem = 4 * ((size_t)kGatherRows * (dst_row_bytes / 4 + 4) +
                           2 * (size_t)dst_row_bytes +
                           (size_t)kGatherRows * (src_row_bytes / 4 + 1));
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(gather_columns_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = rsr::ceil_div(count, (int64_t)kGatherRows);
  RSR_REQUIRE(grid < (int64_t)1 << 31, "rsr_fp4_gather_columns: count too large");
  gather_columns_kernel<<<(unsigned)grid, 256, smem, rsr::as_stream(stream)>>>(
      src, src_stride, count, src_row_bytes, cols, n_cols, dst, dst_stride, dst_row_bytes);
  return rsr::check_launch("gather_columns_kernel");
}
