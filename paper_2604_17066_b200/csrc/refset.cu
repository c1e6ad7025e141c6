// (4) Device-resident reference sets for the Stage-1 loop: the insertion
// semantics of ReferenceSet.insert (boundary.py:87-108, _redundant_under
// :50-54) applied to a batch of boundary-search results without a host round
// trip, so the loop can enqueue iteration i's insertion and iteration i+1's
// classification back to back and read the outcome one iteration later.
//
// Dominance is tested on the FP4 operand rows the classifier streams: with
// E = [r_n >= k] (upper set) or [r_n < k] (lower set) as e2m1 nibbles,
//   candidate c redundant under member m  <=>  E_m & ~E_c == 0
// on both sides (upper: c >= m componentwise <=> every [m_n >= k] bit is set
// in c; lower: c <= m <=> every [m_n < k] bit is set in c), so a pair costs a
// few 16-byte AND-NOTs instead of N byte compares.
//
// Members are never physically removed during the loop: a dropped member is
// flagged dead (alive[m] = 0).  Classification is unaffected (a member is
// dropped only by a candidate whose region contains it) and so is every later
// redundancy decision (transitivity), so only the host's final member list
// (alive rows in physical order = the reference's ordered list) needs the
// flags.  FP4 rows past the member count are never-hit pad rows, so the
// classifier may stream a host-side upper bound of the count.
#include <algorithm>

#include "common.cuh"

namespace {

constexpr int kScanThreads = 128;
constexpr int kScanStage = 32;      // candidates staged in shared memory per pass
constexpr int kMaxWords = RSR_REFSET_MAX_ROW_BYTES / 16;

__device__ __forceinline__ uint32_t nib(int e) { return e ? 0x2u : 0u; }

// Candidate c's FP4 row under its own side's encoding (bias column 0).
__global__ void encode_cands_kernel(const uint8_t* __restrict__ cands,
                                    const uint8_t* __restrict__ cand_side, int N, int M,
                                    uint8_t* __restrict__ out, int row_bytes) {
  const int c = blockIdx.x;
  const uint8_t* x = cands + (int64_t)c * N;
  const bool upper = cand_side[c] == RSR_SIDE_UPPER;
  const int kdim = N * (M - 1);
  for (int b = threadIdx.x; b < row_bytes; b += blockDim.x) {
    uint32_t v = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * b + h;
      if (e < kdim) {
        const int n = e / (M - 1), k = e - n * (M - 1) + 1;
        const bool ge = x[n] >= k;
        v |= nib(upper ? ge : !ge) << (4 * h);
      }
    }
    out[(int64_t)c * row_bytes + b] = (uint8_t)v;
  }
}

// covered[c] |= some alive member m makes c redundant; covers[c] |= c makes
// some alive member redundant.  Thread = member (row words in registers),
// candidates of the member's side staged in shared memory; blockIdx.z takes a
// slice of kScanSlice candidates, so a 64-candidate batch against ~10^4 members
// runs as ~600 CTAs instead of ~80 (the scan is latency-bound, not work-bound).
constexpr int kScanSlice = 16;

__global__ void __launch_bounds__(kScanThreads) scan_kernel(
    const uint8_t* __restrict__ cand_fp4, const uint8_t* __restrict__ cand_side, int B,
    rsr_refset_dev lower, rsr_refset_dev upper, int row_bytes, uint8_t* covered,
    uint8_t* covers) {
  __shared__ uint4 sc[kScanStage][kMaxWords];
  __shared__ int sidx[kScanStage];
  const int side = blockIdx.y;
  const rsr_refset_dev& set = side == RSR_SIDE_UPPER ? upper : lower;
  const int64_t n = set.ctr[0];
  const int64_t m = (int64_t)blockIdx.x * kScanThreads + threadIdx.x;
  if ((int64_t)blockIdx.x * kScanThreads >= n) return;  // block-uniform
  const int nw = row_bytes / 16;
  const bool live = m < n && set.alive[m];
  uint4 mw[kMaxWords];
  if (live) {
    const uint4* src = reinterpret_cast<const uint4*>(set.fp4 + m * row_bytes);
#pragma unroll
    for (int w = 0; w < kMaxWords; ++w)
      if (w < nw) mw[w] = src[w];
  }
  const int cz = blockIdx.z * kScanSlice, cend = min(B, cz + kScanSlice);
  for (int c0 = cz; c0 < cend; c0 += kScanStage) {
    const int cn = min(kScanStage, cend - c0);
    __syncthreads();
    for (int i = threadIdx.x; i < cn * nw; i += kScanThreads) {
      const int c = i / nw, w = i - c * nw;
      sc[c][w] = reinterpret_cast<const uint4*>(cand_fp4 + (int64_t)(c0 + c) * row_bytes)[w];
    }
    if (threadIdx.x < cn) sidx[threadIdx.x] = cand_side[c0 + threadIdx.x] == side ? 1 : 0;
    __syncthreads();
    if (!live) continue;
    for (int c = 0; c < cn; ++c) {
      if (!sidx[c]) continue;
      uint32_t red = 0, cov = 0;
#pragma unroll
      for (int w = 0; w < kMaxWords; ++w) {
        if (w < nw) {
          const uint4 e = sc[c][w];
          red |= (mw[w].x & ~e.x) | (mw[w].y & ~e.y) | (mw[w].z & ~e.z) | (mw[w].w & ~e.w);
          cov |= (e.x & ~mw[w].x) | (e.y & ~mw[w].y) | (e.z & ~mw[w].z) | (e.w & ~mw[w].w);
        }
      }
      if (red == 0) covered[c0 + c] = 1;
      if (cov == 0) covers[c0 + c] = 1;
    }
  }
}

// rel[c * B + j] (same side only): bit0 = j redundant under c, bit1 = c
// redundant under j.
__global__ void rel_kernel(const uint8_t* __restrict__ cand_fp4, const uint8_t* __restrict__ cand_side,
                           int B, int row_bytes, uint8_t* rel) {
  const int c = blockIdx.x;
  const int nw = row_bytes / 16;
  const uint4* ec = reinterpret_cast<const uint4*>(cand_fp4 + (int64_t)c * row_bytes);
  for (int j = threadIdx.x; j < B; j += blockDim.x) {
    uint8_t r = 0;
    if (j != c && cand_side[j] == cand_side[c]) {
      const uint4* ej = reinterpret_cast<const uint4*>(cand_fp4 + (int64_t)j * row_bytes);
      uint32_t j_under_c = 0, c_under_j = 0;
      for (int w = 0; w < nw; ++w) {
        const uint4 a = ec[w], b = ej[w];
        c_under_j |= (b.x & ~a.x) | (b.y & ~a.y) | (b.z & ~a.z) | (b.w & ~a.w);
        j_under_c |= (a.x & ~b.x) | (a.y & ~b.y) | (a.z & ~b.z) | (a.w & ~b.w);
      }
      r = (uint8_t)((j_under_c == 0 ? 1 : 0) | (c_under_j == 0 ? 2 : 0));
    }
    rel[(int64_t)c * B + j] = r;
  }
}

// One CTA resolves the batch.  With "x <= y" for "x redundant under y"
// (transitive) and the set an antichain before the batch, the reference's
// sequential loop (boundary.py:100-108) has a closed form, so every candidate
// is decided in parallel:
//   c redundant    <=> covered[c] or c <= j for some earlier same-side j
//                      (a redundant or dropped j leads, by transitivity, to a
//                      current member above c);
//   inserted j dead <=> j <= c for some later inserted c;
//   member m dead   <=> m <= c for some inserted c (covers[c] flags the
//                      candidates worth checking; rare).
// Rows of inserted candidates follow their side's member count in pick order.
// report (int64 [8]): {lower rows, lower alive, upper rows, upper alive,
// redundant searches (+=), dropped members (+=), sum of calls (this batch),
// capacity overflow (|=)}.
constexpr int kResolveThreads = 1024;

__global__ void __launch_bounds__(kResolveThreads) resolve_kernel(
    const uint8_t* __restrict__ cands, const uint8_t* __restrict__ cand_side,
    const uint8_t* __restrict__ cand_fp4, int B, int N, int row_bytes,
    const uint8_t* __restrict__ covered, const uint8_t* __restrict__ covers,
    const uint8_t* __restrict__ rel_g, rsr_refset_dev lower, rsr_refset_dev upper,
    uint8_t* outcome, int64_t* row_of, const int64_t* calls, int64_t* report, int stage_rel) {
  extern __shared__ __align__(16) uint8_t smem[];
  int64_t* s_row = reinterpret_cast<int64_t*>(smem);             // [B]
  int* s_drop = reinterpret_cast<int*>(smem + 8 * (size_t)B);      // [B] member droppers
  uint8_t* s_side = smem + 12 * (size_t)B;                        // [B] 0 lower, 1 upper
  uint8_t* s_ins = s_side + B;                                    // [B]
  // the B x B relation, staged in shared memory when it fits: the scans below read
  // it row by row (a chain of dependent global loads was most of this kernel's time)
  const uint8_t* rel = rel_g;
  if (stage_rel) {
    uint8_t* s_rel = s_ins + B;                                   // [B][B]
    for (int i = threadIdx.x; i < B * B; i += blockDim.x) s_rel[i] = rel_g[i];
    rel = s_rel;
    __syncthreads();
  }
  __shared__ int64_t s_n0[2], s_nins[2], s_dead[2];
  __shared__ int s_red, s_over, s_ndrop;
  __shared__ long long s_calls;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_n0[0] = lower.ctr[0];
    s_n0[1] = upper.ctr[0];
    s_nins[0] = s_nins[1] = s_dead[0] = s_dead[1] = 0;
    s_red = s_over = s_ndrop = 0;
    s_calls = 0;
  }
  // redundancy (parallel over candidates)
  for (int c = tid; c < B; c += blockDim.x) {
    const uint8_t sd = cand_side[c] == RSR_SIDE_UPPER ? 1 : 0;
    const uint8_t* rr = rel + (int64_t)c * B;
    uint32_t any2 = 0;
    for (int j = 0; j < c; ++j) any2 |= rr[j];  // rel is 0 across sides
    const bool red = covered[c] != 0 || (any2 & 2) != 0;
    s_side[c] = sd;
    s_ins[c] = red ? 0 : 1;
  }
  __syncthreads();
  // member rows of the inserted candidates: prefix counts per side (warp 0)
  if (tid < 32) {
    int64_t base[2] = {s_n0[0], s_n0[1]};
    const int64_t cap[2] = {lower.cap, upper.cap};
    int red = 0, over = 0;
    for (int c0 = 0; c0 < B; c0 += 32) {
      const int c = c0 + tid;
      const bool in = c < B && s_ins[c];
      const int sd = c < B ? s_side[c] : 0;
      red += __popc(__ballot_sync(0xffffffffu, c < B && !in));
      for (int s2 = 0; s2 < 2; ++s2) {
        const unsigned m = __ballot_sync(0xffffffffu, in && sd == s2);
        if (in && sd == s2) {
          const int64_t r = base[s2] + __popc(m & ((1u << tid) - 1u));
          if (r < cap[s2]) {
            s_row[c] = r;
          } else {  // host sized the capacity too small: flag, do not write
            s_row[c] = -1;
            over = 1;
          }
        }
        base[s2] += __popc(m);
      }
      if (c < B && !in) s_row[c] = -1;
    }
    over = __any_sync(0xffffffffu, over);
    if (tid == 0) {
      s_nins[0] = base[0] - s_n0[0];
      s_nins[1] = base[1] - s_n0[1];
      s_red = red;
      s_over = over;
      if (over) {  // keep the counters consistent with the rows actually written
        s_nins[0] = min(s_nins[0], lower.cap - s_n0[0]);
        s_nins[1] = min(s_nins[1], upper.cap - s_n0[1]);
      }
    }
  }
  __syncthreads();
  rsr_refset_dev* sets[2] = {&lower, &upper};
  // outcomes, batch-internal drops, appends
  int local_dead[2] = {0, 0};
  long long local_calls = 0;
  for (int c = tid; c < B; c += blockDim.x) {
    const int64_t r = s_row[c];
    outcome[c] = r >= 0 ? 1 : 2;
    row_of[c] = r;
    if (calls) local_calls += calls[c];
    if (r < 0) continue;
    bool dead = false;
    for (int d = c + 1; d < B; ++d)
      dead |= s_row[d] >= 0 && (rel[(int64_t)d * B + c] & 1);  // c <= later inserted d
    sets[s_side[c]]->alive[r] = dead ? 0 : 1;
    if (dead) ++local_dead[s_side[c]];
    if (covers[c]) s_drop[atomicAdd(&s_ndrop, 1)] = c;
  }
  // appends: one warp per inserted candidate row (u8 row bytewise, FP4 row as 16-byte
  // words; a per-byte index division over the whole batch was this kernel's main cost)
  {
    const int warp = tid >> 5, lane = tid & 31, nwarps = blockDim.x >> 5;
    for (int c = warp; c < B; c += nwarps) {
      const int64_t r = s_row[c];
      if (r < 0) continue;
      const rsr_refset_dev& set = s_side[c] ? upper : lower;
      uint8_t* dst = set.rows + r * N;
      const uint8_t* src = cands + (int64_t)c * N;
      for (int k = lane; k < N; k += 32) dst[k] = src[k];
      uint4* fd = reinterpret_cast<uint4*>(set.fp4 + r * row_bytes);
      const uint4* fs = reinterpret_cast<const uint4*>(cand_fp4 + (int64_t)c * row_bytes);
      for (int k = lane; k < row_bytes / 16; k += 32) fd[k] = fs[k];
    }
  }
  __syncthreads();
  // pre-batch members made redundant by an inserted candidate (rare)
  if (s_ndrop) {
    const int nw = row_bytes / 16;
    for (int s2 = 0; s2 < 2; ++s2) {
      rsr_refset_dev& set = *sets[s2];
      for (int64_t m = tid; m < s_n0[s2]; m += blockDim.x) {
        if (!set.alive[m]) continue;
        const uint4* em = reinterpret_cast<const uint4*>(set.fp4 + m * row_bytes);
        for (int q = 0; q < s_ndrop; ++q) {
          const int c = s_drop[q];
          if (s_side[c] != s2) continue;
          const uint4* ec = reinterpret_cast<const uint4*>(cand_fp4 + (int64_t)c * row_bytes);
          uint32_t acc = 0;  // m <= c: E_c & ~E_m == 0
          for (int w = 0; w < nw; ++w) {
            const uint4 a = em[w], e = ec[w];
            acc |= (e.x & ~a.x) | (e.y & ~a.y) | (e.z & ~a.z) | (e.w & ~a.w);
          }
          if (acc == 0) {
            set.alive[m] = 0;
            ++local_dead[s2];
            break;
          }
        }
      }
    }
  }
  for (int s2 = 0; s2 < 2; ++s2)
    if (local_dead[s2]) atomicAdd(reinterpret_cast<unsigned long long*>(&s_dead[s2]),
                                  (unsigned long long)local_dead[s2]);
  if (local_calls) atomicAdd(reinterpret_cast<unsigned long long*>(&s_calls),
                             (unsigned long long)local_calls);
  __syncthreads();
  if (tid == 0) {
    for (int s2 = 0; s2 < 2; ++s2) {
      sets[s2]->ctr[0] = s_n0[s2] + s_nins[s2];
      sets[s2]->ctr[1] += s_nins[s2] - s_dead[s2];
    }
    report[0] = lower.ctr[0];
    report[1] = lower.ctr[1];
    report[2] = upper.ctr[0];
    report[3] = upper.ctr[1];
    report[4] += s_red;
    report[5] += s_dead[0] + s_dead[1];
    report[6] = s_calls;
    report[7] |= s_over;
  }
}

// out[i] = states[idx[pos[i]]] (N bytes each): rows of picked unclassified samples.
__global__ void gather_picks_kernel(const uint8_t* __restrict__ states, int N,
                                    const int64_t* __restrict__ idx, const int64_t* __restrict__ pos,
                                    uint8_t* __restrict__ out) {
  const int i = blockIdx.x;
  const int64_t row = idx[pos[i]];
  for (int n = threadIdx.x; n < N; n += blockDim.x) out[(int64_t)i * N + n] = states[row * N + n];
}

// dst[i] = src[idx[i]] (copy_bytes per row, 16-byte vectors), i < *count:
// one warp per row, grid-stride (the count lives on the device).
__global__ void gather_rows_dev_kernel(const uint8_t* __restrict__ src, int64_t src_stride,
                                       int vecs, const int64_t* __restrict__ idx,
                                       const int64_t* __restrict__ count_dev, int64_t cap,
                                       uint8_t* __restrict__ dst, int64_t dst_stride) {
  const int64_t n = min(*count_dev, cap);
  const int lane = threadIdx.x & 31;
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n;
       i += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const uint4* s = reinterpret_cast<const uint4*>(src + idx[i] * src_stride);
    uint4* d = reinterpret_cast<uint4*>(dst + i * dst_stride);
    for (int v = lane; v < vecs; v += 32) d[v] = s[v];
  }
}

// flags[idx[i]] |= vals[i], i < *count.
__global__ void scatter_or_dev_kernel(const uint8_t* __restrict__ vals,
                                      const int64_t* __restrict__ idx,
                                      const int64_t* __restrict__ count_dev, int64_t cap,
                                      uint8_t* __restrict__ flags) {
  const int64_t n = min(*count_dev, cap);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (vals[i]) flags[idx[i]] |= vals[i];
}

// Same rows decoded from the FP4 sample operand (A_lo half: element n(M-1)+k-1
// is e2m1 1.0 = 0x2 iff x_n >= k, so x_n = sum_k of those bits).
__global__ void gather_picks_fp4_kernel(const uint8_t* __restrict__ fp4, int row_bytes, int N,
                                        int M, const int64_t* __restrict__ idx,
                                        const int64_t* __restrict__ pos, uint8_t* __restrict__ out) {
  const int i = blockIdx.x;
  const uint8_t* lo = fp4 + idx[pos[i]] * (int64_t)(2 * row_bytes) + row_bytes;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    int x = 0;
    for (int k = 1; k < M; ++k) {
      const int e = n * (M - 1) + k - 1;
      x += (lo[e >> 1] >> (4 * (e & 1) + 1)) & 1;
    }
    out[(int64_t)i * N + n] = (uint8_t)x;
  }
}

}  // namespace

extern "C" int rsr_gather_picks_fp4(const uint8_t* fp4, int row_bytes, int n_components,
                                    int n_states, const int64_t* idx, const int64_t* pos,
                                    int64_t count, uint8_t* out, void* stream) {
  RSR_REQUIRE(n_components >= 1 && n_states >= 2 && count >= 0 && count <= 0x7fffffff,
              "rsr_gather_picks_fp4: bad shape");
  RSR_REQUIRE(row_bytes == rsr_fp4_row_bytes(n_components, n_states),
              "rsr_gather_picks_fp4: row_bytes must be %d", rsr_fp4_row_bytes(n_components, n_states));
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(fp4 && idx && pos && out, "rsr_gather_picks_fp4: null pointer");
  gather_picks_fp4_kernel<<<(unsigned)count, 128, 0, rsr::as_stream(stream)>>>(
      fp4, row_bytes, n_components, n_states, idx, pos, out);
  return rsr::check_launch("gather_picks_fp4_kernel");
}

extern "C" int rsr_gather_rows_dev(const uint8_t* src, int64_t src_stride, int copy_bytes,
                                   const int64_t* idx, const int64_t* count_dev, int64_t cap,
                                   uint8_t* dst, int64_t dst_stride, void* stream) {
  RSR_REQUIRE(copy_bytes > 0 && copy_bytes % 16 == 0 && src_stride % 16 == 0 && dst_stride % 16 == 0,
              "rsr_gather_rows_dev: rows must be whole 16-byte vectors");
  RSR_REQUIRE(cap >= 0, "rsr_gather_rows_dev: bad capacity");
  if (cap == 0) return RSR_OK;
  RSR_REQUIRE(src && idx && count_dev && dst, "rsr_gather_rows_dev: null pointer");
  RSR_REQUIRE(((uintptr_t)src | (uintptr_t)dst) % 16 == 0, "rsr_gather_rows_dev: unaligned rows");
  const int64_t grid = std::min<int64_t>(rsr::ceil_div(cap, 8), 148 * 8);
  gather_rows_dev_kernel<<<(unsigned)grid, 256, 0, rsr::as_stream(stream)>>>(
      src, src_stride, copy_bytes / 16, idx, count_dev, cap, dst, dst_stride);
  return rsr::check_launch("gather_rows_dev_kernel");
}

extern "C" int rsr_scatter_or_dev(const uint8_t* vals, const int64_t* idx, const int64_t* count_dev,
                                  int64_t cap, uint8_t* flags, void* stream) {
  RSR_REQUIRE(cap >= 0, "rsr_scatter_or_dev: bad capacity");
  if (cap == 0) return RSR_OK;
  RSR_REQUIRE(vals && idx && count_dev && flags, "rsr_scatter_or_dev: null pointer");
  const int64_t grid = std::min<int64_t>(rsr::ceil_div(cap, 256), 148 * 4);
  scatter_or_dev_kernel<<<(unsigned)grid, 256, 0, rsr::as_stream(stream)>>>(vals, idx, count_dev,
                                                                            cap, flags);
  return rsr::check_launch("scatter_or_dev_kernel");
}

extern "C" int64_t rsr_refset_scratch(int64_t B, int row_bytes) {
  if (B < 0 || row_bytes < 0) return 0;
  // cand_fp4 [B*rb] | covered [B] | covers [B] | rel [B*B] | row_of int64 [B], 16-aligned parts
  auto a16 = [](int64_t x) { return (x + 15) / 16 * 16; };
  return a16(B * row_bytes) + a16(B) + a16(B) + a16(B * B) + a16(8 * B);
}

extern "C" int rsr_refset_insert(const uint8_t* cands, const uint8_t* cand_side, int64_t B,
                                 int n_components, int n_states, const rsr_refset_dev* lower,
                                 const rsr_refset_dev* upper, const int64_t* calls,
                                 uint8_t* outcome, int64_t* report, void* scratch, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(N >= 1 && M >= 2 && B >= 0, "rsr_refset_insert: bad shape");
  RSR_REQUIRE(B <= 65535, "rsr_refset_insert: at most 65535 candidates per call");
  RSR_REQUIRE(lower && upper && report, "rsr_refset_insert: null set/report");
  const int rb = rsr_fp4_row_bytes(N, M);
  RSR_REQUIRE(rb <= RSR_REFSET_MAX_ROW_BYTES, "rsr_refset_insert: rows wider than %d bytes",
              RSR_REFSET_MAX_ROW_BYTES);
  for (const rsr_refset_dev* s : {lower, upper})
    RSR_REQUIRE(s->rows && s->fp4 && s->alive && s->ctr && s->cap >= 0 && s->n_bound >= 0,
                "rsr_refset_insert: incomplete set descriptor");
  cudaStream_t st = rsr::as_stream(stream);
  if (B == 0) return RSR_OK;
  RSR_REQUIRE(cands && cand_side && outcome && scratch, "rsr_refset_insert: null pointer");
  auto a16 = [](int64_t x) { return (x + 15) / 16 * 16; };
  uint8_t* p = static_cast<uint8_t*>(scratch);
  uint8_t* cand_fp4 = p;
  p += a16(B * rb);
  uint8_t* covered = p;
  p += a16(B);
  uint8_t* covers = p;
  p += a16(B);
  uint8_t* rel = p;
  p += a16(B * B);
  int64_t* row_of = reinterpret_cast<int64_t*>(p);
  RSR_CUDA(cudaMemsetAsync(covered, 0, a16(B) * 2, st));
  encode_cands_kernel<<<(unsigned)B, 128, 0, st>>>(cands, cand_side, N, M, cand_fp4, rb);
  int rc = rsr::check_launch("encode_cands_kernel");
  if (rc) return rc;
  const int64_t nb = std::max(lower->n_bound, upper->n_bound);
  if (nb > 0) {
    dim3 grid((unsigned)rsr::ceil_div(nb, kScanThreads), 2, (unsigned)rsr::ceil_div(B, kScanSlice));
    scan_kernel<<<grid, kScanThreads, 0, st>>>(cand_fp4, cand_side, (int)B, *lower, *upper, rb,
                                               covered, covers);
    rc = rsr::check_launch("scan_kernel");
    if (rc) return rc;
  }
  if (B > 1) {
    rel_kernel<<<(unsigned)B, 128, 0, st>>>(cand_fp4, cand_side, (int)B, rb, rel);
    rc = rsr::check_launch("rel_kernel");
    if (rc) return rc;
  }
  const int stage_rel = (size_t)B * B <= 64 * 1024 ? 1 : 0;
  const size_t rsmem = 14 * (size_t)B + 16 + (stage_rel ? (size_t)B * B : 0);
  RSR_REQUIRE(rsmem <= 200 * 1024, "rsr_refset_insert: batch too large");
  if (rsmem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(resolve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)rsmem));
  resolve_kernel<<<1, kResolveThreads, rsmem, st>>>(cands, cand_side, cand_fp4, (int)B, N, rb,
                                                    covered, covers, rel, *lower, *upper, outcome,
                                                    row_of, calls, report, stage_rel);
  return rsr::check_launch("resolve_kernel");
}

extern "C" int rsr_gather_picks(const uint8_t* states, int n_components, const int64_t* idx,
                                const int64_t* pos, int64_t count, uint8_t* out, void* stream) {
  RSR_REQUIRE(n_components >= 1 && count >= 0 && count <= 0x7fffffff, "rsr_gather_picks: bad shape");
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(states && idx && pos && out, "rsr_gather_picks: null pointer");
  gather_picks_kernel<<<(unsigned)count, 128, 0, rsr::as_stream(stream)>>>(states, n_components, idx,
                                                                            pos, out);
  return rsr::check_launch("gather_picks_kernel");
}
