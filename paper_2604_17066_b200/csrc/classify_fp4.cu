// (2) Dominance classification on block-scaled FP4 tensor cores
// (tcgen05.mma.cta_group::2.kind::mxf4, e2m1 operands, ue8m0 scales chosen so
// the fp32 accumulator's bit pattern is the integer violation count).
//
// Replaces the same reference code as classify_tc.cu -- classify.py:99-148
// (_chunk_hits / _hits_for: any reference with popcount(sample & ~ref) == 0)
// and the precedence step classify.py:240-241 -- at twice the int8 MMA rate.
// 0/1 operands and dot products <= N(M-1) are exact in e2m1 x e2m1 -> fp32, so
// the result is the same integer violation count, but there are no negative
// operands, so each side gets its own sample operand:
//   upper ref r:  D = sum_c [x_n <  k] [r_n >= k]   (A_up = thermometer "below")
//   lower ref r:  D = sum_c [x_n >= k] [r_n <  k]   (A_lo = its complement)
// and D == 0 <=> x dominates r (upper) / is dominated by r (lower).  Column
// Kdim = N(M-1) is a bias column: 1 in both sample operands, 0 in real
// reference rows, 1 in never-hit pad rows (D >= 1).  See include/rsr_b200.h
// ("FP4 layout").
//
// Kernel shape (persistent, one CTA pair per TPC, 384 threads per CTA):
//   * operands are stored in HBM as rows of 32-byte chunks and land in shared
//     memory chunk-major ([chunk][row][32 B], 32-byte swizzle) from ONE 3-D TMA
//     box per operand tile, so a chunk is exactly one MMA K-step (64 e2m1) and
//     no shared memory is spent on K padding;
//   * a group of 256 samples (128 per CTA) holds both A_up and A_lo
//     (2 x cq chunks), double-buffered so the next group loads during compute;
//   * reference tiles of 240 rows (120 per CTA) stream through a ring of
//     whole-tile stages; the leader issues cq MMAs M=256 N=240 K=64 per tile;
//   * TMEM: accumulators at columns 0 and 240 (two buffers, the epilogue of
//     tile j overlaps the MMAs of tile j+1), scale factors at 480..511;
//   * 4 epilogue warps per CTA read the 128 x 240 accumulator with packed
//     16-bit loads (tcgen05.ld 32x32b .pack::16b: each accumulator is the
//     denormal count * 2^-149, so its low 16 bits are the count), min-reduce
//     with 16x2 SIMD mins, OR a hit bit per side, and optionally keep the
//     first matching reference index (explain/strict).
#include <stdlib.h>

#include <algorithm>

#include "fp4_encode.cuh"
#include "tc_common.cuh"

namespace {

constexpr int kRowsA = 128;      // sample rows per CTA
constexpr int kChunk = 32;       // bytes per chunk = 64 e2m1 = one MMA K-step
constexpr int kChunkA = kRowsA * kChunk;  // 4096 B
constexpr uint32_t kSfaCol = 480, kSfbCol = 496;
constexpr uint32_t kSfaByte = 0x00, kSfbByte = 0x69;  // ue8m0 2^-127 and 2^-22
// Paired accumulators (rows of <= 4 K-steps, no first matches): two reference tiles share
// one accumulator buffer.  The second tile's MMAs read B scale 2^-6 (ue8m0 0x79) from TMEM
// column kSfbHiCol, so its products are 2^-133 = 2^16 * 2^-149 and each fp32 accumulator's
// bit pattern is c1 + 2^16 c2 (both counts <= 255 real columns < 2^8, the sum < 2^24:
// exact, and bits 16..23 hold c2 even once the value leaves the denormal range).  The MMA
// time per buffer doubles while the epilogue reads the same 32-bit values (both halves
// min-reduced by the same 16x2 SIMD mins), so the accumulator round trip that bounds
// 4-K-step tiles (~600 cycles vs ~500 of MMAs per tile: 0.855 of the MMA rate) is
// covered again.  Needs kBufs * TN <= kSfbHiCol (TN <= 224).
constexpr uint32_t kSfbHiCol = 464, kSfbHiByte = 0x79;
// PAIR = 2 ("packed pairs"): the second tile's scale is 2^-14 (0x71), so an accumulator holds
// c1 + 2^8 c2 < 2^16 -- a denormal whose low 16 bits carry both counts, read with the same
// .pack::16b loads as an unpaired tile (half the TMEM bytes of PAIR = 1).  The epilogue
// tests tile b by min16 < 256 and tile a by min16 of the low bytes moved up (one PRMT per
// register): two 16x2 min chains instead of one, after the buffer is released.
constexpr uint32_t kSfbHi8Byte = 0x71;
// PAIR = 3 ("shared tail"): rows of 4 K-steps whose columns are [192 main | 32 tail | the
// same 32 tail] on the sample side.  The even tile a of each pair (2p, 2p+1) carries in its
// last K-step [its own tail | tile b's tail] (the host builds that layout), so one MMA
// covers both tiles' tail columns: A scale 2^-127 on K-block 0 and 2^-111 (x 2^16) on
// K-block 1 (TMEM column kSfaTailCol, word p.sfa_tail_word).  Tile a issues 4 MMAs,
// tile b 3: 7 instead of 8 per pair.  Needs kBufs * TN <= kSfaTailCol and pair-aligned
// tile sequences (even rotation, even tile counts: the host pads with never-hit tiles).
constexpr uint32_t kSfaTailCol = 448;
// Paired buffers are read by BOTH epilogue sets, each set its half of the columns (8 warps
// per buffer: TMEM loads at 324 instead of 175 B/clk per SM, tools/tmem_bw.cu), so the
// accumulator round trip shortens by about one half-buffer load; every set ORs its own hit
// bits into the flags.  Measured slightly slower (cfg4 K = 5x10^5: 122.3 vs 121.6 ms; the
// pairs are not round-trip bound), so off: -DRSR_FP4_PAIR_SPLIT=1 builds it.
#ifndef RSR_FP4_PAIR_SPLIT
#define RSR_FP4_PAIR_SPLIT 0
#endif

// Reference tiles are 240 rows (120 per CTA).  TMEM holds two accumulator
// buffers of 240 columns (0..479; 480..511 hold the scale factors), so the
// epilogue of tile j overlaps the MMAs of tile j+1.  Reading a 128 x 240 fp32
// accumulator out of TMEM is the epilogue's cost (tools/tmem_bw.cu: 32x32b
// loads reach 175 / 324 / 459 B/clk per SM with 4 / 8 / 16 warps, and twice that
// with .pack::16b).  Each epilogue warp owns one TMEM lane quarter and a row's
// whole tile (up to 120 packed registers).  kEpiSets sets of 4 warps take turns
// by tile: set e handles tiles e, e + kEpiSets, ... of the cluster's sequence, so
// a set has kEpiSets tile times for each tile's load, release and reduction, and a
// finished tile always finds its set idle.  With one set (r1) the epilogue was
// busy ~430 of each 208-column tile's ~630 cycles and its queueing delayed the
// buffer release (tools/fp4_prof.py; an RSR_FP4_X_NOMIN build that skips the
// reduction ran cfg4 K = 10^3 6 % faster).  Splitting a tile's columns over two
// warps per lane quarter instead (r1) cost more than it saved: 16 arrivals per
// tile and a cross-warp exchange per group.
#ifndef RSR_FP4_EPI_SETS
#define RSR_FP4_EPI_SETS 2
#endif
#ifndef RSR_FP4_SPIN
#define RSR_FP4_SPIN 0
#endif
#ifndef RSR_FP4_SET_RELEASE
#define RSR_FP4_SET_RELEASE 0
#endif
// experiment knobs, both measured slower (spinning warps take issue slots from
// the MMA / TMA warps): RSR_FP4_SPIN spins the MMA warp on buffer release,
// RSR_FP4_EPI_SPIN the epilogue warps on accumulator completion
#ifndef RSR_FP4_EPI_SPIN
#define RSR_FP4_EPI_SPIN 0
#endif
// 1: every set takes every tile, set e reading columns [e TN/kEpiSets, (e+1) TN/kEpiSets)
// (the tile's TMEM load is kEpiSets x shorter, so the buffer returns to the MMA warp
// sooner); 0: sets take turns by tile, each reading whole tiles
#ifndef RSR_FP4_SPLIT_COLS
#define RSR_FP4_SPLIT_COLS 0
#endif
constexpr int kEpiSets = RSR_FP4_EPI_SETS;
// (4 sets measured as a launch failure at 640 threads: profiles/r2_fp4_small_k_experiments.txt)
static_assert(kEpiSets == 1 || kEpiSets == 2, "epilogue sets: 1 or 2");
constexpr int kEpiWarps = 4 * kEpiSets;
constexpr int kThreads = 128 + 32 * kEpiWarps;

// Reference tile geometry for MMA N = TN (a multiple of 16; the launch picks
// TN per call to minimise padded reference rows, e.g. 5 x 208 for 1000 refs):
// TMEM columns 0..479 hold 480 / TN accumulator buffers, 480..511 the scales.
template <int TN>
struct Tile {
  static constexpr int kBufs = 480 / TN;
  static constexpr int kHalfRows = TN / 2;             // reference rows per CTA per tile
  static constexpr int kChunkB = kHalfRows * kChunk;   // bytes per K-step per CTA
  static_assert(TN % 16 == 0 && TN <= 240 && kBufs >= 2 && kBufs <= 4, "bad tile N");
};

// RSR_FP4_PROF builds (tools/ only, never the product library) accumulate
// per-role cycle counters into g_prof: 0 MMA wait b_full, 1 MMA wait t_empty,
// 2 MMA loop total, 3 epilogue wait t_full, 4 epilogue load+release,
// 5 epilogue compute, 6 producer wait b_empty, 7 tiles (MMA warp), 8 epilogue
// group-end exchange, 9 MMA wait a_full, 10 producer wait a_empty, 11 groups (MMA);
// 4 covers load + release + compute of the tile, 5 the bookkeeping after it.
// Counters live in registers (prof[8] per thread) and are flushed once per
// warp at the end, so the instrumentation barely perturbs the timing.
#ifdef RSR_FP4_PROF
constexpr int kProf = 24;
__device__ unsigned long long g_prof[kProf];
#define PROF_DECL unsigned long long prof[kProf] = {}
#define PROF_T(x) const long long x = clock64()
#define PROF_ADD(i, v) (prof[i] += (unsigned long long)(v))
#define PROF_FLUSH                                                   \
  if ((threadIdx.x & 31) == 0)                                       \
    for (int i_ = 0; i_ < kProf; ++i_) atomicAdd(&g_prof[i_], prof[i_])
#else
#define PROF_DECL
#define PROF_T(x)
#define PROF_ADD(i, v)
#define PROF_FLUSH
#endif

struct Fp4Params {
  int64_t S;
  int n_groups;
  int cq;           // chunks per operand row (row bytes / 32)
  int nt_lower;     // tiles of lower refs (come first)
  int nt_total;
  int stages;
  int a_bufs;
  int a_halves;     // sample halves per buffer: 2, or 1 when every tile is of one side
  uint8_t* flags;
  int accumulate;
  int64_t* first_lower;
  int64_t* first_upper;
  int64_t first_base_lower;
  int64_t first_base_upper;
  int64_t n_lower;  // reference rows of this launch per side (columns beyond are masked)
  int64_t n_upper;
  int resident;     // every reference tile has its own stage: loaded once, reused by all groups
  int n_res;        // tiles j < n_res are resident in stage j (loaded once); the others stream
                    // through stages n_res .. stages-1 (n_res = nt_total when resident)
  const int64_t* S_dev;  // optional device sample count (<= S): rows [S_dev, S) are skipped
  int flag_or;      // flags merged with 32-bit atomic ORs (no FIRST; flags 4-byte aligned,
                    // zeroed before the first launch unless accumulating)
  uint32_t sfa_tail_word;  // PAIR = 3: the A scale-factor word of the shared tail K-step
};

// SW32 K-major descriptor: 8-row core groups 256 B apart, version 1, layout 6.
__device__ __forceinline__ uint32_t desc32_lo(uint32_t saddr) {
  return ((saddr >> 4) & 0x3FFFu) | (1u << 16);
}
constexpr uint32_t kDesc32Hi = (256u >> 4) | (1u << 14) | (6u << 29);

// kind::mxf4 instruction descriptor: A = B = e2m1 (1), D = f32, scales ue8m0,
// K-major, K = 64, scale factor ids 0.
__host__ __device__ constexpr uint32_t mxf4_idesc(int m, int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_mxf4_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo,
                                               uint32_t idesc, uint32_t sfa, uint32_t sfb,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 da, {%1, %5};\n\t"
      "mov.b64 db, {%2, %5};\n\t"
      "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], da, db, %3, [%6], [%7], "
      "p;\n\t}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "r"(kDesc32Hi), "r"(sfa), "r"(sfb));
}

__device__ __forceinline__ void tma_load_3d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & kPeerMask), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar,
                                                 int x, int y, int z, int w) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar & kPeerMask), "r"(x), "r"(y), "r"(z), "r"(w)
      : "memory");
}

#define RSR_LD16(addr, v)                                                                      \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15}, [%16];"                                                                       \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),             \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                                                  \
      : "r"(addr))
#define RSR_LD8(addr, v)                                                                        \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"        \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),        \
                 "=r"(v[6]), "=r"(v[7])                                                         \
               : "r"(addr))

// 32x32b loads with .pack::16b: register i holds the low 16 bits of columns
// 2i (bits 0..15) and 2i+1 (bits 16..31), so one register covers two
// accumulators and the TMEM -> register traffic halves (tools/tmem_bw.cu:
// 905 vs 459 B/clk per SM with 16 warps).
#define RSR_LDP16(addr, v)                                                                     \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x16.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11," \
      "%12,%13,%14,%15}, [%16];"                                                               \
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),    \
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),             \
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15])                                                  \
      : "r"(addr))
#define RSR_LDP8(addr, v)                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.pack::16b.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),        \
                 "=r"(v[6]), "=r"(v[7])                                                         \
               : "r"(addr))
#define RSR_LDP4(addr, v)                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.pack::16b.b32 {%0,%1,%2,%3}, [%4];"        \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])                             \
               : "r"(addr))
#define RSR_LDP2(addr, v)                                                                    \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.pack::16b.b32 {%0,%1}, [%2];"              \
               : "=r"(v[0]), "=r"(v[1])                                                     \
               : "r"(addr))

// Load HN consecutive accumulator columns (HN / 2 packed registers).
template <int HN>
__device__ __forceinline__ void ld_cols_packed(uint32_t taddr, uint32_t* v) {
  constexpr int R = HN / 2;
  constexpr int n16 = R / 16, r8 = (R % 16) / 8, r4 = (R % 8) / 4, r2 = (R % 4) / 2;
  constexpr int o8 = 16 * n16, o4 = o8 + 8 * r8, o2 = o4 + 4 * r4;
#pragma unroll
  for (int i = 0; i < n16; ++i) RSR_LDP16(taddr + 32 * i, (v + 16 * i));
  if constexpr (r8 != 0) RSR_LDP8(taddr + 2 * o8, (v + o8));
  if constexpr (r4 != 0) RSR_LDP4(taddr + 2 * o4, (v + o4));
  if constexpr (r2 != 0) RSR_LDP2(taddr + 2 * o2, (v + o2));
  static_assert(HN % 4 == 0, "HN must be a multiple of 4");
}

// Epilogue of one tile for one warp.  The scale factors make every accumulator
// an fp32 denormal whose bit pattern IS the violation count (count * 2^-149,
// exact: tools/mxf4_check.cu), so the low 16 bits carry the whole count and the
// packed load reads two columns per register.  Column c of the MMA is reference
// c of the tile (CTA c / kHalfRows's B row c % kHalfRows); c0 = this warp's
// first column.  Load, release the buffer (as early as possible: the MMA warp
// waits on it), then mask columns past the side's last reference, min-reduce
// the 16-bit halves and find the first zero column.
template <int HC, bool FIRST>
__device__ __forceinline__ void epilogue_tile(uint32_t taddr, uint32_t release_bar, int lane,
                                              int c0, int64_t valid, bool& any, int& zref,
                                              long long& t_loaded, long long* ts_release,
                                              int set_id) {
  constexpr int kCols = HC;  // columns this warp reads, starting at tile column c0
  constexpr int R = kCols / 2;
  uint32_t v[R];
  ld_cols_packed<kCols>(taddr, v);
  tmem_ld_wait();
#ifdef RSR_FP4_PROF
  t_loaded = clock64();
#endif
  tc_fence_before();
  __syncwarp();
#ifdef RSR_FP4_PROF
  if (ts_release && lane == 0) *(volatile long long*)ts_release = clock64();
#endif
#if RSR_FP4_SET_RELEASE
  // experiment: the set's 4 warps of this CTA meet on a named barrier (id 2 + set),
  // then one arrival per CTA (t_empty count 2)
  named_bar_sync(2 + set_id, 128);
  if ((threadIdx.x & 127) == 0) mbar_arrive_leader(release_bar);
#else
  if (lane == 0) mbar_arrive_leader(release_bar);
#endif
  if (valid < c0 + kCols) {
#pragma unroll
    for (int c = 0; c < kCols; ++c)
      if (c0 + c >= valid) v[c / 2] |= (c & 1) ? 0xFFFF0000u : 0x0000FFFFu;
  }
#ifdef RSR_FP4_X_NOMIN
  // timing experiment only (wrong results): no reduction
  any = v[0] == 0u;
  return;
#endif
  // independent SIMD (16x2) min chains, then a tree
  constexpr int W = R >= 8 ? 4 : 2;
  uint32_t m[W];
#pragma unroll
  for (int q = 0; q < W; ++q) m[q] = v[q];
#pragma unroll
  for (int c = W; c < R; ++c) m[c % W] = __vminu2(m[c % W], v[c]);
#pragma unroll
  for (int q = 1; q < W; ++q) m[0] = __vminu2(m[0], m[q]);
  any = (m[0] & 0xFFFFu) == 0 || (m[0] >> 16) == 0;
  if (FIRST && any) {
    int zc = kCols - 1;
#pragma unroll
    for (int c = kCols - 1; c >= 0; --c)
      if (((v[c / 2] >> (16 * (c & 1))) & 0xFFFFu) == 0) zc = c;
    zref = c0 + zc;
  }
}

// Load HN consecutive full 32-bit accumulator columns (HN registers, HN % 8 == 0).
template <int HN>
__device__ __forceinline__ void ld_cols_full(uint32_t taddr, uint32_t* v) {
  static_assert(HN % 8 == 0, "HN must be a multiple of 8");
#pragma unroll
  for (int i = 0; i < HN / 16; ++i) RSR_LD16(taddr + 16 * i, (v + 16 * i));
  if constexpr (HN % 16 != 0) RSR_LD8(taddr + HN / 16 * 16, (v + HN / 16 * 16));
}

// Epilogue of one paired buffer (two reference tiles, see kSfbHiCol) for one warp: two
// rounds of TN/2 full columns (the registers of one packed tile load), the buffer
// released after the second; 16x2 SIMD mins reduce both tiles' counts at once (low
// halves: tile a, high halves: tile b).  Columns past a tile's last reference
// (valid_*) are masked; a missing second tile has valid_b = 0.
template <int HN>
__device__ __forceinline__ void epilogue_pair_half(uint32_t taddr, uint32_t release_bar,
                                                   int lane, int c0, int64_t valid_a,
                                                   int64_t valid_b, bool& any_a, bool& any_b) {
  uint32_t v[HN];
  ld_cols_full<HN>(taddr, v);
  tmem_ld_wait();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_leader(release_bar);
  if (valid_a < c0 + HN || valid_b < c0 + HN) {
#pragma unroll
    for (int c = 0; c < HN; ++c) {
      if (c0 + c >= valid_a) v[c] |= 0x0000FFFFu;
      if (c0 + c >= valid_b) v[c] |= 0xFFFF0000u;
    }
  }
  uint32_t m[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
  for (int c = 0; c < HN; ++c) m[c & 3] = __vminu2(m[c & 3], v[c]);
  const uint32_t r = __vminu2(__vminu2(m[0], m[1]), __vminu2(m[2], m[3]));
  any_a = (r & 0xFFFFu) == 0;
  any_b = (r >> 16) == 0;
}

template <int TN>
__device__ __forceinline__ void epilogue_pair(uint32_t taddr, uint32_t release_bar, int lane,
                                              int64_t valid_a, int64_t valid_b, bool& any_a,
                                              bool& any_b) {
  constexpr int H = TN / 2;
  uint32_t m[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
  for (int part = 0; part < 2; ++part) {
    uint32_t v[H];
    ld_cols_full<H>(taddr + part * H, v);
    tmem_ld_wait();
    if (part == 1) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_leader(release_bar);
    }
    const int c0 = part * H;
    if (valid_a < c0 + H || valid_b < c0 + H) {
#pragma unroll
      for (int c = 0; c < H; ++c) {
        if (c0 + c >= valid_a) v[c] |= 0x0000FFFFu;
        if (c0 + c >= valid_b) v[c] |= 0xFFFF0000u;
      }
    }
#pragma unroll
    for (int c = 0; c < H; ++c) m[c & 3] = __vminu2(m[c & 3], v[c]);
  }
  const uint32_t r = __vminu2(__vminu2(m[0], m[1]), __vminu2(m[2], m[3]));
  any_a = (r & 0xFFFFu) == 0;
  any_b = (r >> 16) == 0;
}

// Epilogue of one packed-pair buffer (PAIR = 2) for one warp: one packed load of the TN
// columns (register i: columns 2i, 2i+1, each c1 + 256 c2), release, then per register
// chain b takes min16(x) (< 256 <=> some c2 == 0) and chain a min16 of the low bytes moved
// to the high bytes (< 256 <=> some c1 == 0).  Masked columns get 0xFF in the tile's byte.
template <int TN>
__device__ __forceinline__ void epilogue_pair8(uint32_t taddr, uint32_t release_bar, int lane,
                                               int64_t valid_a, int64_t valid_b, bool& any_a,
                                               bool& any_b) {
  constexpr int R = TN / 2;
  uint32_t v[R];
  ld_cols_packed<TN>(taddr, v);
  tmem_ld_wait();
  tc_fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive_leader(release_bar);
  if (valid_a < TN || valid_b < TN) {
#pragma unroll
    for (int c = 0; c < TN; ++c) {
      const uint32_t sh = 16 * (c & 1);
      if (c >= valid_a) v[c / 2] |= 0x00FFu << sh;
      if (c >= valid_b) v[c / 2] |= 0xFF00u << sh;
    }
  }
  uint32_t ma[2] = {0xFFFFFFFFu, 0xFFFFFFFFu}, mb[2] = {0xFFFFFFFFu, 0xFFFFFFFFu};
#pragma unroll
  for (int i = 0; i < R; ++i) {
    mb[i & 1] = __vminu2(mb[i & 1], v[i]);
    ma[i & 1] = __vminu2(ma[i & 1], __byte_perm(v[i], 0u, 0x2404));
  }
  const uint32_t a = __vminu2(ma[0], ma[1]), b = __vminu2(mb[0], mb[1]);
  any_a = (a & 0xFFFFu) < 256u || (a >> 16) < 256u;
  any_b = (b & 0xFFFFu) < 256u || (b >> 16) < 256u;
}

// MMA issuer of the pair kernel (leader CTA, warp 1).  CQ > 0: compile-time K-steps.
struct MmaRole {
  uint32_t tm0, a_lo0, b_lo0;
  uint32_t bar_b_full, bar_b_empty, bar_t_full, bar_t_empty, bar_a_full, bar_a_empty;
  uint32_t a_buf_desc, b_stage_desc;
  int cluster, n_clusters, n_groups, nt_l, nt_u, rot_l, rot_u;
#ifdef RSR_FP4_PROF
  long long k_entry;
  long long* ts;  // [0][buf] commit issued (MMA warp), [1][buf] CTA-0 release (epilogue)
#endif
};

#ifdef RSR_FP4_PROF
#define PROF_PARAM , unsigned long long* prof
#define PROF_ARG , prof
#else
#define PROF_PARAM
#define PROF_ARG
#endif

template <int TN, int CQ, int PAIR>
__device__ __forceinline__ void mma_role(const MmaRole& m, const Fp4Params& p PROF_PARAM) {
  constexpr uint32_t idesc = mxf4_idesc(2 * kRowsA, TN);
  constexpr int kBufs = Tile<TN>::kBufs;
  constexpr uint32_t kAstep = kChunkA >> 4, kBstep = Tile<TN>::kChunkB >> 4;
  const uint32_t sfa = m.tm0 + kSfaCol, sfb = m.tm0 + kSfbCol, sfb_hi = m.tm0 + kSfbHiCol;
  const uint32_t sfa_tail = m.tm0 + kSfaTailCol;
  // launch constants in registers (the asm statements' memory clobbers would
  // otherwise reload them from the parameter bank on every tile)
  const int cq = CQ > 0 ? CQ : p.cq;
  const int stages = p.stages, a_bufs = p.a_bufs;
  const int n_res = p.n_res;  // tiles j < n_res sit in stage j for the whole launch
  const uint32_t a_half_desc = p.a_halves == 2 ? (uint32_t)cq * kAstep : 0u;
  int stage = n_res, gi = 0;
  uint32_t phase = 0, buf = 0, tphase = 0;
  int ab = 0;
  uint32_t a_par = 0;
#ifdef RSR_FP4_PROF
  PROF_ADD(12, clock64() - m.k_entry);  // setup before the first group
#endif
  for (int g = m.cluster; g < m.n_groups; g += m.n_clusters, ++gi) {
    PROF_ADD(11, 1);
    const uint32_t a_up = m.a_lo0 + (uint32_t)ab * m.a_buf_desc;
    const uint32_t a_dn = a_up + a_half_desc;
    // resident reference tiles: every such stage completed during group 0
    const bool first_group = gi == 0;
    PROF_T(l0);
    for (int h = 0; h < 2; ++h) {
      const int cnt = h == 0 ? m.nt_l : m.nt_u;
      if (cnt == 0) continue;
      PROF_T(w0);
      mbar_wait(m.bar_a_full + 8 * (2 * ab + h), a_par);  // this side's sample half landed
      PROF_T(w1);
      PROF_ADD(9, w1 - w0);
      tc_fence_after();
      const uint32_t al = h == 0 ? a_dn : a_up;
      const int base = h == 0 ? 0 : m.nt_l;
      int jt = h == 0 ? m.rot_l : m.rot_u;
      for (int t = 0; t < cnt; ++t) {
        const int j = base + jt;
        if (++jt == cnt) jt = 0;
        // resident B: tile j sits in stage j, whose only phase (0) completes once
        const bool res_tile = j < n_res;
        const int bs = res_tile ? j : stage;
        const uint32_t d = m.tm0 + buf * TN;
        const uint32_t bl = m.b_lo0 + (uint32_t)bs * m.b_stage_desc;
        // PAIR: odd tiles of the side accumulate into the even tile's buffer
        const bool second = PAIR != 0 && (t & 1);
        const bool close = !PAIR || second || t + 1 == cnt;
        PROF_T(m0);
        if (!second) {
#if RSR_FP4_SPIN
        mbar_spin(m.bar_t_empty + 8 * buf, tphase ^ 1);
#elif defined(RSR_FP4_X_NOWAIT)
        // timing experiment only (wrong results): never wait for the epilogue
#else
        mbar_wait_inline(m.bar_t_empty + 8 * buf, tphase ^ 1);  // tc_common.cuh: why inline
#endif
        }
        PROF_T(m1);
#ifdef RSR_FP4_PROF
        if (gi > 0) {  // release (CTA 0 epilogue, just before its arrive) -> MMA warp sees it
          PROF_ADD(17, m1 - *(volatile long long*)(m.ts + 4 + buf));
          PROF_ADD(21, 1);
        }
#endif
        if (!res_tile || first_group) mbar_wait(m.bar_b_full + 8 * bs, res_tile ? 0u : phase);
        PROF_T(m2);
        PROF_ADD(1, m1 - m0);
        PROF_ADD(0, m2 - m1);
        PROF_ADD(7, 1);
        tc_fence_after();
        if (elect_one()) {
          const uint32_t sb = second ? sfb_hi : sfb;
          if constexpr (PAIR == 3 && CQ == 4) {
            // main K-steps of either tile; the shared tail K-step with tile a only
#pragma unroll
            for (int ks = 0; ks < 3; ++ks)
              umma_mxf4_pair(d, al + ks * kAstep, bl + ks * kBstep, idesc, sfa, sb,
                             second || ks != 0);
            if (!second)
              umma_mxf4_pair(d, al + 3 * kAstep, bl + 3 * kBstep, idesc, sfa_tail, sfb, true);
          } else if constexpr (CQ > 0) {
#pragma unroll
            for (int ks = 0; ks < CQ; ++ks)
              umma_mxf4_pair(d, al + ks * kAstep, bl + ks * kBstep, idesc, sfa, sb,
                             second || ks != 0);
          } else {
            for (int ks = 0; ks < cq; ++ks)
              umma_mxf4_pair(d, al + ks * kAstep, bl + ks * kBstep, idesc, sfa, sb,
                             second || ks != 0);
          }
          if (close) umma_commit_pair(m.bar_t_full + 8 * buf);
          if (!res_tile) umma_commit_pair(m.bar_b_empty + 8 * stage);
#ifdef RSR_FP4_PROF
          const long long tc = clock64();
          *(volatile long long*)(m.ts + buf) = tc;
          PROF_ADD(18, tc - m2);  // issue of the tile's MMAs + commits
#endif
        }
        __syncwarp();
        if (!res_tile && ++stage == stages) {
          stage = n_res;
          phase ^= 1;
        }
        if (close && ++buf == kBufs) {
          buf = 0;
          tphase ^= 1;
        }
      }
      // the side's sample half is released once its MMAs complete
      if (elect_one()) umma_commit_pair(m.bar_a_empty + 8 * (2 * ab + h));
      __syncwarp();
    }
    if (++ab == a_bufs) {
      ab = 0;
      a_par ^= 1;
    }
    PROF_T(l1);
    PROF_ADD(2, l1 - l0);
  }
}

template <int TN, bool FIRST, int PAIR>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
classify_fp4_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                         const __grid_constant__ CUtensorMap map_lower,
                         const __grid_constant__ CUtensorMap map_upper, const Fp4Params p) {
  constexpr int kTileN = TN;
  constexpr int kBufs = Tile<TN>::kBufs;
  constexpr int kHalfRows = Tile<TN>::kHalfRows;
  constexpr int kChunkB = Tile<TN>::kChunkB;
  static_assert(!PAIR || (!FIRST && kBufs * TN <= (int)kSfbHiCol), "paired accumulators");
  static_assert(PAIR != 3 || kBufs * TN <= (int)kSfaTailCol, "shared-tail pairs");
  extern __shared__ uint8_t smem_raw[];
#ifdef RSR_FP4_PROF
  const long long k_entry = clock64();
  unsigned long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
#endif
  const uint32_t raw_addr = smem_addr(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  const uint32_t a_buf_bytes = (uint32_t)(p.a_halves * p.cq * kChunkA);
  const uint32_t b_stage_bytes = (uint32_t)(p.cq * kChunkB);
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)p.a_bufs * a_buf_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)p.stages * b_stage_bytes);
  uint64_t* b_full = bars;
  uint64_t* b_empty = bars + p.stages;
  // sample buffers are filled and released per half: [buffer][0 = A_lo, 1 = A_up]
  uint64_t* a_full = bars + 2 * p.stages;  // [a_bufs <= 4][2]
  uint64_t* a_empty = a_full + 8;          // [a_bufs <= 4][2]
  uint64_t* t_full = a_full + 16;          // [kBufs <= 4]
  uint64_t* t_empty = a_full + 20;         // [kBufs <= 4]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 24);
  // group-end exchange of the epilogue sets, double-buffered by group parity:
  // hit bits [2][kEpiSets][128] and first-match indices [2][kEpiSets][2][128]
  uint32_t* xchg = reinterpret_cast<uint32_t*>(a_full + 26);
  int64_t* xfirst = reinterpret_cast<int64_t*>(xchg + 2 * kEpiSets * 128);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;
  // sample count: the launch's capacity, or a device-side count (every role
  // reads the same value, so all loops agree on the group range)
  int64_t S_run = p.S;
  if (p.S_dev) {
    const int64_t sd = *p.S_dev;
    S_run = sd < 0 ? 0 : (sd < p.S ? sd : p.S);
  }
  const int n_groups = (int)((S_run + 2 * kRowsA - 1) / (2 * kRowsA));

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lower)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_upper)));
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(smem_addr(&b_full[i]), 2);
      mbar_init(smem_addr(&b_empty[i]), 1);
    }
    for (int i = 0; i < 2 * p.a_bufs; ++i) {
      mbar_init(smem_addr(&a_full[i]), 2);
      mbar_init(smem_addr(&a_empty[i]), 1);
    }
    for (int i = 0; i < kBufs; ++i) {
      mbar_init(smem_addr(&t_full[i]), 1);
      // the 4 warps of the tile's epilogue set in both CTAs (or one arrival per CTA)
      mbar_init(smem_addr(&t_empty[i]),
                RSR_FP4_SET_RELEASE                                      ? 2
                : (RSR_FP4_SPLIT_COLS ||
                   (PAIR != 0 && PAIR != 2 && RSR_FP4_PAIR_SPLIT && kEpiSets == 2))
                    ? 2 * kEpiWarps
                                                                         : 2 * 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (warp >= 4 && warp < 8) {
    // ue8m0 scale factors: A 2^-127 (0x00), B 2^-22 (0x69), so every product
    // is 2^-149 and the fp32 accumulator's bits count the violations
    const uint32_t addr = tmem_base + ((uint32_t)((warp & 3) * 32) << 16);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1};" ::"r"(addr + kSfaCol),
        "r"(kSfaByte * 0x01010101u));
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
        "%1,%1};" ::"r"(addr + kSfbCol),
        "r"(kSfbByte * 0x01010101u));
    if (PAIR)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
          "%1,%1,%1};" ::"r"(addr + kSfbHiCol),
          "r"((PAIR == 2 ? kSfbHi8Byte : kSfbHiByte) * 0x01010101u));
    if (PAIR == 3)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
          "%1,%1,%1};" ::"r"(addr + kSfaTailCol),
          "r"(p.sfa_tail_word));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  // Tile sequence of every group (all three roles walk it): the lower tiles,
  // then the upper ones, each side rotated per cluster to spread L2 load.
  // Side-ordered, the lower half of a sample buffer (A_lo) is free once the
  // group's lower tiles are issued, so the next group's A_lo loads while the
  // upper tiles run (and A_up while the next lower tiles run): single-buffered
  // wide rows (M = 3: 80 KB per buffer) still overlap their sample loads.
  const int nt_l = p.nt_lower, nt_u = p.nt_total - p.nt_lower;
  // PAIR = 3: even rotations keep the (2p, 2p+1) pairs of the host's tail layout together
  const int rot_l = (int)(((int64_t)cluster * nt_l) / n_clusters) & (PAIR == 3 ? ~1 : ~0);
  const int rot_u = (int)(((int64_t)cluster * nt_u) / n_clusters) & (PAIR == 3 ? ~1 : ~0);
  auto tile_of = [&](int jj) -> int {
    if (jj < nt_l) {
      const int j = rot_l + jj;
      return j >= nt_l ? j - nt_l : j;
    }
    const int j = rot_u + (jj - nt_l);
    return nt_l + (j >= nt_u ? j - nt_u : j);
  };
  PROF_DECL;
#ifdef RSR_FP4_PROF
  __shared__ long long prof_ts[8];
#endif

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer (both CTAs)
    int stage = p.n_res, gi = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = smem_addr(sA), sB0 = smem_addr(sB);
    const uint32_t bar_b_full = smem_addr(b_full), bar_b_empty = smem_addr(b_empty);
    for (int g = cluster; g < n_groups; g += n_clusters, ++gi) {
      const int ab = gi % p.a_bufs;
      const uint32_t a_par = (uint32_t)(gi / p.a_bufs) & 1;
      // only the sample halves the launch's reference sides need, A_lo first
      for (int h = 0; h < 2; ++h) {
        if (h == 0 ? nt_l == 0 : nt_u == 0) continue;
        const uint32_t bar_af = smem_addr(&a_full[2 * ab + h]);
        const int plane = h == 0 ? 1 : 0;  // A_lo is plane 1, A_up plane 0
        PROF_T(p0);
        mbar_wait(smem_addr(&a_empty[2 * ab + h]), a_par ^ 1);
        PROF_T(p1);
        PROF_ADD(10, p1 - p0);
        if (elect_one()) {
          if (leader)
            mbar_expect_tx(bar_af, 2 * (uint32_t)(p.cq * kChunkA));
          else
            mbar_arrive_leader(bar_af);
          const uint32_t off = p.a_halves == 2 ? (uint32_t)(plane * p.cq * kChunkA) : 0u;
          tma_load_4d_pair(sA0 + (uint32_t)ab * a_buf_bytes + off, &map_a, bar_af, 0,
                           g * 2 * kRowsA + (int)rank * kRowsA, 0, plane);
        }
        __syncwarp();
      }
      if (p.n_res > 0) {
        // small reference sets (or the first n_res tiles of a mid-size set): tile j
        // lives in stage j for the whole launch
        if (gi == 0) {
          for (int j = 0; j < p.n_res; ++j) {
            const bool low = j < p.nt_lower;
            const int y = (low ? j : j - p.nt_lower) * kTileN + (int)rank * kHalfRows;
            if (elect_one()) {
              if (leader)
                mbar_expect_tx(bar_b_full + 8 * j, 2 * b_stage_bytes);
              else
                mbar_arrive_leader(bar_b_full + 8 * j);
              tma_load_3d_pair(sB0 + (uint32_t)j * b_stage_bytes, low ? &map_lower : &map_upper,
                               bar_b_full + 8 * j, 0, y, 0);
            }
            __syncwarp();
          }
        }
        if (p.resident) continue;
      }
      for (int jj = 0; jj < p.nt_total; ++jj) {
        const int j = tile_of(jj);
        if (j < p.n_res) continue;  // resident
        const bool low = j < p.nt_lower;
        // PAIR = 3 (upper side only): the odd tile of a pair needs its 3 main K-steps only;
        // map_lower then holds the 3-chunk map of the upper rows
        const bool short_b = PAIR == 3 && !low && ((j - p.nt_lower) & 1);
        const CUtensorMap* map = (low || short_b) ? &map_lower : &map_upper;
        const uint32_t tx = short_b ? 2u * 3u * (uint32_t)kChunkB : 2 * b_stage_bytes;
        const int y = (low ? j : j - p.nt_lower) * kTileN + (int)rank * kHalfRows;
        PROF_T(q0);
        mbar_wait(bar_b_empty + 8 * stage, phase ^ 1);
        PROF_T(q1);
        PROF_ADD(6, q1 - q0);
        if (elect_one()) {
          if (leader)
            mbar_expect_tx(bar_b_full + 8 * stage, tx);
          else
            mbar_arrive_leader(bar_b_full + 8 * stage);
          tma_load_3d_pair(sB0 + (uint32_t)stage * b_stage_bytes, map, bar_b_full + 8 * stage, 0,
                           y, 0);
        }
        __syncwarp();
        if (++stage == p.stages) {
          stage = p.n_res;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      MmaRole m;
      m.tm0 = __shfl_sync(0xffffffffu, tmem_base, 0);
      m.a_lo0 = desc32_lo(smem_addr(sA));
      m.b_lo0 = desc32_lo(smem_addr(sB));
      m.bar_b_full = smem_addr(b_full);
      m.bar_b_empty = smem_addr(b_empty);
      m.bar_t_full = smem_addr(t_full);
      m.bar_t_empty = smem_addr(t_empty);
      m.bar_a_full = smem_addr(a_full);
      m.bar_a_empty = smem_addr(a_empty);
      m.a_buf_desc = a_buf_bytes >> 4;
      m.b_stage_desc = b_stage_bytes >> 4;
      m.cluster = cluster;
      m.n_clusters = n_clusters;
      m.n_groups = n_groups;
      m.nt_l = nt_l;
      m.nt_u = nt_u;
      m.rot_l = rot_l;
      m.rot_u = rot_u;
#ifdef RSR_FP4_PROF
      m.k_entry = k_entry;
      m.ts = prof_ts;
#endif
      // the K loop fully unrolled for the common row widths (N(M-1) <= 319: 5 K-steps;
      // <= 639: 10): the MMA warp's instruction count per tile is on the critical path
      // once a tile is only ~500 MMA cycles
      switch (p.cq) {
        case 3: mma_role<TN, 3, PAIR>(m, p PROF_ARG); break;
        case 4: mma_role<TN, 4, PAIR>(m, p PROF_ARG); break;
        case 5: mma_role<TN, 5, PAIR>(m, p PROF_ARG); break;
        case 10: mma_role<TN, 10, PAIR>(m, p PROF_ARG); break;
        default: mma_role<TN, 0, PAIR>(m, p PROF_ARG); break;
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue (both CTAs)
    const int quad = warp & 3;            // TMEM lane quarter (hardware: warp id % 4)
    const int set = (warp - 4) >> 2;      // epilogue set: tiles T with T % kEpiSets == set
    const int r = quad * 32 + lane;       // sample row of this thread within the CTA
    uint32_t T = 0;                       // the cluster's tile counter (every set counts all)
    int gpar = 0;
    for (int g = cluster; g < n_groups; g += n_clusters, gpar ^= 1) {
      uint32_t hit = 0;
      int64_t first[2] = {INT64_MAX, INT64_MAX};
      if constexpr (PAIR) {
        // buffers hold tile pairs of one side in the MMA warp's order (mma_role)
        for (int h = 0; h < 2; ++h) {
          const int cnt = h == 0 ? nt_l : nt_u;
          const int base = h == 0 ? 0 : nt_l;
          const int64_t n_side = h == 0 ? p.n_lower : p.n_upper;
          for (int s2 = 0; s2 < cnt; s2 += 2, ++T) {
            constexpr bool kSplit = RSR_FP4_PAIR_SPLIT && PAIR != 2 && kEpiSets == 2;
            if (!kSplit && (int)(T % kEpiSets) != set) continue;
            const uint32_t buf = T % kBufs, tphase = (T / kBufs) & 1;
            const int ja = tile_of(base + s2) - base;
            const int jb = s2 + 1 < cnt ? tile_of(base + s2 + 1) - base : -1;
            const int64_t va = n_side - (int64_t)ja * kTileN;
            const int64_t vb = jb >= 0 ? n_side - (int64_t)jb * kTileN : 0;
            mbar_wait(smem_addr(&t_full[buf]), tphase);
            tc_fence_after();
            const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * kTileN;
            bool any_a, any_b;
            if constexpr (kSplit)
              epilogue_pair_half<kTileN / 2>(taddr + set * (kTileN / 2), smem_addr(&t_empty[buf]),
                                             lane, set * (kTileN / 2), va, vb, any_a, any_b);
            else if constexpr (PAIR == 2)
              epilogue_pair8<kTileN>(taddr, smem_addr(&t_empty[buf]), lane, va, vb, any_a, any_b);
            else
              epilogue_pair<kTileN>(taddr, smem_addr(&t_empty[buf]), lane, va, vb, any_a, any_b);
            if (any_a || any_b) hit |= h == 0 ? RSR_HIT_LOWER : RSR_HIT_UPPER;
          }
        }
      }
      for (int jj = 0; jj < (PAIR ? 0 : p.nt_total); ++jj, ++T) {
        if (!RSR_FP4_SPLIT_COLS && (int)(T % kEpiSets) != set) continue;
        const uint32_t buf = T % kBufs, tphase = (T / kBufs) & 1;
        const int j = tile_of(jj);
        const bool low = j < p.nt_lower;
        const int64_t t0 = (int64_t)(low ? j : j - p.nt_lower) * kTileN;
        PROF_T(e0);
#if RSR_FP4_EPI_SPIN
        mbar_spin(smem_addr(&t_full[buf]), tphase);
#else
        mbar_wait(smem_addr(&t_full[buf]), tphase);
#endif
        PROF_T(e1);
#ifdef RSR_FP4_PROF
        if (rank == 0 && quad == 0) {  // commit issued (MMA warp) -> this warp sees the tile
          PROF_ADD(16, e1 - *(volatile long long*)(prof_ts + buf));
          PROF_ADD(20, 1);
        }
#endif
        tc_fence_after();
        constexpr int kHC = RSR_FP4_SPLIT_COLS ? kTileN / kEpiSets : kTileN;  // columns per warp
        const int c0 = RSR_FP4_SPLIT_COLS ? set * kHC : 0;
        const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * kTileN + c0;
        const int64_t valid = (low ? p.n_lower : p.n_upper) - t0;
        bool any;
        int zref = 0;
        long long t_loaded = 0;
#ifdef RSR_FP4_PROF
        long long* tsr = (rank == 0 && quad == 0) ? prof_ts + 4 + buf : nullptr;
#else
        long long* tsr = nullptr;
#endif
        epilogue_tile<kHC, FIRST>(taddr, smem_addr(&t_empty[buf]), lane, c0, valid, any, zref,
                                  t_loaded, tsr, set);
        PROF_T(e2);
        PROF_ADD(0, t_loaded - e1);
        if (any) {
          hit |= low ? RSR_HIT_LOWER : RSR_HIT_UPPER;
          if (FIRST) {
            const int64_t ref = (low ? p.first_base_lower : p.first_base_upper) + t0 + zref;
            first[low ? 0 : 1] = min(first[low ? 0 : 1], ref);
          }
        }
        PROF_T(e3);
        PROF_ADD(3, e1 - e0);
        PROF_ADD(4, e2 - e1);
        PROF_ADD(5, e3 - e2);
      }
      PROF_T(x0);
      const int64_t row = (int64_t)g * 2 * kRowsA + rank * kRowsA + r;
      if (!FIRST && p.flag_or) {
        // every set ORs its hit bits straight into the flags (zeroed by the launch when
        // not accumulating): four rows' bytes per 32-bit red.or from one lane, no
        // barrier between the sets (the group-end exchange below cost ~4 % at cfg4
        // K = 10^3: profiles/r2_fp4_epilogue_experiments.txt)
        const uint32_t mine = row < S_run ? hit << (8 * (lane & 3)) : 0u;
        uint32_t word = mine | __shfl_xor_sync(0xffffffffu, mine, 1);
        word |= __shfl_xor_sync(0xffffffffu, word, 2);
        if ((lane & 3) == 0 && word)
          atomicOr(reinterpret_cast<unsigned int*>(p.flags + row), word);
      } else {
      // the sets' partial results for the group's rows meet in shared memory; set 0
      // writes the flags.  One barrier per group: the exchange buffers alternate by
      // group parity, so a set may write group g+1's entries while set 0 still reads
      // group g's.
      uint32_t* xh = xchg + gpar * kEpiSets * 128;
      int64_t* xf = xfirst + gpar * kEpiSets * 256;
#ifdef RSR_FP4_X_NOEXCH
      // timing experiment only (wrong results): no group-end exchange between the sets
      if (false) {
#else
      if constexpr (kEpiSets > 1) {
#endif
        if (set != 0) {
          xh[set * 128 + r] = hit;
          if (FIRST) {
            xf[(set * 2 + 0) * 128 + r] = first[0];
            xf[(set * 2 + 1) * 128 + r] = first[1];
          }
        }
        named_bar_sync(1, 32 * kEpiWarps);
      }
      if (set == 0) {
#pragma unroll
        for (int q = 1; q < kEpiSets; ++q) {
          hit |= xh[q * 128 + r];
          if (FIRST) {
            first[0] = min(first[0], xf[(q * 2 + 0) * 128 + r]);
            first[1] = min(first[1], xf[(q * 2 + 1) * 128 + r]);
          }
        }
        if (row < S_run) {
          const uint8_t prev = p.accumulate ? p.flags[row] : 0;
          p.flags[row] = (uint8_t)(prev | hit);
          if (FIRST) {
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
              int64_t* out = sd ? p.first_upper : p.first_lower;
              if (!out) continue;
              const int64_t mine = first[sd] == INT64_MAX ? -1 : first[sd];
              const int64_t old = p.accumulate ? out[row] : -1;  // earlier chunks win
              out[row] = old >= 0 ? old : mine;
            }
          }
        }
      }
      }
      PROF_T(x1);
      PROF_ADD(8, x1 - x0);
    }
  }

#ifdef RSR_FP4_PROF
  const long long k_loop_end = clock64();
#endif
  tc_fence_before();
  cluster_sync_all();
#ifdef RSR_FP4_PROF
  if (warp == 1 && leader) {
    PROF_ADD(13, clock64() - k_loop_end);  // wait for the other roles
    unsigned long long g_exit;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_exit));
    PROF_ADD(14, g_exit - g_entry);          // ns, entry .. teardown (clock = cycles / ns)
    PROF_ADD(15, clock64() - k_entry);       // cycles over the same span
  }
#endif
  PROF_FLUSH;
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

__global__ void clear_flags4_kernel(uint8_t* flags, int64_t S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S) flags[i] = 0;
}

// rows of `row_bytes` viewed as {32 B, rows, chunks} (strides {row_bytes, 32});
// one box = `box_rows` rows x `box_chunks` (default: all) chunks, landing
// chunk-major, 32 B swizzle.
int make_map3(CUtensorMap* map, const void* base, int64_t rows, int row_bytes, int chunks,
              int box_rows, int box_chunks = 0) {
  auto enc = tensor_map_encoder();
  RSR_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  if (box_chunks <= 0) box_chunks = chunks;
  cuuint64_t dims[3] = {(cuuint64_t)kChunk, (cuuint64_t)rows, (cuuint64_t)chunks};
  cuuint64_t strides[2] = {(cuuint64_t)row_bytes, (cuuint64_t)kChunk};
  cuuint32_t box[3] = {(cuuint32_t)kChunk, (cuuint32_t)box_rows, (cuuint32_t)box_chunks};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    rsr::set_error("cuTensorMapEncodeTiled (fp4) failed (%d)", (int)r);
    return RSR_ECUDA;
  }
  return RSR_OK;
}

// Sample operand: {32 B, rows, chunks, 2 halves} with strides {row stride, 32, plane
// stride}; one box = one half (A_up or A_lo) of 128 rows, landing chunk-major.  The
// interleaved layout ([A_up | A_lo] rows) is row stride 2 x row_bytes, plane stride
// row_bytes; the planar one (A_up and A_lo planes) row stride row_bytes: a launch that
// reads one half then streams exactly its bytes (interleaved rows cost 256 B of DRAM
// traffic per 160-byte half: access granularity).
int make_map_a(CUtensorMap* map, const void* base, int64_t rows, int64_t row_stride,
               int64_t plane_stride, int chunks) {
  auto enc = tensor_map_encoder();
  RSR_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[4] = {(cuuint64_t)kChunk, (cuuint64_t)rows, (cuuint64_t)chunks, 2};
  cuuint64_t strides[3] = {(cuuint64_t)row_stride, (cuuint64_t)kChunk, (cuuint64_t)plane_stride};
  cuuint32_t box[4] = {(cuuint32_t)kChunk, (cuuint32_t)kRowsA, (cuuint32_t)chunks, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    rsr::set_error("cuTensorMapEncodeTiled (fp4 samples) failed (%d)", (int)r);
    return RSR_ECUDA;
  }
  return RSR_OK;
}

struct Fp4Call {
  const uint8_t* A;
  int64_t a_row_stride;    // bytes between sample rows (2 x row_bytes interleaved, row_bytes planar)
  int64_t a_plane_stride;  // bytes from a row's A_up half to its A_lo half
  int64_t S;
  const int64_t* S_dev;
  const uint8_t* B[2];   // lower, upper
  int64_t n[2];          // reference rows that count
  int64_t avail[2];      // rows readable from B (rows n..avail-1 are never-hit pad rows)
  int row_bytes;
  uint8_t* flags;
  int64_t* first[2];
  int accumulate;
  cudaStream_t st;
  int sm_count;
  int64_t chunk_tiles;  // reference tiles per launch (0: the L2-sized default)
  int pair;             // paired accumulators (kSfbHiCol): 0 off, 1 2^16 halves, 2 packed 2^8
  int tail;             // shared-tail layout (PAIR = 3; needs a paired plan at 4 K-steps)
  uint32_t sfa_tail_word;
};

constexpr size_t kMinSmem = 120 * 1024;  // > half of the SM's 228 KB

// Shared-memory plan of one launch: sample buffers (one or both halves), the
// reference ring, and whether every tile stays resident for the whole launch.
struct Fp4Layout {
  int a_halves, a_bufs, stages;
  int ring;  // stages that fit next to the sample buffers
  bool resident;
  int n_res;  // resident tiles (all when `resident`; a prefix of a mid-size set otherwise)
  size_t smem;
};

Fp4Layout fp4_layout(int tn, int64_t nt_l, int64_t nt_u, int cq, bool want_first) {
  Fp4Layout L;
  const size_t max_smem = 227 * 1024;
  // align slack, barriers (<= 16 stages x 2 + 18), hit exchange, first-match exchange
  const size_t bars_bytes = (2 * 16 + 26) * 8;
  const size_t fixed = 1024 + bars_bytes + 2 * kEpiSets * 512 + (want_first ? 2 * kEpiSets * 2048 : 0);
  // one-sided launches buffer only the sample half they read
  L.a_halves = (nt_l == 0 || nt_u == 0) ? 1 : 2;
  const size_t a_buf = (size_t)L.a_halves * cq * kChunkA;
  const size_t b_stage = (size_t)cq * (tn / 2) * kChunk;
  const int64_t nt = nt_l + nt_u;
  // sample-group buffers: 3 when a group has few reference tiles (its MMAs are short,
  // so the next groups' A loads must be further ahead), else 2; 1 if smem is short
  const char* ab_env = getenv("RSR_TC_ABUFS");
  L.a_bufs = ab_env ? atoi(ab_env) : (nt <= 16 ? 3 : 2);
  if (L.a_bufs < 1) L.a_bufs = 1;
  if (L.a_bufs > 4) L.a_bufs = 4;
  while (L.a_bufs > 1 && fixed + L.a_bufs * a_buf + 4 * b_stage > max_smem) --L.a_bufs;
  const char* res_env = getenv("RSR_FP4_RESIDENT");
  const bool allow_resident = !(res_env && atoi(res_env) == 0);
  // resident reference tiles are worth more than a third sample buffer
  if (allow_resident && !ab_env && L.a_bufs == 3 && nt <= 16 &&
      fixed + 3 * a_buf + (size_t)nt * b_stage > max_smem &&
      fixed + 2 * a_buf + (size_t)nt * b_stage <= max_smem)
    L.a_bufs = 2;
  int stages = (int)((max_smem - fixed - L.a_bufs * a_buf) / b_stage);
  if (stages > 16) stages = 16;
  // a launch whose reference tiles all fit in the ring keeps them resident
  L.resident = allow_resident && nt <= stages;
  L.n_res = 0;
  if (L.resident) {
    L.ring = stages;
    stages = (int)nt;
    L.n_res = (int)nt;
  } else {
    // mid-size sets (up to twice the ring): all but kHybridRing stages hold a resident
    // prefix of the tiles, the rest stream through a short ring, so each sample group
    // re-loads only the tail of the set (the whole set re-streamed per group cost about
    // 2500 cycles per group just past residency: cfg4 K = 2500, 0.67 of peak).  Resident
    // stages are worth more than a third sample buffer here too.
    const char* hy_env = getenv("RSR_FP4_HYBRID");
    const bool allow_hybrid = allow_resident && !(hy_env && atoi(hy_env) == 0);
    constexpr int kHybridRing = 3;
    // streaming more than kHybridTail tiles through the short ring measured slower than
    // streaming the whole set through the full ring (profiles/r2_fp4_hybrid.txt: K = 2500 /
    // 3000 gain 0.67 -> 0.73 / 0.72 -> 0.76, K = 3500 / 4000 lose 0.82 -> 0.77 / 0.83 -> 0.79)
    constexpr int kHybridTail = 7;
    auto hybrid_ok = [&](int st) {
      return allow_hybrid && st >= kHybridRing + 2 && nt - (st - kHybridRing) <= kHybridTail;
    };
    if (!ab_env && L.a_bufs == 3) {
      const int st2 = (int)std::min<size_t>(16, (max_smem - fixed - 2 * a_buf) / b_stage);
      if (hybrid_ok(st2)) {
        L.a_bufs = 2;
        stages = st2;
      }
    }
    if (hybrid_ok(stages)) L.n_res = stages - kHybridRing;
    L.ring = stages;
  }
  L.stages = stages;
  L.smem = fixed + L.a_bufs * a_buf + (size_t)stages * b_stage;
  // one CTA per SM: a small resident launch must not let a second CTA onto the
  // SM, whose tcgen05.alloc of all 512 columns would wait for the first to exit
  if (L.smem < kMinSmem) L.smem = kMinSmem;
  return L;
}

// Reference chunks: a launch's B slice must stay L2-resident while every group streams
// it (~123K refs x row_bytes per launch: 20 MB at 160 B).  Sets a little past residency
// run as consecutive resident-sized launches instead (pick_tile_n's chunk_tiles).
int64_t launch_chunk_tiles(int tn, int64_t plan_chunk) {
  const char* ct = getenv("RSR_TC_CHUNK_TILES");
  return ct ? atoll(ct) : plan_chunk > 0 ? plan_chunk : 122880 / tn;
}

// Wide rows (N(M-1) >= 832, e.g. N = 295 at M >= 4) leave no room for a sample buffer
// holding both halves next to a reference ring: such calls run the lower and the upper
// tiles as separate one-sided launches (one sample half each, flags and first matches
// accumulated), so they stay on the tensor cores.
bool split_sides_needed(int tn, int64_t nt_l, int64_t nt_u, int cq, bool want_first) {
  return nt_l > 0 && nt_u > 0 && fp4_layout(tn, nt_l, nt_u, cq, want_first).ring < 2;
}

// End of the launch chunk starting at tile c0 (a chunk never straddles the side
// boundary when the sides are split).
int64_t next_chunk_end(int64_t c0, int64_t chunk, int64_t nt_l, int64_t total, bool split_sides) {
  const int64_t lim = (split_sides && c0 < nt_l) ? nt_l : total;
  return c0 + chunk < lim ? c0 + chunk : lim;
}

template <int TN>
int launch_fp4(const Fp4Call& c) {
  const bool want_first = c.first[0] != nullptr || c.first[1] != nullptr;
  const int64_t nt_l = rsr::ceil_div(c.n[0], TN), nt_u = rsr::ceil_div(c.n[1], TN);
  const int cq = c.row_bytes / kChunk;
  // sample operand: one box = one half (A_up or A_lo) of 128 rows; a launch
  // loads only the halves its reference sides need (upper references alone
  // stream half the sample bytes)
  CUtensorMap ma;
  int rc = make_map_a(&ma, c.A, c.S, c.a_row_stride, c.a_plane_stride, cq);
  if (rc) return rc;

  Fp4Params p;
  p.S = c.S;
  p.S_dev = c.S_dev;
  p.cq = cq;
  p.flags = c.flags;
  p.first_lower = c.first[0];
  p.first_upper = c.first[1];
  p.n_groups = (int)rsr::ceil_div(c.S, (int64_t)2 * kRowsA);
  auto kern = want_first ? classify_fp4_pair_kernel<TN, true, 0>
                         : classify_fp4_pair_kernel<TN, false, 0>;
  if constexpr (Tile<TN>::kBufs * TN <= (int)kSfbHiCol) {
    if (c.pair == 1) kern = classify_fp4_pair_kernel<TN, false, 1>;
    if (c.pair == 2) kern = classify_fp4_pair_kernel<TN, false, 2>;
  }
  if constexpr (Tile<TN>::kBufs * TN <= (int)kSfaTailCol)
    if (c.tail) kern = classify_fp4_pair_kernel<TN, false, 3>;
  p.sfa_tail_word = c.sfa_tail_word;
  int clusters = c.sm_count / 2;
  if (p.n_groups < clusters) clusters = p.n_groups;
  p.flag_or = (!want_first && kEpiSets > 1 && (reinterpret_cast<uintptr_t>(c.flags) & 3) == 0 &&
               !getenv("RSR_FP4_FLAG_EXCHANGE"))
                  ? 1
                  : 0;
  if (p.flag_or && !c.accumulate)  // the atomic ORs need zeroed flags: S bytes, one memset
    RSR_CUDA(cudaMemsetAsync(c.flags, 0, (size_t)c.S, c.st));
  const int64_t chunk = launch_chunk_tiles(TN, c.chunk_tiles);
  const bool split_sides = split_sides_needed(TN, nt_l, nt_u, cq, want_first);
  const int64_t total = nt_l + nt_u;
  bool first_launch = true;
  for (int64_t c0 = 0; c0 < total;) {
    const int64_t c1 = next_chunk_end(c0, chunk, nt_l, total, split_sides);
    const int64_t lo[2] = {c0 < nt_l ? c0 : nt_l, (c0 > nt_l ? c0 : nt_l) - nt_l};
    const int64_t hi[2] = {c1 < nt_l ? c1 : nt_l, (c1 > nt_l ? c1 : nt_l) - nt_l};
    Fp4Params q = p;
    q.nt_lower = (int)(hi[0] - lo[0]);
    q.nt_total = (int)((hi[0] - lo[0]) + (hi[1] - lo[1]));
    q.accumulate = first_launch ? c.accumulate : 1;
    q.first_base_lower = lo[0] * TN;
    q.first_base_upper = lo[1] * TN;
    // shared-memory plan of this launch's tiles (one-sided launches buffer one
    // sample half; small launches keep their tiles resident)
    const Fp4Layout L = fp4_layout(TN, q.nt_lower, q.nt_total - q.nt_lower, cq, want_first);
    RSR_REQUIRE(L.ring >= 2, "rsr_classify_fp4: row_bytes too large for shared memory");
    q.a_halves = L.a_halves;
    q.a_bufs = L.a_bufs;
    q.resident = L.resident;
    q.n_res = L.n_res;
    q.stages = L.stages;
    int rc2 = rsr::ensure_dynamic_smem(reinterpret_cast<const void*>(kern), L.smem);
    if (rc2) return rc2;
    // per side: rows the launch's tiles span; when the caller's readable rows
    // cover them (never-hit pad rows past n) no column is masked, otherwise
    // the TMA box reads past n as zeros and the epilogue masks columns >= n
    const uint8_t* base[2];
    int64_t rows[2];
    for (int sd = 0; sd < 2; ++sd) {
      base[sd] = nullptr;
      rows[sd] = 0;
      if (hi[sd] == lo[sd]) continue;
      const int64_t r0 = lo[sd] * TN, span = (hi[sd] - lo[sd]) * TN;
      const int64_t real = (c.n[sd] < r0 + span ? c.n[sd] : r0 + span) - r0;
      rows[sd] = c.avail[sd] - r0 >= span ? span : real;
      base[sd] = c.B[sd] + r0 * (int64_t)c.row_bytes;
    }
    q.n_lower = rows[0];
    q.n_upper = rows[1];

    CUtensorMap cl, cu;
    if (c.tail)  // shared-tail pairs: the odd tiles' 3-chunk map in the (unused) lower slot
      rc = make_map3(&cl, base[1], rows[1], c.row_bytes, 3, TN / 2);
    else
      rc = make_map3(&cl, base[0] ? base[0] : base[1], base[0] ? rows[0] : rows[1], c.row_bytes,
                     cq, TN / 2);
    if (rc) return rc;
    rc = make_map3(&cu, base[1] ? base[1] : base[0], base[1] ? rows[1] : rows[0], c.row_bytes, cq,
                   TN / 2);
    if (rc) return rc;
    kern<<<2 * clusters, kThreads, L.smem, c.st>>>(ma, cl, cu, q);
    rc = rsr::check_launch("classify_fp4_pair_kernel");
    if (rc) return rc;
    first_launch = false;
    c0 = c1;
  }
  return RSR_OK;
}

// MMA N per call: fewest tiles weighted by the measured cost of one tile of
// each width (tools/tile_n_sweep.sh on cfg2: a tile costs about the same down
// to N = 208 -- the per-tile pipeline round trip, not the MMA columns, sets
// it), so narrower tiles only win when they save whole tiles, e.g. 5 x 224
// instead of 5 x 240 is a wash but 1000 refs in 5 x 208 beat 5 x 240 rows of
// which 200 are padding.  RSR_FP4_TILE_N forces one width.
// Whether a call's tiles at width tn fit shared memory: one two-sided launch, or
// (wide rows) the one-sided launches of each side (see launch_fp4).
bool fp4_feasible(int tn, int64_t nt_l, int64_t nt_u, int cq, bool want_first) {
  if (fp4_layout(tn, nt_l, nt_u, cq, want_first).ring >= 2) return true;
  return (nt_l == 0 || fp4_layout(tn, nt_l, 0, cq, want_first).ring >= 2) &&
         (nt_u == 0 || fp4_layout(tn, 0, nt_u, cq, want_first).ring >= 2);
}

// Reference tiles one resident launch can hold at width tn (a two-sided call's chunks
// hold both sides: sized with both sample halves buffered).
int64_t resident_cap(int tn, bool two_sided, int cq, bool want_first) {
  int64_t cap = 0;
  for (int64_t c = 1; c <= 16; ++c) {
    const Fp4Layout L = two_sided && c >= 2 ? fp4_layout(tn, 1, c - 1, cq, want_first)
                                             : fp4_layout(tn, 0, c, cq, want_first);
    if (!L.resident) break;
    cap = c;
  }
  return cap;
}

struct TilePlan {
  int tn;
  int64_t chunk_tiles;  // 0: default (L2-sized chunks, tiles streamed per sample group)
  int pair;             // paired accumulators: rows of <= 4 K-steps, no first matches
};

// Which paired encoding (RSR_FP4_PAIR8=1: packed c1 + 2^8 c2 instead of c1 + 2^16 c2).
int pair_mode() {
  const char* e = getenv("RSR_FP4_PAIR8");
  return e && e[0] == '1' ? 2 : 1;
}

// Paired accumulators (kSfbHiCol) apply to rows of at most 4 K-steps (every count <= 255)
// without first matches, at the widths that leave TMEM room for the second B scale;
// RSR_FP4_PAIR=0 turns them off.
bool pair_eligible(int cq, bool want_first) {
  const char* env = getenv("RSR_FP4_PAIR");
  // 3 K-steps: the paired epilogue's full-width TMEM loads (twice the bytes of the packed
  // loads) outweigh the longer MMA time per buffer (cfg4 K = 10^4: 2.55 ms paired vs
  // 2.45 unpaired); at 4 K-steps pairing lifts the issued-MMA fraction 0.855 -> 0.98
  // (RSR_FP4_PAIR=force: every width up to 4 K-steps, for measurements)
  // Rows of 1-2 K-steps and resident sets measured slower paired too (the paired
  // epilogue's second load round sits on the round trip: tools/pair_small_n.py), so the
  // planner pairs only streamed sets at 4 K-steps (see pick_tile_n).
  if (want_first || cq > 4 || (env && env[0] == '0')) return false;
  return cq == 4 || (env && env[0] == 'f');
}

TilePlan pick_tile_n(int64_t S, int sm_count, int64_t n_lower, int64_t n_upper, int cq,
                     bool want_first) {
  const char* env = getenv("RSR_FP4_TILE_N");
  const int forced = env ? atoi(env) : 0;
  static const int kCand[] = {240, 224, 208, 192, 176, 160};
  static const int kCost[] = {1000, 957, 971, 920, 843, 778};  // relative time per tile
  // resident tiles (cfg4 K = 10^3 per-tile times, profiles/r1_tile_n_small_k.txt)
  static const int kCostResident[] = {1000, 956, 935, 869, 862, 779};
  // paired accumulators: the round trip no longer sets a tile's time.  Plain pairs: a 208
  // tile takes 0.924 of a 224 tile (cfg4 K = 5x10^5: 121.2 vs 121.9 ms); shared-tail pairs
  // (the host's default layout for 193..224 compacted columns): 224 tiles 111.9 ms, 208
  // 118.4, 192 128.0, 176 137.1 (tools/compact_tile_sweep.sh) -- so 224 unless narrower
  // tiles save padding
  static const int kCostPair[] = {0, 1000, 965, 920, 880, 0};
  (void)kCostPair;
  // Streaming the tiles through the ring costs per sample group, over keeping them
  // resident, about 2.5 tiles for short sets (cfg4 K = 2000: 9 resident tiles of 224 take
  // 0.670 ms, 9 streamed tiles of 240 0.891 ms; profiles/r1_tile_n_small_k.txt) and about
  // one tile for long ones (K >= 7000, fitted below).
  // Past residency, the set can instead run as several resident launches, each
  // re-reading the sample operand: a launch's fixed cost (start, prologue, tail; ~24
  // tile-times per cluster) spread over the cluster's sample groups, plus a little per
  // group (cfg4, 2^22 samples: ~0.12 tile per group per extra launch, so 9-tile resident
  // chunks beat streaming up to K ~ 2x10^4: K = 3000 0.78 -> 0.85, 7000 0.844 -> 0.867,
  // 10^4 0.876 -> 0.887, 2x10^4 tie, 4x10^4 streaming ahead;
  // profiles/r2_fp4_chunked_residency.txt).  Smaller batches have fewer groups per cluster
  // and chunk less.
  const int64_t clusters = std::max(1, sm_count / 2);
  const int64_t gpc = std::max<int64_t>(1, rsr::ceil_div(rsr::ceil_div(S, (int64_t)2 * kRowsA),
                                                          clusters));
  const int64_t kChunkGroupCost = 50 + 24000 / gpc;
  constexpr int64_t kMaxChunks = 16;
  const bool pair_ok = pair_eligible(cq, want_first);
  for (int tn : kCand)
    if (tn == forced) return {tn, 0, pair_ok && tn != 240 && tn != 160 ? pair_mode() : 0};
  constexpr int pair = 0;  // the unpaired plan first
  // wide rows (>= 12 K-steps, e.g. N = 295 at M >= 4): N = 160 tiles with three
  // accumulator buffers measured 15 % faster than any wider tile (M = 4: 0.895 of
  // peak vs 0.736-0.776; profiles/r2_wide_rows_m2_m5.txt)
  if (cq >= 12 && fp4_feasible(160, rsr::ceil_div(n_lower, 160), rsr::ceil_div(n_upper, 160), cq,
                               want_first))
    return {160, 0, 0};
  TilePlan best{0, 0, 0};  // tn 0: no width fits shared memory (rows near the 768-byte limit
                         // with first-match exchange buffers)
  int64_t best_cost = INT64_MAX;
  const bool chunk_ok = !getenv("RSR_FP4_NO_CHUNK_RESIDENT");
  for (int i = 0; i < 6; ++i) {
    const int tn = kCand[i];
    if (pair && (tn == 240 || tn == 160)) continue;  // no TMEM room for the second scale
    const int64_t nt_l = rsr::ceil_div(n_lower, tn), nt_u = rsr::ceil_div(n_upper, tn);
    if (!fp4_feasible(tn, nt_l, nt_u, cq, want_first)) continue;
    const bool resident = fp4_layout(tn, nt_l, nt_u, cq, want_first).resident;
    int64_t cost = (nt_l + nt_u) * (pair ? kCostPair[i] : resident ? kCostResident[i] : kCost[i]);
    if (!resident) cost += nt_l + nt_u <= 16 ? 2500 : 1000;  // streaming penalty (above)
    if (cost < best_cost) {
      best_cost = cost;
      best = {tn, 0, pair};
    }
    // resident-sized chunks of a streamed set measured slower paired (cfg4 K = 10^4 at 3
    // K-steps: 3.39 vs 2.55 ms streamed)
    if (resident || !chunk_ok) continue;
    const int64_t nt = nt_l + nt_u;
    const int64_t cap = resident_cap(tn, nt_l > 0 && nt_u > 0, cq, want_first);
    if (cap < 2) continue;
    const int64_t n_ch = rsr::ceil_div(nt, cap);
    if (n_ch > kMaxChunks) continue;
    const int64_t per = rsr::ceil_div(nt, n_ch);
    const int64_t ccost = nt * kCostResident[i] + (n_ch - 1) * kChunkGroupCost;
    if (ccost < best_cost) {
      best_cost = ccost;
      best = {tn, per, pair};
    }
  }
  // a streamed set at 4 K-steps: paired accumulators, the width by kCostPair (cfg4 K =
  // 10^5 / 5x10^5: 0.855-0.90 -> 0.97-0.98 of the MMA rate; a set the unpaired plan keeps
  // resident, whole or in chunks, stays unpaired: K = 2x10^4 0.918 vs 0.85 paired)
  const char* penv = getenv("RSR_FP4_PAIR");
  const bool force = penv && penv[0] == 'f';  // tests / measurements: pair every plan
  if (pair_ok && best.tn && (force || best.chunk_tiles == 0)) {
    const int64_t bl = rsr::ceil_div(n_lower, best.tn), bu = rsr::ceil_div(n_upper, best.tn);
    if (force || !fp4_layout(best.tn, bl, bu, cq, want_first).resident) {
      TilePlan pb{0, 0, pair_mode()};
      int64_t pc = INT64_MAX;
      for (int i = 1; i < 5; ++i) {
        const int tn = kCand[i];
        const int64_t nt_l = rsr::ceil_div(n_lower, tn), nt_u = rsr::ceil_div(n_upper, tn);
        if (!fp4_feasible(tn, nt_l, nt_u, cq, want_first)) continue;
        const int64_t cost = (nt_l + nt_u) * kCostPair[i];
        if (cost < pc) {
          pc = cost;
          pb.tn = tn;
        }
      }
      if (pb.tn) return pb;
    }
  }
  return best;
}

int classify_fp4_impl(const uint8_t* A, int64_t S, const uint8_t* B_lower, int64_t n_lower,
                      int64_t avail_lower, const uint8_t* B_upper, int64_t n_upper,
                      int64_t avail_upper, int row_bytes, uint8_t* flags, int64_t* first_lower,
                      int64_t* first_upper, int accumulate, void* stream,
                      const int64_t* S_dev = nullptr, int64_t a_plane_stride = 0,
                      int tail_tn = 0) {
  RSR_REQUIRE(S >= 0 && n_lower >= 0 && n_upper >= 0, "rsr_classify_fp4: negative size");
  RSR_REQUIRE(avail_lower >= n_lower && avail_upper >= n_upper,
              "rsr_classify_fp4: readable rows below the reference count");
  RSR_REQUIRE(row_bytes >= kChunk && row_bytes % kChunk == 0,
              "rsr_classify_fp4: row_bytes must be a positive multiple of 32");
  RSR_REQUIRE(row_bytes <= RSR_FP4_MAX_ROW_BYTES, "rsr_classify_fp4: row_bytes > %d unsupported",
              RSR_FP4_MAX_ROW_BYTES);
  RSR_REQUIRE(S <= ((int64_t)1 << 31) - 2 * kRowsA, "rsr_classify_fp4: S too large");
  cudaStream_t st = rsr::as_stream(stream);
  if (S == 0) return RSR_OK;
  RSR_REQUIRE(flags != nullptr && A != nullptr, "rsr_classify_fp4: null pointer");
  if (n_lower + n_upper == 0) {
    if (!accumulate) {
      clear_flags4_kernel<<<(unsigned)rsr::ceil_div(S, 256), 256, 0, st>>>(flags, S);
      int rc0 = rsr::check_launch("clear_flags4_kernel");
      if (rc0) return rc0;
      for (int64_t* f : {first_lower, first_upper})
        if (f) RSR_CUDA(cudaMemsetAsync(f, 0xFF, S * sizeof(int64_t), st));  // -1
    }
    return RSR_OK;
  }
  RSR_REQUIRE(rsr::ceil_div(n_lower, 160) + rsr::ceil_div(n_upper, 160) < (1 << 30),
              "rsr_classify_fp4: too many reference tiles");
  RSR_REQUIRE((n_lower == 0 || B_lower) && (n_upper == 0 || B_upper), "rsr_classify_fp4: null refs");
  RSR_REQUIRE(a_plane_stride == 0 || (a_plane_stride % 16 == 0 && a_plane_stride >= S * row_bytes),
              "rsr_classify_fp4: a_plane_stride must be 0 or a multiple of 16 >= S*row_bytes");
  Fp4Call c;
  c.A = A;
  c.a_row_stride = a_plane_stride ? row_bytes : 2 * (int64_t)row_bytes;
  c.a_plane_stride = a_plane_stride ? a_plane_stride : row_bytes;
  c.S = S;
  c.S_dev = S_dev;
  c.B[0] = B_lower;
  c.B[1] = B_upper;
  c.n[0] = n_lower;
  c.n[1] = n_upper;
  c.avail[0] = avail_lower;
  c.avail[1] = avail_upper;
  c.row_bytes = row_bytes;
  c.flags = flags;
  c.first[0] = first_lower;
  c.first[1] = first_upper;
  c.accumulate = accumulate;
  c.st = st;
  int dev = 0;
  RSR_CUDA(cudaGetDevice(&dev));
  RSR_CUDA(cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, dev));
  const TilePlan plan = pick_tile_n(S, c.sm_count, n_lower, n_upper, row_bytes / kChunk,
                                    first_lower != nullptr || first_upper != nullptr);
  if (plan.tn == 0) {
    rsr::set_error("rsr_classify_fp4: %d-byte rows%s do not fit shared memory "
                   "(rsr_classify_fp4_plan reports tile_n 0; use rsr_classify_tc / _bits)",
                   row_bytes, (first_lower || first_upper) ? " with first matches" : "");
    return RSR_EUNSUPPORTED;
  }
  c.chunk_tiles = plan.chunk_tiles;
  c.pair = plan.pair;
  c.tail = 0;
  c.sfa_tail_word = 0;
  if (tail_tn) {
    // the host built the shared-tail layout for pairs of tail_tn-row tiles
    if (plan.pair != 1 || plan.tn != tail_tn || plan.chunk_tiles != 0) {
      rsr::set_error("rsr_classify_fp4_tail: the plan for this call is not a streamed paired "
                     "plan of %d-row tiles (tile_n %d, paired %d)", tail_tn, plan.tn, plan.pair);
      return RSR_EUNSUPPORTED;
    }
    c.tail = 1;
    const char* w = getenv("RSR_FP4_TAIL_SFA");
    c.sfa_tail_word = w ? (uint32_t)strtoul(w, nullptr, 0) : 0x00001000u;
  }
  switch (plan.tn) {
    case 224: return launch_fp4<224>(c);
    case 208: return launch_fp4<208>(c);
    case 192: return launch_fp4<192>(c);
    case 176: return launch_fp4<176>(c);
    case 160: return launch_fp4<160>(c);
    default: return launch_fp4<240>(c);
  }
}

// ---------------------------------------------------------------- encoders
// Sample operand row i: [A_up (row_bytes) | A_lo (row_bytes)] (interleaved) or A_up / A_lo
// planes, element c in byte c/2, low nibble for even c; e2m1 1.0 = 0x2.  A block converts
// kEncRows rows: their states are one contiguous span, staged in shared memory with aligned
// 16-byte loads (one warp per row with byte loads left too few bytes in flight: 0.41 ms per
// 2^20 rows of N = 295, a quarter of the HBM rate), then the threads build whole 32-bit
// words (8 elements) of both halves, item (row, word).
constexpr int kEncRows = 32;

__global__ void __launch_bounds__(256) encode_samples_fp4_kernel(
    const uint8_t* __restrict__ states, int64_t count, int N, int M, uint8_t* __restrict__ out,
    int row_bytes, int kdim, int64_t row_stride, int64_t plane) {
  extern __shared__ __align__(16) uint8_t span[];
  const int64_t r0 = (int64_t)blockIdx.x * kEncRows;
  const int nr = (int)(count - r0 < kEncRows ? count - r0 : kEncRows);
  // aligned 16-byte loads from the span's first aligned address (within the allocation:
  // device allocations are 256-byte aligned), bytewise at the end of the data
  const uint8_t* pbeg = states + r0 * N;
  const uint8_t* pend = pbeg + (int64_t)nr * N;
  const uint8_t* plim = states + count * N;
  const uint8_t* pa = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(pbeg) & ~(uintptr_t)15);
  const int nvec = (int)((pend - pa + 15) >> 4);
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const uint8_t* q = pa + 16 * (int64_t)v;
    if (q + 16 <= plim) {
      reinterpret_cast<uint4*>(span)[v] = *reinterpret_cast<const uint4*>(q);
    } else {
      for (int j = 0; j < 16; ++j) span[16 * v + j] = q + j < plim ? q[j] : 0;
    }
  }
  __syncthreads();
  const uint8_t* rows = span + (pbeg - pa);
  const uint32_t* span32 = reinterpret_cast<const uint32_t*>(span);
  const int words = row_bytes / 4;
  for (int t = threadIdx.x; t < nr * words; t += blockDim.x) {
    const int r = t / words, w = t - r * words;
    uint32_t up, lo;
    const int c0 = 8 * w;
    if (M == 2 && c0 + 8 <= kdim) {
      // 8 states from three aligned shared-memory words and two funnel shifts
      const uint32_t o = (uint32_t)(rows - span) + (uint32_t)(r * N + c0);
      const uint32_t sh = (o & 3u) * 8u, q = o >> 2;
      const uint32_t w0 = span32[q], w1 = span32[q + 1], w2 = span32[q + 2];
      const uint32_t a = __funnelshift_r(w0, w1, sh), b = __funnelshift_r(w1, w2, sh);
      const uint32_t ta = a | (a >> 4), tb = b | (b >> 4);
      lo = __byte_perm(ta, tb, 0x6420) << 1;  // [x >= 1]
      up = lo ^ 0x22222222u;                  // [x <  1]
    } else {
      rsr::fp4_sample_word(rows + r * N, w, M, kdim, up, lo);
    }
    uint8_t* row = out + (r0 + r) * row_stride;
    reinterpret_cast<uint32_t*>(row)[w] = up;
    reinterpret_cast<uint32_t*>(row + plane)[w] = lo;
  }
}

// Sample operand from the reference's own classification input: rows of
// EncodedBatch(kind="sample").packed (encoding.py:82-98: np.packbits of the
// one-hot N x M rows, MSB first).  One warp per row: the packed row is staged
// in shared memory, decoded to states (x_n = position of the set bit of
// component n), then encoded exactly like encode_samples_fp4_kernel.
__global__ void __launch_bounds__(256) unpack_onehot_fp4_kernel(
    const uint8_t* __restrict__ packed, int64_t count, int N, int M, int in_bytes,
    uint8_t* __restrict__ out, int row_bytes, int kdim, int stage_bytes) {
  extern __shared__ uint8_t stage[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* pk = stage + warp * stage_bytes;
  uint8_t* xs = pk + (in_bytes + 15) / 16 * 16;
  const int words = row_bytes / 4;
  for (int64_t i = (int64_t)blockIdx.x * 8 + warp; i < count; i += (int64_t)gridDim.x * 8) {
    const uint8_t* src = packed + i * in_bytes;
    for (int b = lane; b < in_bytes; b += 32) pk[b] = src[b];
    __syncwarp();
    for (int n = lane; n < N; n += 32) {
      int x = 0;
      for (int m = 0; m < M; ++m) {
        const int j = n * M + m;
        if ((pk[j >> 3] >> (7 - (j & 7))) & 1) x = m;
      }
      xs[n] = (uint8_t)x;
    }
    __syncwarp();
    uint32_t* up_row = reinterpret_cast<uint32_t*>(out + i * (int64_t)(2 * row_bytes));
    uint32_t* lo_row = up_row + words;
    for (int w = lane; w < words; w += 32) {
      uint32_t up, lo;
      rsr::fp4_sample_word(xs, w, M, kdim, up, lo);
      up_row[w] = up;
      lo_row[w] = lo;
    }
    __syncwarp();
  }
}

// M = 2 fast path: a block converts kUnpackRows rows.  The rows' packed
// bytes are one contiguous span, staged in shared memory with aligned 16-byte
// loads (the per-thread byte loads of a naive version leave too few bytes in
// flight to reach HBM speed).  Word w of a row is elements 8w..8w+7 = one-hot
// bit pairs 16w..16w+15 = packed bytes 2w, 2w+1 (MSB first): bit 2n is
// [x_n == 0] = A_up, bit 2n+1 is [x_n == 1] = A_lo.
constexpr int kUnpackRows = 128;

__global__ void __launch_bounds__(256) unpack_onehot_fp4_m2_kernel(
    const uint8_t* __restrict__ packed, int64_t rows, int in_bytes, uint8_t* __restrict__ out,
    int words, int kdim) {
  extern __shared__ __align__(16) uint8_t span[];
  const int64_t r0 = (int64_t)blockIdx.x * kUnpackRows;
  const int nr = (int)(rows - r0 < kUnpackRows ? rows - r0 : kUnpackRows);
  const int64_t beg = r0 * in_bytes, end = beg + (int64_t)nr * in_bytes;
  const int64_t abeg = beg & ~(int64_t)15;
  const int nvec = (int)((end - abeg + 15) >> 4);
  const int64_t total = rows * in_bytes;
  for (int v = threadIdx.x; v < nvec; v += blockDim.x) {
    const int64_t off = abeg + 16 * (int64_t)v;
    if (off + 16 <= total) {
      reinterpret_cast<uint4*>(span)[v] = *reinterpret_cast<const uint4*>(packed + off);
    } else {
      for (int j = 0; j < 16; ++j) span[16 * v + j] = off + j < total ? packed[off + j] : 0;
    }
  }
  __syncthreads();
  const int shift = (int)(beg - abeg);
  // (r, w) of flat index t, advanced incrementally (no division per word)
  int r = threadIdx.x / words, w = threadIdx.x - (threadIdx.x / words) * words;
  const int dr = blockDim.x / words, dw = blockDim.x - dr * words;
  for (; r < nr; r += dr, w += dw) {
    if (w >= words) {
      w -= words;
      ++r;
      if (r >= nr) break;
    }
    const uint8_t* src = span + shift + r * in_bytes;
    uint32_t up = 0, lo = 0;
    const int c0 = 8 * w;
    if (c0 + 8 <= kdim) {
      const uint32_t b0 = src[2 * w], b1 = src[2 * w + 1];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        up |= ((b0 >> (7 - 2 * j)) & 1u) << (4 * j + 1);
        lo |= ((b0 >> (6 - 2 * j)) & 1u) << (4 * j + 1);
        up |= ((b1 >> (7 - 2 * j)) & 1u) << (4 * j + 17);
        lo |= ((b1 >> (6 - 2 * j)) & 1u) << (4 * j + 17);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j;
        uint32_t u, l;
        if (c < kdim) {
          const int bu = 2 * c, bl = 2 * c + 1;
          u = (src[bu >> 3] >> (7 - (bu & 7))) & 1u;
          l = (src[bl >> 3] >> (7 - (bl & 7))) & 1u;
        } else {
          u = l = (c == kdim);
        }
        up |= (u ? 0x2u : 0u) << (4 * j);
        lo |= (l ? 0x2u : 0u) << (4 * j);
      }
    }
    uint32_t* row = reinterpret_cast<uint32_t*>(out + (r0 + r) * (int64_t)(8 * words));
    row[w] = up;
    row[words + w] = lo;
  }
}

// Reference operand rows: upper [r_n >= k], lower [r_n < k], bias column 0;
// rows [count, rows_total) are never-hit pad rows (bias column 1).
__global__ void encode_refs_fp4_kernel(const uint8_t* __restrict__ states, int64_t count,
                                       int64_t rows_total, int N, int M, int side,
                                       uint8_t* __restrict__ out, int row_bytes, int kdim) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows_total * row_bytes) return;
  const int64_t r = t / row_bytes;
  const int b = (int)(t - r * row_bytes);
  uint32_t v = 0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = 2 * b + h;
    uint32_t e;
    if (r >= count) {
      e = c == kdim;
    } else if (c < kdim) {
      const int n = c / (M - 1), k = c - n * (M - 1) + 1;
      const uint32_t lt = states[r * N + n] < k;
      e = side == RSR_SIDE_UPPER ? 1 - lt : lt;
    } else {
      e = 0;
    }
    v |= (e ? 0x2u : 0u) << (4 * h);
  }
  out[t] = (uint8_t)v;
}

}  // namespace

#ifdef RSR_FP4_PROF
extern "C" int rsr_fp4_prof(unsigned long long* host8, int reset) {
  RSR_CUDA(cudaMemcpyFromSymbol(host8, g_prof, sizeof(g_prof)));
  if (reset) {
    unsigned long long z[kProf] = {0};
    RSR_CUDA(cudaMemcpyToSymbol(g_prof, z, sizeof(z)));
  }
  return RSR_OK;
}
#endif

extern "C" int rsr_fp4_row_bytes(int n_components, int n_states) {
  if (n_components < 1 || n_states < 2) return 0;
  const int kdim = n_components * (n_states - 1);
  return (kdim + 1 + 63) / 64 * 32;
}

extern "C" int rsr_encode_samples_fp4_ex(const uint8_t* states, int64_t count, int n_components,
                                         int n_states, uint8_t* out, int row_bytes,
                                         int64_t plane_stride, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(plane_stride == 0 || (plane_stride % 16 == 0 && plane_stride >= count * row_bytes),
              "rsr_encode_samples_fp4: plane_stride must be 0 or a multiple of 16 >= count*row_bytes");
  RSR_REQUIRE(N >= 1 && M >= 2 && count >= 0, "rsr_encode_samples_fp4: bad shape");
  RSR_REQUIRE(row_bytes == rsr_fp4_row_bytes(N, M), "rsr_encode_samples_fp4: row_bytes must be %d",
              rsr_fp4_row_bytes(N, M));
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(states != nullptr && out != nullptr, "rsr_encode_samples_fp4: null pointer");
  RSR_REQUIRE((reinterpret_cast<uintptr_t>(out) & 3) == 0,
              "rsr_encode_samples_fp4: out must be 4-byte aligned");
  const size_t smem = ((size_t)kEncRows * N + 48 + 15) / 16 * 16;  // + funnel-load slack
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(encode_samples_fp4_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int64_t grid = rsr::ceil_div(count, kEncRows);
  RSR_REQUIRE(grid < (int64_t)1 << 31, "rsr_encode_samples_fp4: count too large");
  encode_samples_fp4_kernel<<<(unsigned)grid, 256, smem, rsr::as_stream(stream)>>>(
      states, count, N, M, out, row_bytes, N * (M - 1),
      plane_stride ? row_bytes : 2 * (int64_t)row_bytes, plane_stride ? plane_stride : row_bytes);
  return rsr::check_launch("encode_samples_fp4_kernel");
}

extern "C" int rsr_encode_samples_fp4(const uint8_t* states, int64_t count, int n_components,
                                      int n_states, uint8_t* out, int row_bytes, void* stream) {
  return rsr_encode_samples_fp4_ex(states, count, n_components, n_states, out, row_bytes, 0,
                                   stream);
}

extern "C" int rsr_encode_refs_fp4(const uint8_t* states, int64_t count, int64_t rows_total,
                                   int n_components, int n_states, int side, uint8_t* out,
                                   int row_bytes, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(N >= 1 && M >= 2 && count >= 0 && rows_total >= count,
              "rsr_encode_refs_fp4: bad shape");
  RSR_REQUIRE(side == RSR_SIDE_LOWER || side == RSR_SIDE_UPPER, "rsr_encode_refs_fp4: bad side");
  RSR_REQUIRE(row_bytes == rsr_fp4_row_bytes(N, M), "rsr_encode_refs_fp4: row_bytes must be %d",
              rsr_fp4_row_bytes(N, M));
  if (rows_total == 0) return RSR_OK;
  RSR_REQUIRE(out != nullptr && (count == 0 || states != nullptr),
              "rsr_encode_refs_fp4: null pointer");
  const int64_t total = rows_total * row_bytes;
  encode_refs_fp4_kernel<<<(unsigned)rsr::ceil_div(total, 256), 256, 0,
                           rsr::as_stream(stream)>>>(states, count, rows_total, N, M, side, out,
                                                     row_bytes, N * (M - 1));
  return rsr::check_launch("encode_refs_fp4_kernel");
}

extern "C" int rsr_classify_fp4(const uint8_t* A, int64_t S, const uint8_t* B_lower,
                                int64_t n_lower, const uint8_t* B_upper, int64_t n_upper,
                                int row_bytes, uint8_t* flags, int accumulate, void* stream) {
  return classify_fp4_impl(A, S, B_lower, n_lower, n_lower, B_upper, n_upper, n_upper, row_bytes,
                           flags, nullptr, nullptr, accumulate, stream);
}

extern "C" int rsr_classify_fp4_ex(const uint8_t* A, int64_t S, const int64_t* S_dev,
                                   const uint8_t* B_lower, int64_t n_lower, int64_t avail_lower,
                                   const uint8_t* B_upper, int64_t n_upper, int64_t avail_upper,
                                   int row_bytes, uint8_t* flags, int64_t* first_lower,
                                   int64_t* first_upper, int accumulate, void* stream) {
  return classify_fp4_impl(A, S, B_lower, n_lower, avail_lower, B_upper, n_upper, avail_upper,
                           row_bytes, flags, first_lower, first_upper, accumulate, stream, S_dev);
}

extern "C" int rsr_classify_fp4_planar(const uint8_t* A, int64_t a_plane_stride, int64_t S,
                                       const int64_t* S_dev, const uint8_t* B_lower,
                                       int64_t n_lower, int64_t avail_lower,
                                       const uint8_t* B_upper, int64_t n_upper,
                                       int64_t avail_upper, int row_bytes, uint8_t* flags,
                                       int64_t* first_lower, int64_t* first_upper,
                                       int accumulate, void* stream) {
  RSR_REQUIRE(a_plane_stride > 0, "rsr_classify_fp4_planar: a_plane_stride must be > 0");
  return classify_fp4_impl(A, S, B_lower, n_lower, avail_lower, B_upper, n_upper, avail_upper,
                           row_bytes, flags, first_lower, first_upper, accumulate, stream, S_dev,
                           a_plane_stride);
}

extern "C" int rsr_classify_fp4_tail(const uint8_t* A, int64_t a_plane_stride, int64_t S,
                                     const uint8_t* B_upper, int64_t n_upper, int row_bytes,
                                     int tile_n, uint8_t* flags, int accumulate, void* stream) {
  RSR_REQUIRE(row_bytes == 4 * kChunk, "rsr_classify_fp4_tail: rows must be 4 K-steps (128 B)");
  RSR_REQUIRE(tile_n == 224 || tile_n == 208 || tile_n == 192 || tile_n == 176,
              "rsr_classify_fp4_tail: tile_n must be 176..224");
  RSR_REQUIRE(n_upper % (2 * tile_n) == 0,
              "rsr_classify_fp4_tail: n_upper must be whole tile pairs (pad with never-hit rows)");
  RSR_REQUIRE(a_plane_stride > 0, "rsr_classify_fp4_tail: planar sample operand required");
  return classify_fp4_impl(A, S, nullptr, 0, 0, B_upper, n_upper, n_upper, row_bytes, flags,
                           nullptr, nullptr, accumulate, stream, nullptr, a_plane_stride, tile_n);
}

extern "C" int rsr_classify_fp4_plan_ex(int64_t S, int64_t n_lower, int64_t n_upper,
                                        int row_bytes, int want_first, int* tile_n,
                                        int64_t* launches, int* paired) {
  int rc = rsr_classify_fp4_plan(S, n_lower, n_upper, row_bytes, want_first, tile_n, launches);
  if (rc || !paired) return rc;
  int sm_count = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sm_count = v;
  }
  cudaGetLastError();
  const TilePlan plan = pick_tile_n(S, sm_count, n_lower, n_upper, row_bytes / kChunk,
                                    want_first != 0);
  *paired = plan.pair == 1 && plan.chunk_tiles == 0 ? 1 : 0;
  return RSR_OK;
}

extern "C" int rsr_classify_fp4_dev(const uint8_t* A, int64_t S_cap, const int64_t* S_dev,
                                    const uint8_t* B_lower, int64_t n_lower, const uint8_t* B_upper,
                                    int64_t n_upper, int row_bytes, uint8_t* flags, int accumulate,
                                    void* stream) {
  RSR_REQUIRE(S_dev != nullptr, "rsr_classify_fp4_dev: null device count");
  return classify_fp4_impl(A, S_cap, B_lower, n_lower, n_lower, B_upper, n_upper, n_upper,
                           row_bytes, flags, nullptr, nullptr, accumulate, stream, S_dev);
}

extern "C" int rsr_classify_fp4_explain(const uint8_t* A, int64_t S, const uint8_t* B_lower,
                                        int64_t n_lower, const uint8_t* B_upper, int64_t n_upper,
                                        int row_bytes, uint8_t* flags, int64_t* first_lower,
                                        int64_t* first_upper, int accumulate, void* stream) {
  return classify_fp4_impl(A, S, B_lower, n_lower, n_lower, B_upper, n_upper, n_upper, row_bytes,
                           flags, first_lower, first_upper, accumulate, stream);
}

extern "C" int rsr_classify_fp4_plan(int64_t S, int64_t n_lower, int64_t n_upper, int row_bytes,
                                     int want_first, int* tile_n, int64_t* launches) {
  RSR_REQUIRE(S >= 0 && n_lower >= 0 && n_upper >= 0, "rsr_classify_fp4_plan: negative size");
  RSR_REQUIRE(row_bytes >= kChunk && row_bytes % kChunk == 0 && row_bytes <= RSR_FP4_MAX_ROW_BYTES,
              "rsr_classify_fp4_plan: bad row_bytes");
  RSR_REQUIRE(tile_n && launches, "rsr_classify_fp4_plan: null output");
  const int cq = row_bytes / kChunk;
  int sm_count = 148;  // host-only query: the current device's SM count when there is one
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
      sm_count = v;
  }
  cudaGetLastError();  // no device: clear the sticky error of the probe
  const TilePlan plan = pick_tile_n(S, sm_count, n_lower, n_upper, cq, want_first != 0);
  *tile_n = plan.tn;
  *launches = 0;
  if (plan.tn == 0) return RSR_OK;  // infeasible: no width fits shared memory
  const int64_t nt_l = rsr::ceil_div(n_lower, plan.tn), nt_u = rsr::ceil_div(n_upper, plan.tn);
  const int64_t total = nt_l + nt_u, chunk = launch_chunk_tiles(plan.tn, plan.chunk_tiles);
  const bool split = split_sides_needed(plan.tn, nt_l, nt_u, cq, want_first != 0);
  int64_t n = 0;
  for (int64_t c0 = 0; c0 < total; c0 = next_chunk_end(c0, chunk, nt_l, total, split)) ++n;
  *tile_n = plan.tn;
  *launches = n;
  return RSR_OK;
}

extern "C" int rsr_unpack_onehot_fp4(const uint8_t* packed, int64_t count, int n_components,
                                     int n_states, uint8_t* out, int row_bytes, void* stream) {
  const int N = n_components, M = n_states;
  RSR_REQUIRE(N >= 1 && M >= 2 && M <= 255 && count >= 0, "rsr_unpack_onehot_fp4: bad shape");
  RSR_REQUIRE(row_bytes == rsr_fp4_row_bytes(N, M), "rsr_unpack_onehot_fp4: row_bytes must be %d",
              rsr_fp4_row_bytes(N, M));
  if (count == 0) return RSR_OK;
  RSR_REQUIRE(packed != nullptr && out != nullptr, "rsr_unpack_onehot_fp4: null pointer");
  const int in_bytes = (N * M + 7) / 8;
  if (M == 2) {
    const size_t span = ((size_t)kUnpackRows * in_bytes + 31) / 16 * 16;
    if (span > 48 * 1024)
      RSR_CUDA(cudaFuncSetAttribute(unpack_onehot_fp4_m2_kernel,
                                    cudaFuncAttributeMaxDynamicSharedMemorySize, (int)span));
    unpack_onehot_fp4_m2_kernel<<<(unsigned)rsr::ceil_div(count, kUnpackRows), 256, span,
                                   rsr::as_stream(stream)>>>(packed, count, in_bytes, out,
                                                             row_bytes / 4, N);
    return rsr::check_launch("unpack_onehot_fp4_m2_kernel");
  }
  const int stage_bytes = (in_bytes + 15) / 16 * 16 + (N + 15) / 16 * 16;
  const size_t smem = 8 * (size_t)stage_bytes;
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(unpack_onehot_fp4_kernel,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int64_t grid = rsr::ceil_div(count, 8);
  if (grid > 148 * 64) grid = 148 * 64;
  unpack_onehot_fp4_kernel<<<(unsigned)grid, 256, smem, rsr::as_stream(stream)>>>(
      packed, count, N, M, in_bytes, out, row_bytes, N * (M - 1), stage_bytes);
  return rsr::check_launch("unpack_onehot_fp4_kernel");
}
