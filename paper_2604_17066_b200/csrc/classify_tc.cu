// (2) Dominance classification on tcgen05 int8 tensor cores.
//
// Replaces classify.py:99-148 (_chunk_hits / _hits_for: popcount of
// sample & ~ref over bit-packed rows, any-zero per sample) and the precedence
// step classify.py:240-241.  The violation product is recast as a thermometer
// contraction D = A . B^T (see include/rsr_b200.h): A = [x_n < k] samples,
// B = refs with a bias column, D >= 0 and D == 0 <=> dominated.  The S x K
// matrix D never leaves TMEM: the epilogue reduces each accumulator row to a
// min and ORs a hit bit per side.
//
// Kernel shape (persistent, one CTA per SM):
//   * a "group" is MT x 128 sample rows; its A tiles (MT x KB x 16 KB, K-major,
//     128-byte swizzle) are loaded once by TMA and stay resident while every
//     reference tile streams past;
//   * reference tiles are 128 rows; each k-block (128 bytes of K) of a tile is
//     one pipeline stage (16 KB), STAGES deep;
//   * warp 0 = TMA producer, warp 1 = MMA issuer (one thread issues
//     tcgen05.mma.cta_group::1.kind::i8, M=128 N=128 K=32), warp 2 = TMEM
//     allocator, warps 4 .. 4+4*MT-1 = epilogue (one thread per sample row,
//     tcgen05.ld 32x32b, min-reduce over 128 columns);
//   * TMEM holds 2 buffers x MT accumulators of 128 int32 columns, so the
//     epilogue of tile j overlaps the MMAs of tile j+1.
#include <stdlib.h>

#include "tc_common.cuh"

namespace {

constexpr int kTileM = 128;
constexpr int kTileN = 128;
constexpr int kKBlock = 128;  // bytes of K per swizzle atom row
constexpr int kKStep = 32;    // UMMA K for kind::i8
constexpr int kTileBytes = kTileM * kKBlock;  // 16 KB

struct TcParams {
  int64_t S;
  int n_groups;
  int kb;           // k-blocks per row
  int ksteps_last;  // UMMA k-steps in the last k-block
  int nt_lower;     // reference tiles holding lower refs (come first)
  int nt_total;
  int stages;
  uint8_t* flags;
  int accumulate;
  int debug;  // RSR_TC_DEBUG: bit0 = no B reloads after the first ring, bit1 = no TMEM loads
  int a_bufs;  // pair kernel: 1 or 2 sample-tile buffers
  int64_t* first_lower;  // pair kernel FIRST variant: smallest matching ref index, -1 if none
  int64_t* first_upper;
  int64_t first_base_lower;  // reference index of this launch's first lower / upper row
  int64_t first_base_upper;
};

// Reference tiles are visited in a per-CTA rotated order so that the 148 SMs
// do not all stream the same tile out of the same L2 slices at once; the
// OR-reduction of hits is order independent.
__device__ __forceinline__ int tile_at(int j, int rot, int nt) {
  const int t = j + rot;
  return t >= nt ? t - nt : t;
}

template <int MT>
__global__ void __launch_bounds__(128 + 128 * MT, 1)
classify_tc_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_lower,
                   const __grid_constant__ CUtensorMap map_upper, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte alignment for the 128-byte swizzle atoms.
  const uint32_t raw_addr = smem_addr(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)MT * p.kb * kTileBytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)p.stages * kTileBytes);
  uint64_t* b_full = bars;
  uint64_t* b_empty = bars + p.stages;
  uint64_t* a_full = bars + 2 * p.stages;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_full + 2;   // [2]
  uint64_t* t_empty = a_full + 4;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 6);

  constexpr uint32_t kTmemCols = MT == 2 ? 512 : 256;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lower)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_upper)));
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(smem_addr(&b_full[i]), 1);
      mbar_init(smem_addr(&b_empty[i]), 1);
    }
    mbar_init(smem_addr(a_full), 1);
    mbar_init(smem_addr(a_empty), 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_addr(&t_full[i]), 1);
      mbar_init(smem_addr(&t_empty[i]), 4 * MT);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int rot = (int)(((int64_t)blockIdx.x * p.nt_total) / gridDim.x);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer
    // The whole warp runs the (warp-uniform) loop so addresses and coordinates
    // stay in uniform registers; one elected lane issues each TMA.
    int stage = 0, loads = 0;
    uint32_t phase = 0, a_phase = 0;
    const uint32_t sA0 = smem_addr(sA), sB0 = smem_addr(sB);
    const uint32_t bar_b_full = smem_addr(b_full), bar_b_empty = smem_addr(b_empty);
    for (int g = blockIdx.x; g < p.n_groups; g += gridDim.x) {
      mbar_wait(smem_addr(a_empty), a_phase ^ 1);
      if (elect_one()) {
        mbar_expect_tx(smem_addr(a_full), (uint32_t)(MT * p.kb * kTileBytes));
        for (int mt = 0; mt < MT; ++mt)
          for (int kb = 0; kb < p.kb; ++kb)
            tma_load_2d(sA0 + (uint32_t)(mt * p.kb + kb) * kTileBytes, &map_a, smem_addr(a_full),
                        kb * kKBlock, (g * MT + mt) * kTileM);
      }
      __syncwarp();
      a_phase ^= 1;
      for (int jj = 0; jj < p.nt_total; ++jj) {
        const int j = tile_at(jj, rot, p.nt_total);
        const bool low = j < p.nt_lower;
        const CUtensorMap* map = low ? &map_lower : &map_upper;
        const int y = (low ? j : j - p.nt_lower) * kTileN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(bar_b_empty + 8 * stage, phase ^ 1);
          if (elect_one()) {
            if ((p.debug & 1) && loads >= p.stages) {
              mbar_arrive(bar_b_full + 8 * stage);
            } else {
              mbar_expect_tx(bar_b_full + 8 * stage, (uint32_t)kTileBytes);
              tma_load_2d(sB0 + (uint32_t)stage * kTileBytes, map, bar_b_full + 8 * stage,
                          kb * kKBlock, y);
            }
          }
          __syncwarp();
          ++loads;
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer
    // Warp-uniform loop; descriptors are precomputed 32-bit words so each MMA
    // costs two uniform adds (a single-lane loop would force an R2UR
    // waterfall per MMA and cap the issue rate well below the tensor pipe).
    constexpr uint32_t idesc = i8_idesc(kTileM, kTileN);
    const uint32_t tm0 = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint32_t a_lo0 = desc_lo(smem_addr(sA)), b_lo0 = desc_lo(smem_addr(sB));
    const uint32_t bar_b_full = smem_addr(b_full), bar_b_empty = smem_addr(b_empty);
    const int kb_full = (p.ksteps_last == kKBlock / kKStep) ? p.kb : p.kb - 1;
    int stage = 0;
    uint32_t phase = 0, a_phase = 0, tc = 0;
    for (int g = blockIdx.x; g < p.n_groups; g += gridDim.x) {
      mbar_wait(smem_addr(a_full), a_phase);
      a_phase ^= 1;
      tc_fence_after();
      for (int j = 0; j < p.nt_total; ++j, ++tc) {
        const uint32_t buf = tc & 1, tphase = (tc >> 1) & 1;
        mbar_wait_inline(smem_addr(&t_empty[buf]), tphase ^ 1);  // tc_common.cuh: why inline
        tc_fence_after();
        const uint32_t d0 = tm0 + buf * MT * kTileN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(bar_b_full + 8 * stage, phase);
          tc_fence_after();
          const uint32_t bl = b_lo0 + (uint32_t)stage * (kTileBytes >> 4);
          if (elect_one()) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint32_t al = a_lo0 + (uint32_t)(mt * p.kb + kb) * (kTileBytes >> 4);
              const uint32_t d = d0 + mt * kTileN;
              if (kb < kb_full) {
#pragma unroll
                for (int ks = 0; ks < kKBlock / kKStep; ++ks)
                  umma_i8_lo(d, al + ks * (kKStep >> 4), bl + ks * (kKStep >> 4), idesc,
                             (kb | ks) != 0);
              } else {
                for (int ks = 0; ks < p.ksteps_last; ++ks)
                  umma_i8_lo(d, al + ks * (kKStep >> 4), bl + ks * (kKStep >> 4), idesc,
                             (kb | ks) != 0);
              }
            }
            umma_commit(bar_b_empty + 8 * stage);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit(smem_addr(&t_full[buf]));
        __syncwarp();
      }
      if (elect_one()) umma_commit(smem_addr(a_empty));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue
    const int mt = (warp - 4) >> 2;
    const int quad = warp & 3;
    uint32_t tc = 0;
    for (int g = blockIdx.x; g < p.n_groups; g += gridDim.x) {
      uint32_t hit = 0;
      for (int jj = 0; jj < p.nt_total; ++jj, ++tc) {
        const int j = tile_at(jj, rot, p.nt_total);
        const uint32_t buf = tc & 1, tphase = (tc >> 1) & 1;
        mbar_wait(smem_addr(&t_full[buf]), tphase);
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quad * 32) << 16) + (buf * MT + mt) * kTileN;
        uint32_t mn = 0xFFFFFFFFu;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (p.debug & 2) {
            mn = 1;
            break;
          }
          uint32_t v[64];
          RSR_LD32(taddr + half * 64, v);
          RSR_LD32(taddr + half * 64 + 32, (v + 32));
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 64; ++i) mn = min(mn, v[i]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_addr(&t_empty[buf]));
        if (mn == 0) hit |= (j < p.nt_lower) ? RSR_HIT_LOWER : RSR_HIT_UPPER;
      }
      const int64_t row = ((int64_t)g * MT + mt) * kTileM + quad * 32 + lane;
      if (row < p.S) {
        const uint8_t prev = p.accumulate ? p.flags[row] : 0;
        p.flags[row] = (uint8_t)(prev | hit);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

// ---------------------------------------------------------------------------
// CTA-pair variant (default): cta_group::2, one MMA = 256 samples x 256 refs
// x 32 K.  A cluster of two CTAs on one TPC owns a group of 256 sample rows
// (128 per CTA, resident in shared memory); every reference tile of 256 rows
// is split 128/128 between the two CTAs' shared memory.  The leader CTA
// (rank 0) issues the MMAs; each CTA's TMEM holds the 128 x 256 int32
// accumulator of its own rows (2 buffers = 512 columns).  Per unit of work
// this halves the MMA instruction count and each SM's operand reads compared
// with the 1-SM M=128/N=128 kernel above, at the same L2 traffic.
//   barriers (leader copy used unless noted):
//     b_full[s]  count 2 (leader arrive.expect_tx + peer arrive) + TMA bytes of both CTAs
//     b_empty[s] per CTA, count 1 (multicast tcgen05.commit)
//     a_full     count 2, like b_full;  a_empty per CTA (multicast commit)
//     t_full[b]  per CTA, count 1 (multicast commit)
//     t_empty[b] count 16 (8 epilogue warps x 2 CTAs, remote arrives)
constexpr int kPairN = 256;

__device__ __forceinline__ void umma_i8_pair(uint32_t d_tmem, uint32_t a_lo, uint32_t b_lo,
                                             uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "mov.b64 da, {%1, %5};\n\t"
      "mov.b64 db, {%2, %5};\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], da, db, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_lo), "r"(b_lo), "r"(idesc), "r"(accumulate), "r"(kDescHi));
}

template <bool FIRST>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
classify_tc_pair_kernel(const __grid_constant__ CUtensorMap map_a,
                        const __grid_constant__ CUtensorMap map_lower,
                        const __grid_constant__ CUtensorMap map_upper, const TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_addr(smem_raw);
  uint8_t* smem = smem_raw + ((1024u - (raw_addr & 1023u)) & 1023u);
  // a_bufs x kb x 16 KB of A (this CTA's 128 rows; double-buffered so the next
  // group's samples load while the current group's MMAs run), then the B ring.
  uint8_t* sA = smem;
  uint8_t* sB = sA + (size_t)p.a_bufs * p.kb * kTileBytes;  // stages x 16 KB (128 ref rows)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)p.stages * kTileBytes);
  uint64_t* b_full = bars;
  uint64_t* b_empty = bars + p.stages;
  uint64_t* a_full = bars + 2 * p.stages;  // [2]
  uint64_t* a_empty = a_full + 2;          // [2]
  uint64_t* t_full = a_full + 4;           // [2]
  uint64_t* t_empty = a_full + 6;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(a_full + 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1;
  const int n_clusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_lower)));
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_upper)));
    for (int i = 0; i < p.stages; ++i) {
      mbar_init(smem_addr(&b_full[i]), 2);
      mbar_init(smem_addr(&b_empty[i]), 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(smem_addr(&a_full[i]), 2);
      mbar_init(smem_addr(&a_empty[i]), 1);
      mbar_init(smem_addr(&t_full[i]), 1);
      mbar_init(smem_addr(&t_empty[i]), 16);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        smem_addr(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int rot = (int)(((int64_t)cluster * p.nt_total) / n_clusters);

  if (warp == 0) {
    // ------------------------------------------------------ TMA producer (both CTAs)
    int stage = 0, gi = 0;
    uint32_t phase = 0;
    const uint32_t sA0 = smem_addr(sA), sB0 = smem_addr(sB);
    const uint32_t bar_b_full = smem_addr(b_full), bar_b_empty = smem_addr(b_empty);
    const uint32_t a_bytes = (uint32_t)(2 * p.kb * kTileBytes);
    for (int g = cluster; g < p.n_groups; g += n_clusters, ++gi) {
      const int ab = gi % p.a_bufs;
      const uint32_t a_par = (uint32_t)(gi / p.a_bufs) & 1;
      const uint32_t bar_af = smem_addr(&a_full[ab]);
      mbar_wait(smem_addr(&a_empty[ab]), a_par ^ 1);
      if (elect_one()) {
        if (leader)
          mbar_expect_tx(bar_af, a_bytes);
        else
          mbar_arrive_leader(bar_af);
        for (int kb = 0; kb < p.kb; ++kb)
          tma_load_2d_pair(sA0 + (uint32_t)(ab * p.kb + kb) * kTileBytes, &map_a, bar_af,
                           kb * kKBlock, g * 2 * kTileM + (int)rank * kTileM);
      }
      __syncwarp();
      for (int jj = 0; jj < p.nt_total; ++jj) {
        const int j = tile_at(jj, rot, p.nt_total);
        const bool low = j < p.nt_lower;
        const CUtensorMap* map = low ? &map_lower : &map_upper;
        const int y = (low ? j : j - p.nt_lower) * kPairN + (int)rank * kTileN;
        for (int kb = 0; kb < p.kb; ++kb) {
          mbar_wait(bar_b_empty + 8 * stage, phase ^ 1);
          if (elect_one()) {
            if (leader)
              mbar_expect_tx(bar_b_full + 8 * stage, (uint32_t)(2 * kTileBytes));
            else
              mbar_arrive_leader(bar_b_full + 8 * stage);
            tma_load_2d_pair(sB0 + (uint32_t)stage * kTileBytes, map, bar_b_full + 8 * stage,
                             kb * kKBlock, y);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------ MMA issuer (leader only)
    if (leader) {
      constexpr uint32_t idesc = i8_idesc(2 * kTileM, kPairN);
      const uint32_t tm0 = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t a_lo0 = desc_lo(smem_addr(sA)), b_lo0 = desc_lo(smem_addr(sB));
      const uint32_t bar_b_full = smem_addr(b_full), bar_b_empty = smem_addr(b_empty);
      const int kb_full = (p.ksteps_last == kKBlock / kKStep) ? p.kb : p.kb - 1;
      int stage = 0, gi = 0;
      uint32_t phase = 0, tc = 0;
      for (int g = cluster; g < p.n_groups; g += n_clusters, ++gi) {
        const int ab = gi % p.a_bufs;
        mbar_wait(smem_addr(&a_full[ab]), (uint32_t)(gi / p.a_bufs) & 1);
        tc_fence_after();
        const uint32_t a_lo_g = a_lo0 + (uint32_t)(ab * p.kb) * (kTileBytes >> 4);
        for (int j = 0; j < p.nt_total; ++j, ++tc) {
          const uint32_t buf = tc & 1, tphase = (tc >> 1) & 1;
          mbar_wait_inline(smem_addr(&t_empty[buf]), tphase ^ 1);  // tc_common.cuh: why inline
          tc_fence_after();
          const uint32_t d = tm0 + buf * kPairN;
          for (int kb = 0; kb < p.kb; ++kb) {
            mbar_wait(bar_b_full + 8 * stage, phase);
            tc_fence_after();
            const uint32_t bl = b_lo0 + (uint32_t)stage * (kTileBytes >> 4);
            const uint32_t al = a_lo_g + (uint32_t)kb * (kTileBytes >> 4);
            if (elect_one()) {
              if (kb < kb_full) {
#pragma unroll
                for (int ks = 0; ks < kKBlock / kKStep; ++ks)
                  umma_i8_pair(d, al + ks * (kKStep >> 4), bl + ks * (kKStep >> 4), idesc,
                               (kb | ks) != 0);
              } else {
                for (int ks = 0; ks < p.ksteps_last; ++ks)
                  umma_i8_pair(d, al + ks * (kKStep >> 4), bl + ks * (kKStep >> 4), idesc,
                               (kb | ks) != 0);
              }
              umma_commit_pair(bar_b_empty + 8 * stage);
            }
            __syncwarp();
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (elect_one()) umma_commit_pair(smem_addr(&t_full[buf]));
          __syncwarp();
        }
        if (elect_one()) umma_commit_pair(smem_addr(&a_empty[ab]));
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------ epilogue (both CTAs)
    const int quad = warp & 3;
    const int colhalf = (warp - 4) >> 2;
    uint32_t tc = 0;
    for (int g = cluster; g < p.n_groups; g += n_clusters) {
      uint32_t hit = 0;
      // FIRST: smallest matching reference index per side (accumulator column n
      // of pair tile j is reference j*256 + n: columns 0-127 come from CTA 0's
      // B half, 128-255 from CTA 1's)
      int64_t first[2] = {INT64_MAX, INT64_MAX};
      for (int jj = 0; jj < p.nt_total; ++jj, ++tc) {
        const int j = tile_at(jj, rot, p.nt_total);
        const uint32_t buf = tc & 1, tphase = (tc >> 1) & 1;
        mbar_wait(smem_addr(&t_full[buf]), tphase);
        tc_fence_after();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(quad * 32) << 16) + buf * kPairN + colhalf * kTileN;
        uint32_t mn = 0xFFFFFFFFu;
        int zero_col = -1;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
          if (p.debug & 2) {
            mn = 1;
            break;
          }
          uint32_t v[64];
          RSR_LD32(taddr + half * 64, v);
          RSR_LD32(taddr + half * 64 + 32, (v + 32));
          tmem_ld_wait();
          uint32_t mh = 0xFFFFFFFFu;
#pragma unroll
          for (int i = 0; i < 64; ++i) mh = min(mh, v[i]);
          if (FIRST && mh == 0 && zero_col < 0) {
            for (int i = 0; i < 64; ++i)
              if (v[i] == 0) {
                zero_col = half * 64 + i;
                break;
              }
          }
          mn = min(mn, mh);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_leader(smem_addr(&t_empty[buf]));
        if (mn == 0) {
          const bool low = j < p.nt_lower;
          hit |= low ? RSR_HIT_LOWER : RSR_HIT_UPPER;
          if (FIRST) {
            const int64_t ref = (low ? p.first_base_lower + (int64_t)j * kPairN
                                     : p.first_base_upper + (int64_t)(j - p.nt_lower) * kPairN) +
                                colhalf * kTileN + zero_col;
            first[low ? 0 : 1] = min(first[low ? 0 : 1], ref);
          }
        }
      }
      // the two column halves of a row live in two warps: combine through smem-free
      // atomics on the flags byte would race, so OR via a warp-pair exchange instead
      const int64_t row = (int64_t)g * 2 * kTileM + rank * kTileM + quad * 32 + lane;
      uint32_t* xchg = reinterpret_cast<uint32_t*>(a_full + 10);  // [128] scratch
      int64_t* xfirst = reinterpret_cast<int64_t*>(xchg + 128);   // [2][128] (FIRST)
      named_bar_sync(1, 256);
      if (colhalf == 1) {
        xchg[quad * 32 + lane] = hit;
        if (FIRST) {
          xfirst[quad * 32 + lane] = first[0];
          xfirst[128 + quad * 32 + lane] = first[1];
        }
      }
      named_bar_sync(1, 256);
      if (colhalf == 0) {
        hit |= xchg[quad * 32 + lane];
        if (row < p.S) {
          const uint8_t prev = p.accumulate ? p.flags[row] : 0;
          p.flags[row] = (uint8_t)(prev | hit);
          if (FIRST) {
#pragma unroll
            for (int sd = 0; sd < 2; ++sd) {
              int64_t* out = sd ? p.first_upper : p.first_lower;
              if (!out) continue;
              const int64_t f = min(first[sd], xfirst[sd * 128 + quad * 32 + lane]);
              const int64_t mine = f == INT64_MAX ? -1 : f;
              // chunks run in increasing reference order: an earlier chunk's hit wins
              const int64_t old = p.accumulate ? out[row] : -1;
              out[row] = old >= 0 ? old : mine;
            }
          }
        }
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base));
  }
}

__global__ void clear_flags_kernel(uint8_t* flags, int64_t S) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S) flags[i] = 0;
}

int make_map(CUtensorMap* map, const void* base, int64_t rows, int kpad) {
  auto enc = tensor_map_encoder();
  RSR_REQUIRE(enc != nullptr, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {(cuuint64_t)kpad, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kpad};
  cuuint32_t box[2] = {(cuuint32_t)kKBlock, (cuuint32_t)kTileM};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    rsr::set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return RSR_ECUDA;
  }
  return RSR_OK;
}

template <int MT>
int launch_tc(const CUtensorMap& ma, const CUtensorMap& ml, const CUtensorMap& mu, TcParams p,
              size_t smem, int sm_count, cudaStream_t st) {
  auto k = classify_tc_kernel<MT>;
  RSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = p.n_groups < sm_count ? p.n_groups : sm_count;
  k<<<grid, 128 + 128 * MT, smem, st>>>(ma, ml, mu, p);
  return rsr::check_launch("classify_tc_kernel");
}

}  // namespace

namespace {

int classify_tc_impl(const int8_t* A, int64_t S, const int8_t* B_lower, int64_t n_lower,
                     const int8_t* B_upper, int64_t n_upper, int Kpad, uint8_t* flags,
                     int accumulate, int64_t* first_lower, int64_t* first_upper, void* stream) {
  const bool want_first = first_lower != nullptr || first_upper != nullptr;
  RSR_REQUIRE(S >= 0 && n_lower >= 0 && n_upper >= 0, "rsr_classify_tc: negative size");
  RSR_REQUIRE(Kpad >= 32 && Kpad % 32 == 0, "rsr_classify_tc: Kpad must be a multiple of 32");
  RSR_REQUIRE(Kpad <= 6 * kKBlock, "rsr_classify_tc: Kpad > 768 unsupported");
  RSR_REQUIRE(S <= ((int64_t)1 << 31) - kTileM * 2, "rsr_classify_tc: S too large");
  cudaStream_t st = rsr::as_stream(stream);
  if (S == 0) return RSR_OK;
  RSR_REQUIRE(flags != nullptr && A != nullptr, "rsr_classify_tc: null pointer");
  // Reference rows are tiled by 256 (pair kernel) -- callers pad B to a
  // multiple of 256 rows with never-hit rows (rsr_encode_refs rows_total).
  const int impl = getenv("RSR_TC_IMPL") ? atoi(getenv("RSR_TC_IMPL")) : 2;
  const int tile_n = impl == 1 ? kTileN : kPairN;
  const int64_t nt_l = rsr::ceil_div(n_lower, tile_n), nt_u = rsr::ceil_div(n_upper, tile_n);
  if (nt_l + nt_u == 0) {
    if (!accumulate) {
      clear_flags_kernel<<<(unsigned)rsr::ceil_div(S, 256), 256, 0, st>>>(flags, S);
      int rc0 = rsr::check_launch("clear_flags_kernel");
      if (rc0) return rc0;
      for (int64_t* f : {first_lower, first_upper})
        if (f) RSR_CUDA(cudaMemsetAsync(f, 0xFF, S * sizeof(int64_t), st));  // -1
    }
    return RSR_OK;
  }
  RSR_REQUIRE(nt_l + nt_u < (1 << 30), "rsr_classify_tc: too many reference tiles");
  RSR_REQUIRE((nt_l == 0 || B_lower) && (nt_u == 0 || B_upper), "rsr_classify_tc: null refs");

  int dev = 0, sm_count = 0;
  RSR_CUDA(cudaGetDevice(&dev));
  RSR_CUDA(cudaDeviceGetAttribute(&sm_count, cudaDevAttrMultiProcessorCount, dev));

  CUtensorMap ma, ml, mu;
  int rc = make_map(&ma, A, S, Kpad);
  if (rc) return rc;
  const int8_t* bl = nt_l ? B_lower : B_upper;
  const int8_t* bu = nt_u ? B_upper : B_lower;
  rc = make_map(&ml, bl, (nt_l ? nt_l : nt_u) * tile_n, Kpad);
  if (rc) return rc;
  rc = make_map(&mu, bu, (nt_u ? nt_u : nt_l) * tile_n, Kpad);
  if (rc) return rc;

  TcParams p;
  p.S = S;
  p.kb = (int)rsr::ceil_div(Kpad, kKBlock);
  p.ksteps_last = (Kpad - (p.kb - 1) * kKBlock) / kKStep;
  p.nt_lower = (int)nt_l;
  p.nt_total = (int)(nt_l + nt_u);
  p.flags = flags;
  p.accumulate = accumulate;
  p.first_lower = first_lower;
  p.first_upper = first_upper;
  p.first_base_lower = p.first_base_upper = 0;
#ifdef RSR_TC_EXPERIMENTS
  // timing experiments only (results are wrong when set): compiled out of the
  // product library
  const char* dbg = getenv("RSR_TC_DEBUG");
  p.debug = dbg ? atoi(dbg) : 0;
#else
  p.debug = 0;
#endif
  const size_t max_smem = 227 * 1024;

  if (impl != 1) {
    // align slack + barriers + hit exchange (+ first-match exchange, 2 x 128 int64)
    const size_t fixed = 1024 + 1024 + (want_first ? 2048 : 0);
    // double-buffer the sample tile when at least 4 B stages still fit
    const char* ab_env = getenv("RSR_TC_ABUFS");
    p.a_bufs = 2;
    if ((ab_env && atoi(ab_env) == 1) ||
        (size_t)2 * p.kb * kTileBytes + 4 * kTileBytes + fixed > max_smem)
      p.a_bufs = 1;
    const size_t a_bytes = (size_t)p.a_bufs * p.kb * kTileBytes;
    int stages = (int)((max_smem - fixed - a_bytes) / kTileBytes);
    if (stages > 12) stages = 12;
    RSR_REQUIRE(stages >= 2, "rsr_classify_tc: Kpad too large for shared memory");
    p.stages = stages;
    const size_t smem = fixed + a_bytes + (size_t)stages * kTileBytes;
    p.n_groups = (int)rsr::ceil_div(S, (int64_t)2 * kTileM);
    auto kern = want_first ? classify_tc_pair_kernel<true> : classify_tc_pair_kernel<false>;
    RSR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int clusters = sm_count / 2;
    if (p.n_groups < clusters) clusters = p.n_groups;
    // Reference chunks: every group streams all tiles of a launch, so a launch's
    // B slice must stay L2-resident (126 MB L2); 256 tiles = 64K refs x Kpad
    // bytes (20 MB at Kpad = 320).  Flags accumulate across launches.
    const char* ct = getenv("RSR_TC_CHUNK_TILES");
    const int64_t chunk = ct ? atoll(ct) : 256;
    const int64_t total = nt_l + nt_u;
    for (int64_t c0 = 0; c0 < total; c0 += chunk) {
      const int64_t c1 = c0 + chunk < total ? c0 + chunk : total;
      const int64_t l0 = c0 < nt_l ? c0 : nt_l, l1 = c1 < nt_l ? c1 : nt_l;
      const int64_t u0 = (c0 > nt_l ? c0 : nt_l) - nt_l, u1 = (c1 > nt_l ? c1 : nt_l) - nt_l;
      TcParams q = p;
      q.nt_lower = (int)(l1 - l0);
      q.nt_total = (int)((l1 - l0) + (u1 - u0));
      q.accumulate = c0 == 0 ? accumulate : 1;
      q.first_base_lower = l0 * kPairN;
      q.first_base_upper = u0 * kPairN;
      CUtensorMap cl = ml, cu = mu;
      if (total > chunk) {
        const int8_t* lb = l1 > l0 ? B_lower + l0 * kPairN * (int64_t)Kpad : nullptr;
        const int8_t* ub = u1 > u0 ? B_upper + u0 * kPairN * (int64_t)Kpad : nullptr;
        rc = make_map(&cl, lb ? lb : ub, ((lb ? l1 - l0 : u1 - u0)) * kPairN, Kpad);
        if (rc) return rc;
        rc = make_map(&cu, ub ? ub : lb, ((ub ? u1 - u0 : l1 - l0)) * kPairN, Kpad);
        if (rc) return rc;
      }
      kern<<<2 * clusters, 384, smem, st>>>(ma, cl, cu, q);
      rc = rsr::check_launch("classify_tc_pair_kernel");
      if (rc) return rc;
    }
    return RSR_OK;
  }

  RSR_REQUIRE(!want_first, "rsr_classify_tc: first-match needs the CTA-pair kernel");
  const size_t fixed = 1024 /*align slack*/ + 256 /*barriers*/;
  const int mt = ((size_t)2 * p.kb * kTileBytes + 4 * kTileBytes + fixed <= max_smem) ? 2 : 1;
  const size_t a_bytes = (size_t)mt * p.kb * kTileBytes;
  int stages = (int)((max_smem - fixed - a_bytes) / kTileBytes);
  if (stages > 8) stages = 8;
  RSR_REQUIRE(stages >= 2, "rsr_classify_tc: Kpad too large for shared memory");
  p.stages = stages;
  const size_t smem = fixed + a_bytes + (size_t)stages * kTileBytes;
  p.n_groups = (int)rsr::ceil_div(S, (int64_t)mt * kTileM);
  if (mt == 2) return launch_tc<2>(ma, ml, mu, p, smem, sm_count, st);
  return launch_tc<1>(ma, ml, mu, p, smem, sm_count, st);
}

}  // namespace

extern "C" int rsr_classify_tc(const int8_t* A, int64_t S, const int8_t* B_lower, int64_t n_lower,
                               const int8_t* B_upper, int64_t n_upper, int Kpad, uint8_t* flags,
                               int accumulate, void* stream) {
  return classify_tc_impl(A, S, B_lower, n_lower, B_upper, n_upper, Kpad, flags, accumulate,
                          nullptr, nullptr, stream);
}

extern "C" int rsr_classify_tc_explain(const int8_t* A, int64_t S, const int8_t* B_lower,
                                       int64_t n_lower, const int8_t* B_upper, int64_t n_upper,
                                       int Kpad, uint8_t* flags, int64_t* first_lower,
                                       int64_t* first_upper, int accumulate, void* stream) {
  return classify_tc_impl(A, S, B_lower, n_lower, B_upper, n_upper, Kpad, flags, accumulate,
                          first_lower, first_upper, stream);
}
