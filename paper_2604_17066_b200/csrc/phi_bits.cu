// (3)+(4) Bitset-BFS Phi for simple graphs with <= 256 nodes.
//
// Same results as csrc/phi.cu (and the reference union-find, sysfn.py:62-98):
// the connected component of s in the alive subgraph {e : x_e >= level}.
// Per warp, shared memory holds the alive adjacency of every level as node
// bitsets adj[level][v][W] (W = ceil(n/32) words); node v = 32*q + lane sits at
// bit `lane` of word q, so a BFS level is: each lane ORs the adjacency words of
// its frontier nodes, `redux.sync.or` combines them across the warp (the
// frontier stays warp-uniform in registers), new = acc & ~visited.  A
// boundary-search step changes one component by +-1, i.e. flips at most one
// edge in one level: the adjacency is updated with two XORs instead of being
// rebuilt.  (XOR toggling needs a simple graph: the host sets
// RSR_PHI_FLAG_SIMPLE only when no two edges share their endpoints.)
#include "common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct BitGraph {
  int kind, N, n, s, t, levels;
  const int32_t* eu;
  const int32_t* ev;
};

__host__ __device__ inline int levels_of(const rsr_phi_desc& d) {
  return d.kind == RSR_PHI_WIDEST_PATH ? d.n_states - 1 : 1;
}

__host__ __device__ inline size_t x_bytes(int N) { return ((size_t)N + 15) / 16 * 16; }

template <int W>
__host__ __device__ inline size_t warp_bytes(const rsr_phi_desc& d) {
  return x_bytes(d.n_components) + (size_t)levels_of(d) * d.n_nodes * W * 4;
}

// Alive adjacency of every level from the component states x.
template <int W>
__device__ void adj_build(const BitGraph& g, const volatile uint8_t* x, uint32_t* adj, int lane) {
  const int words = g.levels * g.n * W;
  for (int i = lane; i < words; i += 32) adj[i] = 0;
  __syncwarp();
  for (int e = lane; e < g.N; e += 32) {
    const int xe = x[e], u = g.eu[e], v = g.ev[e];
    for (int L = 1; L <= g.levels && xe >= L; ++L) {
      uint32_t* a = adj + (size_t)(L - 1) * g.n * W;
      atomicOr(&a[u * W + (v >> 5)], 1u << (v & 31));
      atomicOr(&a[v * W + (u >> 5)], 1u << (u & 31));
    }
  }
  __syncwarp();
}

// Edge e moves from state xo to xn: flip its adjacency bits in the levels whose
// aliveness changes (at most one level for a unit step).
template <int W>
__device__ void adj_toggle(const BitGraph& g, uint32_t* adj, int e, int xo, int xn, int lane) {
  if (lane == 0) {
    const int u = g.eu[e], v = g.ev[e];
    for (int L = 1; L <= g.levels; ++L) {
      if ((xo >= L) != (xn >= L)) {
        uint32_t* a = adj + (size_t)(L - 1) * g.n * W;
        a[u * W + (v >> 5)] ^= 1u << (v & 31);
        a[v * W + (u >> 5)] ^= 1u << (u & 31);
      }
    }
  }
  __syncwarp();
}

// BFS from s over one level's adjacency.  t >= 0: is t reached (early exit);
// t < 0: are all n nodes reached.
template <int W>
__device__ bool bfs(const uint32_t* adj, int n, int s, int t, int lane) {
  uint32_t F[W], V[W];
#pragma unroll
  for (int w = 0; w < W; ++w) F[w] = V[w] = (w == (s >> 5)) ? (1u << (s & 31)) : 0u;
  while (true) {
    uint32_t acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = 32 * q + lane;
      if (v < n && ((F[q] >> lane) & 1u)) {
        const uint32_t* a = adj + v * W;
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] |= a[w];
      }
    }
    uint32_t any = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t nw = __reduce_or_sync(kFull, acc[w]) & ~V[w];
      V[w] |= nw;
      F[w] = nw;
      any |= nw;
    }
    if (t >= 0) {
      bool hit = false;
#pragma unroll
      for (int w = 0; w < W; ++w)
        if (w == (t >> 5)) hit = (V[w] >> (t & 31)) & 1u;
      if (hit) return true;
    }
    if (!any) break;
  }
  if (t >= 0) return false;
  bool all = true;
#pragma unroll
  for (int w = 0; w < W; ++w) {
    const int lo = 32 * w;
    const uint32_t want = n >= lo + 32 ? kFull : (n > lo ? ((1u << (n - lo)) - 1u) : 0u);
    all &= (V[w] & want) == want;
  }
  return all;
}

template <int W>
__device__ int phi_bits(const BitGraph& g, const uint32_t* adj, int lane) {
  switch (g.kind) {
    case RSR_PHI_ST_CONNECTIVITY:
      return bfs<W>(adj, g.n, g.s, g.t, lane) ? 1 : 0;
    case RSR_PHI_WIDEST_PATH:
      for (int L = g.levels; L >= 1; --L)
        if (bfs<W>(adj + (size_t)(L - 1) * g.n * W, g.n, g.s, g.t, lane)) return L;
      return 0;
    default:  // RSR_PHI_GLOBAL_CONNECTIVITY
      return bfs<W>(adj, g.n, 0, -1, lane) ? 1 : 0;
  }
}

__device__ BitGraph load_graph(const rsr_phi_desc& d, uint8_t* smem, uint8_t** tail) {
  BitGraph g;
  g.kind = d.kind;
  g.N = d.n_components;
  g.n = d.n_nodes;
  g.s = d.source;
  g.t = d.target;
  g.levels = levels_of(d);
  int32_t* eu = reinterpret_cast<int32_t*>(smem);
  int32_t* ev = eu + g.N;
  for (int i = threadIdx.x; i < g.N; i += blockDim.x) {
    eu[i] = d.edge_u[i];
    ev[i] = d.edge_v[i];
  }
  g.eu = eu;
  g.ev = ev;
  *tail = reinterpret_cast<uint8_t*>(ev + g.N);
  __syncthreads();
  return g;
}

template <int W>
__global__ void phi_eval_bits_kernel(const rsr_phi_desc d, const uint8_t* __restrict__ states,
                                     const int64_t* __restrict__ idx, int64_t count,
                                     uint8_t* __restrict__ out, int threshold,
                                     unsigned long long* count_leq) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* tail;
  const BitGraph g = load_graph(d, smem, &tail);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  uint8_t* mine = tail + warp * warp_bytes<W>(d);
  volatile uint8_t* x = mine;
  uint32_t* adj = reinterpret_cast<uint32_t*>(mine + x_bytes(g.N));
  unsigned long long leq = 0;
  for (int64_t i = (int64_t)blockIdx.x * warps + warp; i < count; i += (int64_t)gridDim.x * warps) {
    const int64_t row = idx ? idx[i] : i;
    const uint8_t* src = states + row * g.N;
    for (int e = lane; e < g.N; e += 32) x[e] = src[e];
    __syncwarp();
    adj_build<W>(g, x, adj, lane);
    const int v = phi_bits<W>(g, adj, lane);
    if (lane == 0 && out) out[i] = (uint8_t)v;
    leq += (v <= threshold);
    __syncwarp();
  }
  if (count_leq && lane == 0 && leq) atomicAdd(count_leq, leq);
}

template <int W>
__global__ void boundary_bits_kernel(const rsr_phi_desc d, int threshold,
                                     const uint8_t* __restrict__ x0, int64_t B,
                                     uint8_t* __restrict__ out_refs, uint8_t* __restrict__ out_side,
                                     int64_t* __restrict__ out_calls) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* tail;
  const BitGraph g = load_graph(d, smem, &tail);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  uint8_t* mine = tail + warp * warp_bytes<W>(d);
  volatile uint8_t* x = mine;
  uint32_t* adj = reinterpret_cast<uint32_t*>(mine + x_bytes(g.N));
  const int M = d.n_states;
  for (int64_t b = (int64_t)blockIdx.x * warps + warp; b < B; b += (int64_t)gridDim.x * warps) {
    const uint8_t* src = x0 + b * g.N;
    for (int e = lane; e < g.N; e += 32) x[e] = src[e];
    __syncwarp();
    adj_build<W>(g, x, adj, lane);
    int64_t calls = 1;
    const bool lower = phi_bits<W>(g, adj, lane) <= threshold;
    const int step = lower ? 1 : -1, limit = lower ? M - 1 : 0;
    for (int n = 0; n < g.N; ++n) {
      while (true) {
        const int xo = x[n];
        if (xo == limit) break;
        const int xn = xo + step;
        __syncwarp();
        if (lane == 0) x[n] = (uint8_t)xn;
        adj_toggle<W>(g, adj, n, xo, xn, lane);
        const int s = phi_bits<W>(g, adj, lane);
        ++calls;
        const bool crossed = lower ? (s > threshold) : (s <= threshold);
        if (crossed) {
          if (lane == 0) x[n] = (uint8_t)xo;
          adj_toggle<W>(g, adj, n, xn, xo, lane);
          break;
        }
      }
    }
    __syncwarp();
    uint8_t* dst = out_refs + b * g.N;
    for (int e = lane; e < g.N; e += 32) dst[e] = x[e];
    if (lane == 0) {
      out_side[b] = lower ? RSR_SIDE_LOWER : RSR_SIDE_UPPER;
      out_calls[b] = calls;
    }
    __syncwarp();
  }
}

template <int W>
int launch(const rsr_phi_desc& d, bool boundary, int threshold, const uint8_t* states,
           const int64_t* idx, int64_t count, uint8_t* out, int64_t* count_leq, uint8_t* out_side,
           int64_t* out_calls, cudaStream_t st) {
  const size_t fixed = 2 * sizeof(int32_t) * (size_t)d.n_components;
  const size_t per_warp = warp_bytes<W>(d);
  const size_t budget = 160 * 1024;
  int warps = (int)((budget - fixed) / per_warp);
  if (warps > 8) warps = 8;
  if (warps < 1) return -1;
  int64_t grid = (count + warps - 1) / warps;
  if (grid > 148 * 16) grid = 148 * 16;
  if (grid < 1) grid = 1;
  const size_t smem = fixed + warps * per_warp;
  if (boundary) {
    auto k = boundary_bits_kernel<W>;
    if (smem > 48 * 1024)
      RSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k<<<(unsigned)grid, warps * 32, smem, st>>>(d, threshold, states, count, out, out_side,
                                                out_calls);
    return rsr::check_launch("boundary_bits_kernel");
  }
  auto k = phi_eval_bits_kernel<W>;
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)grid, warps * 32, smem, st>>>(d, states, idx, count, out, threshold,
                                              reinterpret_cast<unsigned long long*>(count_leq));
  return rsr::check_launch("phi_eval_bits_kernel");
}

}  // namespace

namespace rsr {

// Returns -1 when the bitset path does not apply (caller falls back).
int phi_bits_dispatch(const rsr_phi_desc& d, bool boundary, int threshold, const uint8_t* states,
                      const int64_t* idx, int64_t count, uint8_t* out, int64_t* count_leq,
                      uint8_t* out_side, int64_t* out_calls, cudaStream_t st) {
  if (!(d.flags & RSR_PHI_FLAG_SIMPLE)) return -1;
  if (d.kind != RSR_PHI_ST_CONNECTIVITY && d.kind != RSR_PHI_WIDEST_PATH &&
      d.kind != RSR_PHI_GLOBAL_CONNECTIVITY)
    return -1;
  if (d.n_nodes < 1 || d.n_nodes > 256) return -1;
  const int W = (d.n_nodes + 31) / 32;
  const int w = W <= 1 ? 1 : W <= 2 ? 2 : W <= 4 ? 4 : 8;
  switch (w) {
    case 1: return launch<1>(d, boundary, threshold, states, idx, count, out, count_leq, out_side, out_calls, st);
    case 2: return launch<2>(d, boundary, threshold, states, idx, count, out, count_leq, out_side, out_calls, st);
    case 4: return launch<4>(d, boundary, threshold, states, idx, count, out, count_leq, out_side, out_calls, st);
    default: return launch<8>(d, boundary, threshold, states, idx, count, out, count_leq, out_side, out_calls, st);
  }
}

}  // namespace rsr
