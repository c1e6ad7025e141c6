// (4) Boundary search for graph-connectivity Phi without re-evaluating Phi.
//
// Same walk, same result and same Phi-call count as the reference
// boundary_search (boundary.py:116-147) for s-t connectivity (sysfn.py:87-98)
// and the widest-path level (builder-defined), but each step is
// decided by a graph operation instead of a full Phi evaluation.
//
// With L = m' + 1 and G_L(x) = {e : x_e >= L}:  Phi(x) > m'  <=>  s and t are
// connected in G_L(x)  (s-t connectivity: Phi = [connected in G_1], m' = 0;
// widest path: G_k shrink with k).  A unit step of component n changes G_L
// only when x_n crosses L, so per component:
//   lower side (start disconnected, step up to M-1): the step L-1 -> L adds
//     edge n to G_L; it crosses iff it joins the components of s and t --
//     a union-find query, O(alpha) instead of a BFS;
//   upper side (start connected, step down to 0): the step L -> L-1 removes
//     edge n from G_L; it crosses iff no s-t path survives.  A witness s-t path
//     P is kept: removing an edge off P cannot disconnect (P survives), so only
//     edges on P need a BFS (bitset BFS, one warp), which also yields the next
//     witness path.
// All other steps leave G_L unchanged and cannot cross; they are counted as the
// Phi calls the reference makes for them.  One warp per start vector; lane 0
// runs the union-find, the warp runs the BFS.  Simple graphs (no parallel
// edges: RSR_PHI_FLAG_SIMPLE) with <= 256 nodes; other cases use csrc/phi_bits.cu
// or csrc/phi.cu.
#include "common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;

struct GraphSmem {
  int N, n, s, t;
  const int32_t* eu;
  const int32_t* ev;
  const int16_t* eid;  // n x n edge ids (-1: none) when n <= kEidMaxNodes, else nullptr
};

constexpr int kEidMaxNodes = 128;

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) / 16 * 16; }

// per-warp scratch: x (N bytes), union-find parents (n int16), on-path bits
// (ceil(N/32) words), adjacency of G_L (n x W words), BFS levels (n x W words)
template <int W>
__host__ __device__ inline size_t warp_scratch(int N, int n) {
  return align16(N) + align16(2 * (size_t)n) + align16(4 * (((size_t)N + 31) / 32)) +
         2 * (size_t)n * W * 4;
}

__device__ __forceinline__ int uf_find(int16_t* par, int a) {
  while (par[a] != a) {
    par[a] = par[par[a]];  // path halving
    a = par[a];
  }
  return a;
}

// BFS from s in adj recording each level's new nodes; on success levels[0..d]
// hold the layers and the return value is d (>= 1), else 0 (t unreachable).
template <int W>
__device__ int bfs_layers(const uint32_t* adj, uint32_t* levels, int n, int s, int t, int lane) {
  uint32_t F[W], V[W];
#pragma unroll
  for (int w = 0; w < W; ++w) F[w] = V[w] = (w == (s >> 5)) ? (1u << (s & 31)) : 0u;
#pragma unroll
  for (int w = 0; w < W; ++w)
    if (lane == w) levels[w] = F[w];
  for (int d = 1; d < n; ++d) {
    uint32_t acc[W];
#pragma unroll
    for (int w = 0; w < W; ++w) acc[w] = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = 32 * q + lane;
      if (v < n && ((F[q] >> lane) & 1u)) {
#pragma unroll
        for (int w = 0; w < W; ++w) acc[w] |= adj[v * W + w];
      }
    }
    uint32_t any = 0;
    bool hit = false;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t nw = __reduce_or_sync(kFull, acc[w]) & ~V[w];
      V[w] |= nw;
      F[w] = nw;
      any |= nw;
      if (w == (t >> 5)) hit = (nw >> (t & 31)) & 1u;
    }
    if (lane < W) {
#pragma unroll
      for (int w = 0; w < W; ++w)
        if (w == lane) levels[d * W + w] = F[w];
    }
    if (hit) {
      __syncwarp();
      return d;
    }
    if (!any) break;
  }
  __syncwarp();
  return 0;
}

// Mark the edges of one shortest s-t path (from bfs_layers) in `onpath`.
template <int W>
__device__ void trace_path(const GraphSmem& g, const uint32_t* adj, const uint32_t* levels,
                           int d, uint32_t* onpath, int lane) {
  const int words = (g.N + 31) / 32;
  for (int i = lane; i < words; i += 32) onpath[i] = 0;
  __syncwarp();
  int cur = g.t;
  for (int k = d; k >= 1; --k) {
    // parent: lowest node of layer k-1 adjacent to cur
    int p = -1;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = adj[cur * W + w] & levels[(k - 1) * W + w];
      if (p < 0 && c) p = 32 * w + __ffs(c) - 1;
    }
    // the (unique, simple graph) edge joining p and cur
    int e_found = g.eid ? g.eid[p * g.n + cur] : -1;
    for (int e0 = 0; e_found < 0 && e0 < g.N; e0 += 32) {
      const int e = e0 + lane;
      const bool m = e < g.N && ((g.eu[e] == p && g.ev[e] == cur) || (g.eu[e] == cur && g.ev[e] == p));
      const unsigned b = __ballot_sync(kFull, m);
      if (b) {
        e_found = e0 + __ffs(b) - 1;
        break;
      }
    }
    if (lane == 0) onpath[e_found >> 5] |= 1u << (e_found & 31);
    cur = p;
  }
  __syncwarp();
}

__device__ __forceinline__ void toggle_edge(uint32_t* adj, int W, int u, int v, int lane) {
  if (lane == 0) {
    adj[u * W + (v >> 5)] ^= 1u << (v & 31);
    adj[v * W + (u >> 5)] ^= 1u << (u & 31);
  }
  __syncwarp();
}

template <int W>
__global__ void boundary_graph_kernel(const rsr_phi_desc d, int L, const uint8_t* __restrict__ x0,
                                      int64_t B, uint8_t* __restrict__ out_refs,
                                      uint8_t* __restrict__ out_side,
                                      int64_t* __restrict__ out_calls) {
  extern __shared__ __align__(16) uint8_t smem[];
  GraphSmem g;
  g.N = d.n_components;
  g.n = d.n_nodes;
  g.s = d.source;
  g.t = d.target;
  int32_t* eu = reinterpret_cast<int32_t*>(smem);
  int32_t* ev = eu + g.N;
  for (int i = threadIdx.x; i < g.N; i += blockDim.x) {
    eu[i] = d.edge_u[i];
    ev[i] = d.edge_v[i];
  }
  g.eu = eu;
  g.ev = ev;
  uint8_t* after = reinterpret_cast<uint8_t*>(ev + g.N);
  g.eid = nullptr;
  if (g.n <= kEidMaxNodes) {
    int16_t* eid = reinterpret_cast<int16_t*>(after);
    for (int i = threadIdx.x; i < g.n * g.n; i += blockDim.x) eid[i] = -1;
    __syncthreads();
    for (int e = threadIdx.x; e < g.N; e += blockDim.x) {
      eid[eu[e] * g.n + ev[e]] = (int16_t)e;
      eid[ev[e] * g.n + eu[e]] = (int16_t)e;
    }
    g.eid = eid;
    after += align16(2 * (size_t)g.n * g.n);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  uint8_t* mine = after + (size_t)warp * (warp_scratch<W>(g.N, g.n) + 16);
  mine = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(mine) + 15) & ~uintptr_t(15));
  uint8_t* x = mine;
  int16_t* par = reinterpret_cast<int16_t*>(mine + align16(g.N));
  uint32_t* onpath = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(par) + align16(2 * g.n));
  uint32_t* adj = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(onpath) +
                                              align16(4 * ((g.N + 31) / 32)));
  uint32_t* levels = adj + g.n * W;
  const int M = d.n_states;

  for (int64_t b = (int64_t)blockIdx.x * warps + warp; b < B; b += (int64_t)gridDim.x * warps) {
    const uint8_t* src = x0 + b * g.N;
    for (int e = lane; e < g.N; e += 32) x[e] = src[e];
    for (int v = lane; v < g.n; v += 32) par[v] = (int16_t)v;
    __syncwarp();
    // initial Phi(x0): connectivity of G_L by union-find (lane 0)
    int connected = 0;
    if (lane == 0) {
      for (int e = 0; e < g.N; ++e) {
        if (x[e] >= L) {
          const int a = uf_find(par, eu[e]), c = uf_find(par, ev[e]);
          if (a != c) par[a] = (int16_t)c;
        }
      }
      connected = uf_find(par, g.s) == uf_find(par, g.t);
    }
    connected = __shfl_sync(kFull, connected, 0);
    int64_t calls = 1;
    if (!connected) {
      // ---------------- lower side: union-find, no Phi evaluation needed
      if (lane == 0) {
        for (int n = 0; n < g.N; ++n) {
          const int xn = x[n];
          if (xn >= M - 1) continue;
          if (xn >= L) {  // already in G_L: every step up leaves G_L unchanged
            calls += M - 1 - xn;
            x[n] = (uint8_t)(M - 1);
            continue;
          }
          calls += L - xn;  // steps up to L, the last one adds edge n to G_L
          const int a = uf_find(par, eu[n]), c = uf_find(par, ev[n]);
          const int rs = uf_find(par, g.s), rt = uf_find(par, g.t);
          if ((a == rs && c == rt) || (a == rt && c == rs)) {
            x[n] = (uint8_t)(L - 1);  // crossing: reverted, walk moves to n + 1
            continue;
          }
          if (a != c) par[a] = (int16_t)c;
          calls += M - 1 - L;
          x[n] = (uint8_t)(M - 1);
        }
      }
    } else {
      // ---------------- upper side: witness path + BFS for edges on it
      for (int i = lane; i < g.n * W; i += 32) adj[i] = 0;
      __syncwarp();
      for (int e = lane; e < g.N; e += 32) {
        if (x[e] >= L) {
          const int u = eu[e], v = ev[e];
          atomicOr(&adj[u * W + (v >> 5)], 1u << (v & 31));
          atomicOr(&adj[v * W + (u >> 5)], 1u << (u & 31));
        }
      }
      __syncwarp();
      int dd = bfs_layers<W>(adj, levels, g.n, g.s, g.t, lane);
      trace_path<W>(g, adj, levels, dd, onpath, lane);
      for (int n = 0; n < g.N; ++n) {
        const int xn = x[n];
        if (xn == 0) continue;
        if (xn < L) {  // not in G_L: every step down leaves G_L unchanged
          calls += xn;
          if (lane == 0) x[n] = 0;
          continue;
        }
        calls += xn - L + 1;  // steps down to L-1, the last one removes edge n
        const bool on = (onpath[n >> 5] >> (n & 31)) & 1u;
        if (on) {
          const int u = eu[n], v = ev[n];
          toggle_edge(adj, W, u, v, lane);
          // cheap witness repair first: a common neighbour w of u and v turns
          // the path into a walk through (u,w),(w,v) that still contains an s-t
          // path (the witness may be a superset of a path: a later test of one
          // of its edges then just runs the exact BFS below)
          int wn = -1;
#pragma unroll
          for (int q = 0; q < W; ++q) {
            const uint32_t c = adj[u * W + q] & adj[v * W + q];
            if (wn < 0 && c) wn = 32 * q + __ffs(c) - 1;
          }
          if (wn >= 0 && g.eid) {
            if (lane == 0) {
              const int e1 = g.eid[u * g.n + wn], e2 = g.eid[wn * g.n + v];
              onpath[n >> 5] &= ~(1u << (n & 31));
              onpath[e1 >> 5] |= 1u << (e1 & 31);
              onpath[e2 >> 5] |= 1u << (e2 & 31);
            }
            calls += L - 1;
            if (lane == 0) x[n] = 0;
            __syncwarp();
            continue;
          }
          dd = bfs_layers<W>(adj, levels, g.n, g.s, g.t, lane);
          if (dd == 0) {  // crossing: reverted, walk moves to n + 1
            toggle_edge(adj, W, eu[n], ev[n], lane);
            if (lane == 0) x[n] = (uint8_t)L;
            __syncwarp();
            continue;
          }
          trace_path<W>(g, adj, levels, dd, onpath, lane);
        } else {
          toggle_edge(adj, W, eu[n], ev[n], lane);
        }
        calls += L - 1;
        if (lane == 0) x[n] = 0;
        __syncwarp();
      }
    }
    __syncwarp();
    uint8_t* dst = out_refs + b * g.N;
    for (int e = lane; e < g.N; e += 32) dst[e] = x[e];
    if (lane == 0) {
      out_side[b] = connected ? RSR_SIDE_UPPER : RSR_SIDE_LOWER;
      out_calls[b] = calls;
    }
    __syncwarp();
  }
}

template <int W>
int launch_graph(const rsr_phi_desc& d, int L, const uint8_t* x0, int64_t B, uint8_t* out_refs,
                 uint8_t* out_side, int64_t* out_calls, cudaStream_t st) {
  const size_t fixed = 2 * sizeof(int32_t) * (size_t)d.n_components + 16 +
                       (d.n_nodes <= kEidMaxNodes ? align16(2 * (size_t)d.n_nodes * d.n_nodes) : 0);
  const size_t per_warp = warp_scratch<W>(d.n_components, d.n_nodes) + 16;
  int warps = (int)((160 * 1024 - fixed) / per_warp);
  if (warps > 4) warps = 4;
  if (warps < 1) return -1;
  int64_t grid = (B + warps - 1) / warps;
  if (grid > 148 * 32) grid = 148 * 32;
  const size_t smem = fixed + warps * per_warp;
  auto k = boundary_graph_kernel<W>;
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<(unsigned)grid, warps * 32, smem, st>>>(d, L, x0, B, out_refs, out_side, out_calls);
  return rsr::check_launch("boundary_graph_kernel");
}

}  // namespace

namespace rsr {

// Returns -1 when the graph-operation search does not apply (caller falls back).
int boundary_graph_dispatch(const rsr_phi_desc& d, int threshold, const uint8_t* x0, int64_t B,
                            uint8_t* out_refs, uint8_t* out_side, int64_t* out_calls,
                            cudaStream_t st) {
  if (!(d.flags & RSR_PHI_FLAG_SIMPLE)) return -1;
  int L;
  if (d.kind == RSR_PHI_ST_CONNECTIVITY) {
    if (threshold != 0) return -1;
    L = 1;
  } else if (d.kind == RSR_PHI_WIDEST_PATH) {
    if (threshold < 0 || threshold > d.n_states - 2) return -1;
    L = threshold + 1;
  } else {
    return -1;
  }
  if (d.n_nodes < 2 || d.n_nodes > 256 || d.source == d.target) return -1;
  const int W = (d.n_nodes + 31) / 32;
  const int w = W <= 1 ? 1 : W <= 2 ? 2 : W <= 4 ? 4 : 8;
  switch (w) {
    case 1: return launch_graph<1>(d, L, x0, B, out_refs, out_side, out_calls, st);
    case 2: return launch_graph<2>(d, L, x0, B, out_refs, out_side, out_calls, st);
    case 4: return launch_graph<4>(d, L, x0, B, out_refs, out_side, out_calls, st);
    default: return launch_graph<8>(d, L, x0, B, out_refs, out_side, out_calls, st);
  }
}

}  // namespace rsr
