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
#include <stdlib.h>

#include "common.cuh"

namespace {

constexpr unsigned kFull = 0xffffffffu;

// experiment knob: a three-edge detour repair before the BFS (measured a wash on
// the config 3/5 loops: -2 % / +5 %), off
#ifndef RSR_BOUNDARY_HOP3
#define RSR_BOUNDARY_HOP3 0
#endif

// experiment builds (make prof): 0 searches, 1 upper-side searches, 2 BFS runs,
// 3 BFS steps, 4 cycles in BFS, 5 cycles in trace_bidir, 6 cycles in the initial
// union-find, 7 total cycles
#ifdef RSR_FP4_PROF
__device__ unsigned long long g_bprof[8];
#define BPROF_ADD(i, v) \
  if ((threadIdx.x & 31) == 0) atomicAdd(&g_bprof[i], (unsigned long long)(v))
#define BPROF_T(x) const long long x = clock64()
#else
#define BPROF_ADD(i, v)
#define BPROF_T(x)
#endif

struct GraphSmem {
  int N, n, s, t;
  const int32_t* eu;
  const int32_t* ev;
  const int16_t* eid;  // n x n edge ids (-1: none) when n <= kEidMaxNodes, else nullptr
};

constexpr int kEidMaxNodes = 128;

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) / 16 * 16; }

// per-warp scratch: x (N bytes), union-find parents (n int32), on-path bits
// (ceil(N/32) words), adjacency of G_L (n x W words), BFS levels from s and
// from t (n x W words each)
template <int W>
__host__ __device__ inline size_t warp_scratch(int N, int n) {
  return align16(N) + align16(4 * (size_t)n) + align16(4 * (((size_t)N + 31) / 32)) +
         align16(3 * (size_t)n * W * 4);
}

__device__ __forceinline__ int uf_find(int32_t* par, int a) {
  while (par[a] != a) {
    par[a] = par[par[a]];  // path halving
    a = par[a];
  }
  return a;
}

// Adjacency of G_L as node bitsets (node v = word v/32, bit v%32), two
// storages behind one interface:
//   AdjSmem: rows in shared memory (any n <= 256);
//   AdjReg:  rows in registers, lane l owning the rows of nodes l, l+32, ...
//            (n <= 128: W*W = 16 registers).
// A BFS level is a pull step: lane l tests whether node 32q+l has a neighbour
// in the frontier (W*W ANDs) and one ballot per word assembles the next
// frontier -- no cross-lane OR reduction (redux.sync) on the critical path.
template <int W>
struct AdjSmem {
  static constexpr bool kRegisters = false;
  uint32_t* a;
  __device__ void load(const uint32_t*, int, int) {}  // shared memory is the master copy
  // next[q] bit l = node 32q+l has a neighbour in F (pull step, one ballot per word)
  __device__ void pull(const uint32_t (&F)[W], uint32_t (&next)[W], int n, int lane) const {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int v = 32 * q + lane;
      uint32_t hit = 0;
      if (v < n) {
#pragma unroll
        for (int w = 0; w < W; ++w) hit |= a[v * W + w] & F[w];
      }
      next[q] = __ballot_sync(kFull, hit != 0);
    }
  }
  __device__ uint32_t row(int node, int w) const { return a[node * W + w]; }
  __device__ void toggle(int u, int v, int lane) {
    if (lane == 0) {
      a[u * W + (v >> 5)] ^= 1u << (v & 31);
      a[v * W + (u >> 5)] ^= 1u << (u & 31);
    }
    __syncwarp();
  }
};

template <int W>
struct AdjReg {
  static constexpr bool kRegisters = true;
  uint32_t r[W][W];
  __device__ void load(const uint32_t* a, int n, int lane) {
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int w = 0; w < W; ++w) r[q][w] = (32 * q + lane < n) ? a[(32 * q + lane) * W + w] : 0u;
  }
  __device__ void pull(const uint32_t (&F)[W], uint32_t (&next)[W], int, int) const {
#pragma unroll
    for (int q = 0; q < W; ++q) {
      uint32_t hit = 0;
#pragma unroll
      for (int w = 0; w < W; ++w) hit |= r[q][w] & F[w];
      next[q] = __ballot_sync(kFull, hit != 0);
    }
  }
  // (selects are written as masks: a branch on q == node/32 lets the compiler
  // turn r into a dynamically indexed, i.e. local-memory, array)
  __device__ uint32_t row(int node, int w) const {  // node is warp-uniform
    uint32_t val = 0;
#pragma unroll
    for (int q = 0; q < W; ++q) val |= r[q][w] & (0u - (uint32_t)(q == (node >> 5)));
    return __shfl_sync(kFull, val, node & 31);
  }
  __device__ void toggle(int u, int v, int lane) {
    const uint32_t bu = (lane == (u & 31)) ? 1u << (v & 31) : 0u;
    const uint32_t bv = (lane == (v & 31)) ? 1u << (u & 31) : 0u;
#pragma unroll
    for (int q = 0; q < W; ++q)
#pragma unroll
      for (int w = 0; w < W; ++w)
        r[q][w] ^= (bu & (0u - (uint32_t)(q == (u >> 5) && w == (v >> 5)))) |
                   (bv & (0u - (uint32_t)(q == (v >> 5) && w == (u >> 5))));
  }
};

// Bidirectional BFS: the frontiers from s and from t grow in lockstep (two
// independent pull chains per step, so the latency of one step is about that
// of a one-sided level) until they touch -- about half the levels of the
// one-sided search -- or one side stops growing (t or s unreachable: for a
// bridge near either end this takes only as many steps as that side's
// component is deep).  Returns 1 and the meeting node with its levels on both
// sides, or 0 when s and t are disconnected.
struct Meet {
  int m, ks, kt;
};

template <int W>
__device__ __forceinline__ int level_of(const uint32_t* lev, const uint32_t (&F)[W], int k, int m) {
  uint32_t in_f = 0;  // mask select: no dynamically indexed register array
#pragma unroll
  for (int w = 0; w < W; ++w) in_f |= (F[w] >> (m & 31)) & (uint32_t)(w == (m >> 5));
  if (in_f & 1u) return k;
  for (int j = k - 1; j > 0; --j)
    if ((lev[j * W + (m >> 5)] >> (m & 31)) & 1u) return j;
  return 0;
}

template <int W, class Adj>
__device__ __forceinline__ int bfs_bidir(const Adj& adj, uint32_t* lev_s, uint32_t* lev_t, int n,
                                         int s, int t, int lane, Meet& mt) {
  uint32_t Fs[W], Vs[W], Ft[W], Vt[W];
#pragma unroll
  for (int w = 0; w < W; ++w) {
    Fs[w] = Vs[w] = (w == (s >> 5)) ? (1u << (s & 31)) : 0u;
    Ft[w] = Vt[w] = (w == (t >> 5)) ? (1u << (t & 31)) : 0u;
  }
  auto word_of = [&](const uint32_t (&X)[W]) {
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < W; ++w) r |= X[w] & (0u - (uint32_t)(lane == w));
    return r;
  };
  if (lane < W) {
    lev_s[lane] = word_of(Fs);
    lev_t[lane] = word_of(Ft);
  }
  for (int k = 1; k < n; ++k) {
    uint32_t ns[W], nt[W];
    adj.pull(Fs, ns, n, lane);
    adj.pull(Ft, nt, n, lane);
    uint32_t anys = 0, anyt = 0;
    int m = -1;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      ns[w] &= ~Vs[w];
      nt[w] &= ~Vt[w];
      Vs[w] |= ns[w];
      Vt[w] |= nt[w];
      Fs[w] = ns[w];
      Ft[w] = nt[w];
      anys |= ns[w];
      anyt |= nt[w];
      const uint32_t c = Vs[w] & Vt[w];
      if (m < 0 && c) m = 32 * w + __ffs(c) - 1;
    }
    if (lane < W) {
      lev_s[k * W + lane] = word_of(Fs);
      lev_t[k * W + lane] = word_of(Ft);
    }
    __syncwarp();
    if (m >= 0) {
      mt.m = m;
      mt.ks = level_of<W>(lev_s, Fs, k, m);
      mt.kt = level_of<W>(lev_t, Ft, k, m);
      BPROF_ADD(3, k);
      return 1;
    }
    if (!anys || !anyt) {
      BPROF_ADD(3, k);
      return 0;
    }
  }
  return 0;
}

// Mark the edges of a path from `start` down the recorded levels d..0.
template <int W, class Adj>
__device__ __forceinline__ void trace_down(const GraphSmem& g, const Adj& adj, const uint32_t* levels,
                                           int d, int start, uint32_t* onpath, int lane) {
  int cur = start;
  for (int k = d; k >= 1; --k) {
    int p = -1;  // lowest node of layer k-1 adjacent to cur
#pragma unroll
    for (int w = 0; w < W; ++w) {
      const uint32_t c = adj.row(cur, w) & levels[(k - 1) * W + w];
      if (p < 0 && c) p = 32 * w + __ffs(c) - 1;
    }
    int e_found = g.eid ? g.eid[p * g.n + cur] : -1;
    for (int e0 = 0; e_found < 0 && e0 < g.N; e0 += 32) {
      const int e = e0 + lane;
      const bool mm = e < g.N && ((g.eu[e] == p && g.ev[e] == cur) || (g.eu[e] == cur && g.ev[e] == p));
      const unsigned bal = __ballot_sync(kFull, mm);
      if (bal) e_found = e0 + __ffs(bal) - 1;
    }
    if (lane == 0) onpath[e_found >> 5] |= 1u << (e_found & 31);
    cur = p;
  }
}

// New witness: the s-m and m-t halves of the bidirectional search.
template <int W, class Adj>
__device__ __forceinline__ void trace_bidir(const GraphSmem& g, const Adj& adj, const uint32_t* lev_s,
                                            const uint32_t* lev_t, const Meet& mt, uint32_t* onpath,
                                            int lane) {
  const int words = (g.N + 31) / 32;
  for (int i = lane; i < words; i += 32) onpath[i] = 0;
  __syncwarp();
  trace_down<W>(g, adj, lev_s, mt.ks, mt.m, onpath, lane);
  trace_down<W>(g, adj, lev_t, mt.kt, mt.m, onpath, lane);
  __syncwarp();
}

// Upper side of the walk (start connected in G_L): witness path + BFS for edges
// on it.  x[] is updated by lane 0; returns the Phi-call count of the walk
// after the initial evaluation.
template <int W, class Adj>
__device__ __forceinline__ int64_t upper_walk(const GraphSmem& g, Adj& adj, uint32_t* adj_smem,
                                              uint8_t* x, uint32_t* levels, uint32_t* onpath, int L,
                                              int lane) {
  int64_t calls = 0;
  uint32_t* lev_t = levels + g.n * W;
  Meet mt;
  bfs_bidir<W>(adj, levels, lev_t, g.n, g.s, g.t, lane, mt);  // connected: the start is upper
  trace_bidir<W>(g, adj, levels, lev_t, mt, onpath, lane);
  BPROF_ADD(1, 1);
  const int words = (g.N + 31) / 32;
  int n = 0;
  while (n < g.N) {
    // next witness-path edge at or after n (path edges are in G_L)
    int nstar = g.N;
    for (int w = n >> 5; w < words; ++w) {
      uint32_t bits = onpath[w];
      if (w == (n >> 5)) bits &= ~0u << (n & 31);
      if (bits) {
        nstar = 32 * w + __ffs(bits) - 1;
        break;
      }
    }
    if (nstar > n) {
      // edges n .. nstar-1 are off the witness path: every step down is taken
      // (the path survives), so they all drop to 0 at once -- x_n Phi calls
      // each -- and leave G_L together (bulk update of the shared-memory
      // adjacency, then the register copy is reloaded)
      int c = 0;
      for (int e = n + lane; e < nstar; e += 32) {
        const int xe = x[e];
        if (xe) {
          c += xe;
          x[e] = 0;
          if (xe >= L) {
            const int u = g.eu[e], v = g.ev[e];
            atomicAnd(&adj_smem[u * W + (v >> 5)], ~(1u << (v & 31)));
            atomicAnd(&adj_smem[v * W + (u >> 5)], ~(1u << (u & 31)));
          }
        }
      }
      calls += __reduce_add_sync(kFull, (unsigned)c);
      __syncwarp();
      adj.load(adj_smem, g.n, lane);
      n = nstar;
      if (n >= g.N) break;
    }
    const int xn = x[n];
    calls += xn - L + 1;  // steps down to L-1, the last one removes edge n
    const int u = g.eu[n], v = g.ev[n];
    adj.toggle(u, v, lane);
    if (Adj::kRegisters && lane == 0) {  // keep the shared-memory master copy in step
      adj_smem[u * W + (v >> 5)] ^= 1u << (v & 31);
      adj_smem[v * W + (u >> 5)] ^= 1u << (u & 31);
    }
    __syncwarp();
    {
      // cheap witness repair first: a common neighbour w of u and v turns the
      // path into a walk through (u,w),(w,v) that still contains an s-t path
      // (the witness may be a superset of a path: a later test of one of its
      // edges then just runs the exact BFS below)
      int wn = -1;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const uint32_t c = adj.row(u, q) & adj.row(v, q);
        if (wn < 0 && c) wn = 32 * q + __ffs(c) - 1;
      }
      int wa = -1, wb = -1;
#if RSR_BOUNDARY_HOP3
      // next cheapest: a detour u-a-b-v (a neighbour a of u sharing a neighbour b
      // with v; edge (u,v) is already gone from the adjacency)
      if (wn < 0 && g.eid) {
        for (int q = 0; q < W && wa < 0; ++q) {
          uint32_t na = adj.row(u, q);
          while (na && wa < 0) {
            const int a = 32 * q + __ffs(na) - 1;
            na &= na - 1;
#pragma unroll
            for (int q2 = 0; q2 < W; ++q2) {
              const uint32_t c = adj.row(a, q2) & adj.row(v, q2);
              if (wa < 0 && c) {
                wa = a;
                wb = 32 * q2 + __ffs(c) - 1;
              }
            }
          }
        }
      }
#endif
      if (wn >= 0 && g.eid) {
        if (lane == 0) {
          const int e1 = g.eid[u * g.n + wn], e2 = g.eid[wn * g.n + v];
          onpath[n >> 5] &= ~(1u << (n & 31));
          onpath[e1 >> 5] |= 1u << (e1 & 31);
          onpath[e2 >> 5] |= 1u << (e2 & 31);
        }
        __syncwarp();
      } else if (wa >= 0) {
        if (lane == 0) {
          const int e1 = g.eid[u * g.n + wa], e2 = g.eid[wa * g.n + wb], e3 = g.eid[wb * g.n + v];
          onpath[n >> 5] &= ~(1u << (n & 31));
          onpath[e1 >> 5] |= 1u << (e1 & 31);
          onpath[e2 >> 5] |= 1u << (e2 & 31);
          onpath[e3 >> 5] |= 1u << (e3 & 31);
        }
        __syncwarp();
      } else {
        BPROF_T(b0);
        const int dd = bfs_bidir<W>(adj, levels, lev_t, g.n, g.s, g.t, lane, mt);
        BPROF_T(b1);
        BPROF_ADD(2, 1);
        BPROF_ADD(4, b1 - b0);
        if (dd == 0) {  // crossing: reverted, walk moves to n + 1
          adj.toggle(u, v, lane);
          if (lane == 0) {
            if (Adj::kRegisters) {
              adj_smem[u * W + (v >> 5)] ^= 1u << (v & 31);
              adj_smem[v * W + (u >> 5)] ^= 1u << (u & 31);
            }
            x[n] = (uint8_t)L;
          }
          __syncwarp();
          ++n;
          continue;
        }
        BPROF_T(c0);
        trace_bidir<W>(g, adj, levels, lev_t, mt, onpath, lane);
        BPROF_T(c1);
        BPROF_ADD(5, c1 - c0);
      }
    }
    calls += L - 1;
    if (lane == 0) x[n] = 0;
    __syncwarp();
    ++n;
  }
  __syncwarp();
  return calls;
}

// Upper side in closed form (default).  With edge weights = component index, the
// reference's walk deletes, in index order, every edge of G_L whose removal keeps s
// and t connected; the edges it keeps are exactly the s-t path of the MAXIMUM
// spanning forest of G_L (proof: an edge e off that path P is deleted because P
// survives without it; an edge e on P is the heaviest edge across its fundamental
// cut, so every other edge across the cut has a smaller index, was considered
// earlier and deleted while P was intact, and removing e then disconnects s and t).
// So: Kruskal by descending index on lane 0 until s and t meet (later unions cannot
// change their tree path), one bitset BFS over the tree edges for the path, and the
// result and Phi-call count follow per component: an edge of P stops at L after
// x_n - L + 1 calls, every other component drops to 0 after x_n calls.  One BFS
// instead of one per witness-path edge (~36 per cfg3 search).
template <int W>
__device__ __forceinline__ int64_t upper_mst(const GraphSmem& g, uint32_t* tree, uint8_t* x,
                                             int32_t* par, uint32_t* levels, uint32_t* onpath,
                                             int L, int lane) {
  for (int v = lane; v < g.n; v += 32) par[v] = v;
  for (int i = lane; i < g.n * W; i += 32) tree[i] = 0;
  __syncwarp();
  BPROF_T(k0);
  // The maximum spanning forest by Boruvka rounds, warp-parallel (distinct weights =
  // edge indices, so the forest is Kruskal's): every component picks its largest-index
  // edge to another component (atomicMax per component), the picks join the forest,
  // components link along them (a mutual pick links the larger label to the smaller,
  // the only cycles being such pairs) and pointer jumping relabels; ~log2(n) rounds.
  // The rounds stop once s and t share a component: the forest then holds their
  // whole tree path.  (A lane-0 Kruskal union-find took ~105K cycles per search.)
  int32_t* lab = par;                      // component label (= parent pointer of roots)
  int32_t* best = reinterpret_cast<int32_t*>(levels);  // scratch until the BFS below
  while (true) {
    for (int v = lane; v < g.n; v += 32) best[v] = -1;
    __syncwarp();
    for (int e = lane; e < g.N; e += 32) {
      if (x[e] < L) continue;
      const int a = lab[g.eu[e]], c = lab[g.ev[e]];
      if (a != c) {
        atomicMax(&best[a], e);
        atomicMax(&best[c], e);
      }
    }
    __syncwarp();
    int link[W];  // new parent of each root this lane owns (read phase, then write)
#pragma unroll
    for (int q = 0; q < W; ++q) {
      const int r = 32 * q + lane;
      link[q] = -1;
      if (r < g.n && lab[r] == r && best[r] >= 0) {
        const int e = best[r];
        const int a = lab[g.eu[e]], c = lab[g.ev[e]];
        const int o = a == r ? c : a;
        const uint32_t u = g.eu[e], v = g.ev[e];
        atomicOr(&tree[u * W + (v >> 5)], 1u << (v & 31));
        atomicOr(&tree[v * W + (u >> 5)], 1u << (u & 31));
        link[q] = (best[o] == e && o > r) ? -1 : o;  // mutual pick: the larger label links
      }
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < W; ++q)
      if (link[q] >= 0) lab[32 * q + lane] = link[q];
    __syncwarp();
    while (true) {  // pointer jumping to the roots
      bool moved = false;
#pragma unroll
      for (int q = 0; q < W; ++q) {
        const int v = 32 * q + lane;
        if (v < g.n) {
          const int p = lab[v], pp = lab[p];
          if (pp != p) {
            lab[v] = pp;
            moved = true;
          }
        }
      }
      __syncwarp();
      if (!__any_sync(kFull, moved)) break;
    }
    if (lab[g.s] == lab[g.t]) break;
  }
  __syncwarp();
  BPROF_T(k1);
  BPROF_ADD(2, k1 - k0);
  AdjSmem<W> ta{tree};
  static_assert(!AdjSmem<W>::kRegisters, "tree adjacency lives in shared memory");
  uint32_t* lev_t = levels + g.n * W;
  Meet mt;
  bfs_bidir<W>(ta, levels, lev_t, g.n, g.s, g.t, lane, mt);  // s, t are connected in the tree
  trace_bidir<W>(g, ta, levels, lev_t, mt, onpath, lane);
  BPROF_T(k2);
  BPROF_ADD(4, k2 - k1);
  BPROF_ADD(1, 1);
  unsigned c = 0;
  for (int e = lane; e < g.N; e += 32) {
    const int xe = x[e];
    if (xe >= L && ((onpath[e >> 5] >> (e & 31)) & 1u)) {
      c += (unsigned)(xe - L + 1);
      x[e] = (uint8_t)L;
    } else {
      c += (unsigned)xe;
      x[e] = 0;
    }
  }
  const unsigned calls = __reduce_add_sync(kFull, c);
  __syncwarp();
  return calls;
}

template <int W>
__global__ void boundary_graph_kernel(const rsr_phi_desc d, int L, const uint8_t* __restrict__ x0,
                                      int64_t B, uint8_t* __restrict__ out_refs,
                                      uint8_t* __restrict__ out_side,
                                      int64_t* __restrict__ out_calls, int mst) {
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
  // offsets (not integer-cast pointers) keep every scratch pointer in the
  // shared address space, so the compiler emits LDS/STS instead of generic ops
  size_t off = align16(2 * sizeof(int32_t) * (size_t)g.N);
  g.eid = nullptr;
  if (g.n <= kEidMaxNodes) {
    int16_t* eid = reinterpret_cast<int16_t*>(smem + off);
    for (int i = threadIdx.x; i < g.n * g.n; i += blockDim.x) eid[i] = -1;
    __syncthreads();
    for (int e = threadIdx.x; e < g.N; e += blockDim.x) {
      eid[eu[e] * g.n + ev[e]] = (int16_t)e;
      eid[ev[e] * g.n + eu[e]] = (int16_t)e;
    }
    g.eid = eid;
    off += align16(2 * (size_t)g.n * g.n);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, warps = blockDim.x >> 5;
  uint8_t* mine = smem + off + (size_t)warp * warp_scratch<W>(g.N, g.n);
  uint8_t* x = mine;
  int32_t* par = reinterpret_cast<int32_t*>(mine + align16(g.N));
  uint32_t* onpath = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(par) + align16(4 * g.n));
  uint32_t* adj = reinterpret_cast<uint32_t*>(reinterpret_cast<uint8_t*>(onpath) +
                                              align16(4 * ((g.N + 31) / 32)));
  uint32_t* levels = adj + g.n * W;
  const int M = d.n_states;

  for (int64_t b = (int64_t)blockIdx.x * warps + warp; b < B; b += (int64_t)gridDim.x * warps) {
    BPROF_T(s0);
    BPROF_ADD(0, 1);
    const uint8_t* src = x0 + b * g.N;
    for (int e = lane; e < g.N; e += 32) x[e] = src[e];
    for (int v = lane; v < g.n; v += 32) par[v] = v;
    __syncwarp();
    // initial Phi(x0): components of G_L by warp-parallel min-label propagation
    // with pointer jumping; the converged labels (component minimum, roots point
    // to themselves) are a depth-1 union-find forest for the lower-side walk
    BPROF_T(i0);
    while (true) {
      bool changed = false;
      for (int e = lane; e < g.N; e += 32) {
        if (x[e] >= L) {
          const int a = par[eu[e]], c = par[ev[e]];
          if (a != c) {
            const int m = a < c ? a : c;
            atomicMin(&par[eu[e]], m);
            atomicMin(&par[ev[e]], m);
            atomicMin(&par[a], m);
            atomicMin(&par[c], m);
            changed = true;
          }
        }
      }
      __syncwarp();
      for (int v = lane; v < g.n; v += 32) {
        int r = par[v];
        while (par[r] != r) r = par[r];
        par[v] = r;
      }
      __syncwarp();
      if (!__any_sync(kFull, changed)) break;
    }
    const int connected = par[g.s] == par[g.t];
    BPROF_T(i1);
    BPROF_ADD(6, i1 - i0);
    int64_t calls = 1;
    if (!connected) {
      // ---------------- lower side: union-find, no Phi evaluation needed
      if (lane == 0) {
        // the roots of s and t are tracked through the links (no finds for them)
        int rs = uf_find(par, g.s), rt = uf_find(par, g.t);
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
          if ((a == rs && c == rt) || (a == rt && c == rs)) {
            x[n] = (uint8_t)(L - 1);  // crossing: reverted, walk moves to n + 1
            continue;
          }
          if (a != c) {
            par[a] = c;
            if (rs == a) rs = c;
            if (rt == a) rt = c;
          }
          calls += M - 1 - L;
          x[n] = (uint8_t)(M - 1);
        }
      }
    } else if (mst) {
      // ---------------- upper side: maximum spanning forest path (closed form)
      calls += upper_mst<W>(g, adj, x, par, levels, onpath, L, lane);
    } else {
      // ---------------- upper side: witness path + BFS for edges on it (round 1)
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
      if constexpr (W <= 4) {
        AdjReg<W> ra;
        ra.load(adj, g.n, lane);
        calls += upper_walk<W>(g, ra, adj, x, levels, onpath, L, lane);
      } else {
        AdjSmem<W> sa{adj};
        calls += upper_walk<W>(g, sa, adj, x, levels, onpath, L, lane);
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
    BPROF_T(s1);
    BPROF_ADD(7, s1 - s0);
  }
}

template <int W>
int launch_graph(const rsr_phi_desc& d, int L, const uint8_t* x0, int64_t B, uint8_t* out_refs,
                 uint8_t* out_side, int64_t* out_calls, cudaStream_t st) {
  const size_t fixed = align16(2 * sizeof(int32_t) * (size_t)d.n_components) +
                       (d.n_nodes <= kEidMaxNodes ? align16(2 * (size_t)d.n_nodes * d.n_nodes) : 0);
  const size_t per_warp = warp_scratch<W>(d.n_components, d.n_nodes);
  int warps = (int)((160 * 1024 - fixed) / per_warp);
  if (warps > 4) warps = 4;
  if (warps < 1) return -1;
  int64_t grid = (B + warps - 1) / warps;
  if (grid > 148 * 32) grid = 148 * 32;
  const size_t smem = fixed + warps * per_warp;
  auto k = boundary_graph_kernel<W>;
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // RSR_BOUNDARY_MST=0: the round-1 witness-path walk (A/B and cross-checks)
  static const int mst = [] {
    const char* e = getenv("RSR_BOUNDARY_MST");
    return e && atoi(e) == 0 ? 0 : 1;
  }();
  k<<<(unsigned)grid, warps * 32, smem, st>>>(d, L, x0, B, out_refs, out_side, out_calls, mst);
  return rsr::check_launch("boundary_graph_kernel");
}

}  // namespace

#ifdef RSR_FP4_PROF
extern "C" int rsr_boundary_prof(unsigned long long* host8, int reset) {
  RSR_CUDA(cudaMemcpyFromSymbol(host8, g_bprof, sizeof(g_bprof)));
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    RSR_CUDA(cudaMemcpyToSymbol(g_bprof, z, sizeof(z)));
  }
  return RSR_OK;
}
#endif

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
