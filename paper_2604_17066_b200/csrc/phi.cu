// (3) Batched system-function evaluation and (4) batched boundary search.
//
// Replaces model.py:88-97 (SystemModel.evaluate) -> sysfn.py:62-185 (union-find
// s-t / global connectivity, k-out-of-n) plus the builder-defined widest-path
// level and the cone-sum monotone function of the reference test
// fixtures (tests/conftest.py:53-75); and boundary.py:116-147
// (boundary_search), boundary.py:50-54 (_redundant_under).
//
// One warp per sample.  Connectivity is label propagation over the alive edges
// (x_e >= level): lanes sweep the edge list, OR-ing a per-node reach flag in
// shared memory, until a sweep changes nothing (or t is reached).  The result
// equals the union-find answer of the reference: both compute the connected
// component of s in the alive subgraph.
#include <stdlib.h>

#include "common.cuh"

namespace {

constexpr int kWarps = 8;
constexpr unsigned kFull = 0xffffffffu;

struct Phi {
  int kind, N, M, n_nodes, s, t, k, n_anchors;
  const int32_t* eu;  // smem copies for graph kinds
  const int32_t* ev;
  const uint8_t* anchors;
  const int32_t* alevel;
};

__device__ bool reach_from(const Phi& f, const volatile uint8_t* x, volatile uint8_t* reach,
                           int source, int stop_at, int level, int lane) {
  __syncwarp();  // previous readers of reach[] are done
  for (int i = lane; i < f.n_nodes; i += 32) reach[i] = (uint8_t)(i == source);
  __syncwarp();
  bool result;
  while (true) {
    int changed = 0;
    for (int e = lane; e < f.N; e += 32) {
      if (x[e] >= level) {
        const int u = f.eu[e], v = f.ev[e];
        const uint8_t ru = reach[u], rv = reach[v];
        if (ru != rv) {
          reach[u] = 1;
          reach[v] = 1;
          changed = 1;
        }
      }
    }
    __syncwarp();
    const bool at_stop = stop_at >= 0 ? reach[stop_at] != 0 : true;
    if (!__any_sync(kFull, changed) || (stop_at >= 0 && at_stop)) {
      result = at_stop;
      break;
    }
  }
  __syncwarp();
  return result;
}

// Unit-capacity max-flow from node 0 to every t, capped at the running minimum
// (sysfn.py:112-174).  Arc 2e / 2e+1 are the two directions of edge e, each of
// capacity 1 when x_e >= 1; augmenting along arc a moves a unit to a ^ 1.  BFS
// parents are claimed with atomicCAS so the BFS tree stays acyclic; the flow
// value (hence Phi) does not depend on which augmenting paths are found.
__device__ int edge_disjoint_warp(const Phi& f, const volatile uint8_t* x, volatile uint8_t* res,
                                  volatile int* parent, int lane) {
  int level = f.k;
  for (int t = 1; t < f.n_nodes && level > 0; ++t) {
    __syncwarp();
    for (int a = lane; a < 2 * f.N; a += 32) res[a] = x[a >> 1] >= 1 ? 1 : 0;
    __syncwarp();
    int flow = 0;
    while (flow < level) {
      for (int v = lane; v < f.n_nodes; v += 32) parent[v] = v == 0 ? -2 : -1;
      __syncwarp();
      int reached = 0;
      while (true) {
        int changed = 0;
        for (int a = lane; a < 2 * f.N; a += 32) {
          if (res[a]) {
            const int e = a >> 1;
            const int u = (a & 1) ? f.ev[e] : f.eu[e];
            const int v = (a & 1) ? f.eu[e] : f.ev[e];
            if (parent[u] != -1 && parent[v] == -1 &&
                atomicCAS(const_cast<int*>(&parent[v]), -1, a) == -1)
              changed = 1;
          }
        }
        __syncwarp();
        reached = __shfl_sync(kFull, lane == 0 ? (parent[t] != -1) : 0, 0);
        if (reached || !__any_sync(kFull, changed)) break;
      }
      if (!reached) break;
      if (lane == 0) {
        int v = t;
        while (v != 0) {
          const int a = parent[v];
          res[a] = (uint8_t)(res[a] - 1);
          res[a ^ 1] = (uint8_t)(res[a ^ 1] + 1);
          const int e = a >> 1;
          v = (a & 1) ? f.ev[e] : f.eu[e];  // tail of arc a
        }
      }
      __syncwarp();
      ++flow;
    }
    if (flow < level) level = flow;
  }
  return level;
}

__device__ int phi_warp(const Phi& f, const volatile uint8_t* x, volatile uint8_t* reach, int lane,
                        volatile uint8_t* xtra) {
  switch (f.kind) {
    case RSR_PHI_EDGE_DISJOINT:
      return edge_disjoint_warp(
          f, x, xtra, reinterpret_cast<volatile int*>(xtra + ((2 * (size_t)f.N + 15) / 16 * 16)),
          lane);
    case RSR_PHI_ST_CONNECTIVITY:
      return reach_from(f, x, reach, f.s, f.t, 1, lane) ? 1 : 0;
    case RSR_PHI_WIDEST_PATH:
      for (int level = f.M - 1; level >= 1; --level)
        if (reach_from(f, x, reach, f.s, f.t, level, lane)) return level;
      return 0;
    case RSR_PHI_GLOBAL_CONNECTIVITY: {
      reach_from(f, x, reach, 0, -1, 1, lane);
      int all = 1;
      for (int i = lane; i < f.n_nodes; i += 32) all &= reach[i] != 0;
      return __all_sync(kFull, all) ? 1 : 0;
    }
    case RSR_PHI_K_OUT_OF_N: {
      for (int v = f.M - 1; v >= 1; --v) {
        int c = 0;
        for (int e = lane; e < f.N; e += 32) c += x[e] >= v;
#pragma unroll
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
        if (c >= f.k) return v;
      }
      return 0;
    }
    case RSR_PHI_CONE_SUM: {
      unsigned levels_hit = 0;
      for (int a = 0; a < f.n_anchors; ++a) {
        const uint8_t* an = f.anchors + (int64_t)a * f.N;
        int ok = 1;
        for (int e = lane; e < f.N; e += 32) ok &= x[e] >= an[e];
        if (__all_sync(kFull, ok)) levels_hit |= 1u << f.alevel[a];
      }
      return __popc(levels_hit);
    }
  }
  return 0;
}

// Shared-memory layout per block: edges (graph kinds), then per warp x[N] and
// reach[n_nodes].
__device__ Phi load_phi(const rsr_phi_desc& d, uint8_t* smem, int32_t** tail) {
  Phi f;
  f.kind = d.kind;
  f.N = d.n_components;
  f.M = d.n_states;
  f.n_nodes = d.n_nodes;
  f.s = d.source;
  f.t = d.target;
  f.k = d.k;
  f.n_anchors = d.n_anchors;
  f.anchors = d.anchors;
  f.alevel = d.anchor_level;
  int32_t* eu = reinterpret_cast<int32_t*>(smem);
  int32_t* ev = eu + (d.edge_u ? f.N : 0);
  if (d.edge_u) {
    for (int i = threadIdx.x; i < f.N; i += blockDim.x) {
      eu[i] = d.edge_u[i];
      ev[i] = d.edge_v[i];
    }
  }
  f.eu = eu;
  f.ev = ev;
  *tail = ev + (d.edge_u ? f.N : 0);
  __syncthreads();
  return f;
}

// per warp: x[N] + reach[n] (+ edge-disjoint: res[2N] + parent[n] int32)
__host__ __device__ inline size_t base_warp_bytes(int N, int n) {
  return ((size_t)N + (size_t)n + 15) / 16 * 16;
}
__host__ __device__ inline size_t warp_bytes(int kind, int N, int n) {
  size_t b = base_warp_bytes(N, n);
  if (kind == RSR_PHI_EDGE_DISJOINT) b += (2 * (size_t)N + 15) / 16 * 16 + 4 * (size_t)n;
  return (b + 15) / 16 * 16;
}

__host__ __device__ inline size_t phi_smem_bytes(const rsr_phi_desc& d) {
  const size_t edges = d.edge_u ? 2 * sizeof(int32_t) * (size_t)d.n_components : 0;
  return edges + kWarps * warp_bytes(d.kind, d.n_components, d.n_nodes);
}

__global__ void __launch_bounds__(kWarps * 32)
phi_eval_kernel(const rsr_phi_desc d, const uint8_t* __restrict__ states,
                const int64_t* __restrict__ idx, int64_t count, uint8_t* __restrict__ out,
                int threshold, unsigned long long* count_leq) {
  extern __shared__ uint8_t smem[];
  int32_t* tail;
  const Phi f = load_phi(d, smem, &tail);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = warp_bytes(f.kind, f.N, f.n_nodes);
  volatile uint8_t* x = reinterpret_cast<uint8_t*>(tail) + warp * per_warp;
  volatile uint8_t* reach = x + f.N;
  volatile uint8_t* xtra = x + base_warp_bytes(f.N, f.n_nodes);
  unsigned long long leq = 0;
  for (int64_t i = (int64_t)blockIdx.x * kWarps + warp; i < count;
       i += (int64_t)gridDim.x * kWarps) {
    const int64_t row = idx ? idx[i] : i;
    const uint8_t* src = states + row * f.N;
    for (int e = lane; e < f.N; e += 32) x[e] = src[e];
    __syncwarp();
    const int v = phi_warp(f, x, reach, lane, xtra);
    if (lane == 0 && out) out[i] = (uint8_t)v;
    leq += (v <= threshold);
    __syncwarp();
  }
  if (count_leq && lane == 0 && leq) atomicAdd(count_leq, leq);
}

__global__ void __launch_bounds__(kWarps * 32)
boundary_kernel(const rsr_phi_desc d, int threshold, const uint8_t* __restrict__ x0, int64_t B,
                uint8_t* __restrict__ out_refs, uint8_t* __restrict__ out_side,
                int64_t* __restrict__ out_calls) {
  extern __shared__ uint8_t smem[];
  int32_t* tail;
  const Phi f = load_phi(d, smem, &tail);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = warp_bytes(f.kind, f.N, f.n_nodes);
  volatile uint8_t* x = reinterpret_cast<uint8_t*>(tail) + warp * per_warp;
  volatile uint8_t* reach = x + f.N;
  volatile uint8_t* xtra = x + base_warp_bytes(f.N, f.n_nodes);
  for (int64_t b = (int64_t)blockIdx.x * kWarps + warp; b < B; b += (int64_t)gridDim.x * kWarps) {
    const uint8_t* src = x0 + b * f.N;
    for (int e = lane; e < f.N; e += 32) x[e] = src[e];
    __syncwarp();
    int64_t calls = 1;
    const bool lower = phi_warp(f, x, reach, lane, xtra) <= threshold;
    const int step = lower ? 1 : -1, limit = lower ? f.M - 1 : 0;
    for (int n = 0; n < f.N; ++n) {
      while (x[n] != limit) {
        __syncwarp();
        if (lane == 0) x[n] = (uint8_t)(x[n] + step);
        __syncwarp();
        const int s = phi_warp(f, x, reach, lane, xtra);
        ++calls;
        const bool crossed = lower ? (s > threshold) : (s <= threshold);
        if (crossed) {
          __syncwarp();
          if (lane == 0) x[n] = (uint8_t)(x[n] - step);
          __syncwarp();
          break;
        }
      }
    }
    __syncwarp();
    uint8_t* dst = out_refs + b * f.N;
    for (int e = lane; e < f.N; e += 32) dst[e] = x[e];
    if (lane == 0) {
      out_side[b] = lower ? RSR_SIDE_LOWER : RSR_SIDE_UPPER;
      out_calls[b] = calls;
    }
    __syncwarp();
  }
}

__global__ void gather_kernel(const uint8_t* __restrict__ states, int N,
                              const int64_t* __restrict__ idx, int64_t count,
                              uint8_t* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count * N) return;
  const int64_t i = t / N;
  const int n = (int)(t - i * N);
  out[t] = states[idx[i] * N + n];
}

// a is redundant given b: lower a <= b, upper a >= b (boundary.py:50-54)
__device__ __forceinline__ bool redundant_under(int side, const uint8_t* a, const uint8_t* b,
                                                int N) {
  if (side == RSR_SIDE_LOWER) {
    for (int n = 0; n < N; ++n)
      if (a[n] > b[n]) return false;
  } else {
    for (int n = 0; n < N; ++n)
      if (a[n] < b[n]) return false;
  }
  return true;
}

__global__ void dominance_kernel(const uint8_t* __restrict__ cands, int64_t B,
                                 const uint8_t* __restrict__ members, int64_t K, int N, int side,
                                 uint8_t* covered, uint8_t* covers, int mask_c,
                                 uint8_t* member_mask) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t c = blockIdx.y;
  if (m >= K || c >= B) return;
  const uint8_t* cv = cands + c * N;
  const uint8_t* mv = members + m * N;
  const bool red = redundant_under(side, cv, mv, N);
  if (covered && red) covered[c] = 1;
  const bool dropped = redundant_under(side, mv, cv, N);
  if (covers && dropped) covers[c] = 1;
  if (member_mask) {
    if (mask_c < 0)  // full relation matrix [B x K]
      member_mask[c * K + m] = (uint8_t)((dropped ? 1 : 0) | (red ? 2 : 0));
    else if (c == mask_c)
      member_mask[m] = dropped ? 1 : 0;
  }
}

int check_phi(const rsr_phi_desc* d) {
  RSR_REQUIRE(d != nullptr, "null phi descriptor");
  RSR_REQUIRE(d->n_components >= 1 && d->n_states >= 2, "phi: bad N/M");
  switch (d->kind) {
    case RSR_PHI_ST_CONNECTIVITY:
    case RSR_PHI_WIDEST_PATH:
      RSR_REQUIRE(d->source >= 0 && d->source < d->n_nodes && d->target >= 0 &&
                      d->target < d->n_nodes && d->source != d->target,
                  "phi: bad source/target");
      /* fallthrough */
    case RSR_PHI_GLOBAL_CONNECTIVITY:
      RSR_REQUIRE(d->edge_u && d->edge_v && d->n_nodes >= 1, "phi: graph kinds need edges");
      break;
    case RSR_PHI_K_OUT_OF_N:
      RSR_REQUIRE(d->k >= 1 && d->k <= d->n_components, "phi: bad k");
      break;
    case RSR_PHI_EDGE_DISJOINT:
      RSR_REQUIRE(d->edge_u && d->edge_v && d->n_nodes >= 2 && d->k >= 1,
                  "phi: edge_disjoint_level needs edges, >= 2 nodes and max_level >= 1");
      break;
    case RSR_PHI_CONE_SUM:
      RSR_REQUIRE(d->n_anchors >= 0 && (d->n_anchors == 0 || (d->anchors && d->anchor_level)),
                  "phi: cone sum needs anchors");
      break;
    default:
      RSR_REQUIRE(false, "phi: unknown kind %d", d->kind);
  }
  RSR_REQUIRE(phi_smem_bytes(*d) <= 200 * 1024, "phi: graph too large for shared memory");
  return RSR_OK;
}

int grid_for(int64_t items) {
  int64_t g = rsr::ceil_div(items, kWarps);
  if (g > 148 * 16) g = 148 * 16;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

extern "C" int rsr_phi_eval(const rsr_phi_desc* phi, const uint8_t* states, const int64_t* idx,
                            int64_t count, uint8_t* out, int threshold, int64_t* count_leq,
                            void* stream) {
  int rc = check_phi(phi);
  if (rc) return rc;
  RSR_REQUIRE(count >= 0, "rsr_phi_eval: negative count");
  if (count == 0) return RSR_OK;
  const char* bits_env = getenv("RSR_PHI_BITS");
  if (!(bits_env && atoi(bits_env) == 0)) {
    const int r = rsr::phi_bits_dispatch(*phi, false, threshold, states, idx, count, out,
                                         count_leq, nullptr, nullptr, rsr::as_stream(stream));
    if (r != -1) return r;
  }
  const size_t smem = phi_smem_bytes(*phi);
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(phi_eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  phi_eval_kernel<<<grid_for(count), kWarps * 32, smem, rsr::as_stream(stream)>>>(
      *phi, states, idx, count, out, threshold,
      reinterpret_cast<unsigned long long*>(count_leq));
  return rsr::check_launch("phi_eval_kernel");
}

extern "C" int rsr_boundary_search(const rsr_phi_desc* phi, int threshold, const uint8_t* x0,
                                   int64_t B, uint8_t* out_refs, uint8_t* out_side,
                                   int64_t* out_calls, void* stream) {
  int rc = check_phi(phi);
  if (rc) return rc;
  RSR_REQUIRE(B >= 0, "rsr_boundary_search: negative count");
  if (B == 0) return RSR_OK;
  const char* graph_env = getenv("RSR_BOUNDARY_GRAPH");
  if (!(graph_env && atoi(graph_env) == 0)) {
    const int r = rsr::boundary_graph_dispatch(*phi, threshold, x0, B, out_refs, out_side,
                                               out_calls, rsr::as_stream(stream));
    if (r != -1) return r;
  }
  const char* bits_env = getenv("RSR_PHI_BITS");
  if (!(bits_env && atoi(bits_env) == 0)) {
    const int r = rsr::phi_bits_dispatch(*phi, true, threshold, x0, nullptr, B, out_refs, nullptr,
                                         out_side, out_calls, rsr::as_stream(stream));
    if (r != -1) return r;
  }
  const size_t smem = phi_smem_bytes(*phi);
  if (smem > 48 * 1024)
    RSR_CUDA(cudaFuncSetAttribute(boundary_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)smem));
  boundary_kernel<<<grid_for(B), kWarps * 32, smem, rsr::as_stream(stream)>>>(
      *phi, threshold, x0, B, out_refs, out_side, out_calls);
  return rsr::check_launch("boundary_kernel");
}

// Exact enumeration (oracle.py:49-63, CLI `oracle --mode exact`): vector number
// `first + i` in itertools.product order (last component fastest) and its
// probability prod_n probs[n, x_n], multiplied in component order like the
// reference's scalar loop.
namespace {
__global__ void enumerate_kernel(const double* __restrict__ probs, int N, int M, int64_t first,
                                 int64_t count, uint8_t* __restrict__ out,
                                 double* __restrict__ prob) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  int64_t code = first + i;
  uint8_t* row = out + i * N;
  for (int n = N - 1; n >= 0; --n) {
    row[n] = (uint8_t)(code % M);
    code /= M;
  }
  double p = 1.0;
  for (int n = 0; n < N; ++n) p = __dmul_rn(p, probs[(int64_t)n * M + row[n]]);
  prob[i] = p;
}

// mass[s] += p and count[s] += 1 in enumeration order (single thread: the
// reference's sequential float64 sum, oracle.py:56-61).
__global__ void state_mass_kernel(const uint8_t* __restrict__ phi, const double* __restrict__ prob,
                                  int64_t count, int n_sys, double* mass, int64_t* counts) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t i = 0; i < count; ++i) {
    const int s = phi[i];
    if (s < n_sys) {
      mass[s] = __dadd_rn(mass[s], prob[i]);
      counts[s] += 1;
    }
  }
}

}  // namespace

extern "C" int rsr_state_mass(const uint8_t* phi_values, const double* probs, int64_t count,
                              int n_system_states, double* mass, int64_t* counts, void* stream) {
  RSR_REQUIRE(count >= 0 && n_system_states >= 1, "rsr_state_mass: bad arguments");
  if (count == 0) return RSR_OK;
  state_mass_kernel<<<1, 1, 0, rsr::as_stream(stream)>>>(phi_values, probs, count, n_system_states,
                                                         mass, counts);
  return rsr::check_launch("state_mass_kernel");
}

extern "C" int rsr_enumerate_states(const double* probs, int n_components, int n_states,
                                    int64_t first, int64_t count, uint8_t* out_states,
                                    double* out_prob, void* stream) {
  RSR_REQUIRE(n_components >= 1 && n_states >= 2 && first >= 0 && count >= 0,
              "rsr_enumerate_states: bad arguments");
  if (count == 0) return RSR_OK;
  enumerate_kernel<<<(unsigned)rsr::ceil_div(count, 256), 256, 0, rsr::as_stream(stream)>>>(
      probs, n_components, n_states, first, count, out_states, out_prob);
  return rsr::check_launch("enumerate_kernel");
}

extern "C" int rsr_gather_rows(const uint8_t* states, int n_components, const int64_t* idx,
                               int64_t count, uint8_t* out, void* stream) {
  RSR_REQUIRE(n_components >= 1 && count >= 0, "rsr_gather_rows: bad shape");
  if (count == 0) return RSR_OK;
  const int64_t total = count * n_components;
  gather_kernel<<<(unsigned)rsr::ceil_div(total, 256), 256, 0, rsr::as_stream(stream)>>>(
      states, n_components, idx, count, out);
  return rsr::check_launch("gather_kernel");
}

extern "C" int rsr_dominance_scan(const uint8_t* cands, int64_t B, const uint8_t* members,
                                  int64_t K, int n_components, int side, uint8_t* covered,
                                  uint8_t* covers, int mask_candidate, uint8_t* member_mask,
                                  void* stream) {
  RSR_REQUIRE(B >= 0 && K >= 0 && n_components >= 1, "rsr_dominance_scan: bad shape");
  RSR_REQUIRE(side == RSR_SIDE_LOWER || side == RSR_SIDE_UPPER, "rsr_dominance_scan: bad side");
  RSR_REQUIRE(B <= 65535, "rsr_dominance_scan: at most 65535 candidates per call");
  cudaStream_t st = rsr::as_stream(stream);
  if (covered && B) RSR_CUDA(cudaMemsetAsync(covered, 0, B, st));
  if (covers && B) RSR_CUDA(cudaMemsetAsync(covers, 0, B, st));
  if (B == 0 || K == 0) return RSR_OK;
  dim3 grid((unsigned)rsr::ceil_div(K, 128), (unsigned)B);
  dominance_kernel<<<grid, 128, 0, st>>>(cands, B, members, K, n_components, side, covered,
                                         covers, mask_candidate, member_mask);
  return rsr::check_launch("dominance_kernel");
}
