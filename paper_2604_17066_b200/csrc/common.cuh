// Shared helpers for librsr_b200: error reporting and small device utilities.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "../../include/rsr_b200.h"

namespace rsr {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Return RSR_ECUDA with a message if the last launch failed.
int check_launch(const char* what);

// cudaFuncAttributeMaxDynamicSharedMemorySize >= bytes for kernel fn on the
// current device, set once per (device, kernel) and size.
int ensure_dynamic_smem(const void* fn, size_t bytes);

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// csrc/phi_bits.cu: bitset-BFS Phi / boundary search for simple graphs
// (returns -1 when not applicable).
int phi_bits_dispatch(const rsr_phi_desc& d, bool boundary, int threshold, const uint8_t* states,
                      const int64_t* idx, int64_t count, uint8_t* out, int64_t* count_leq,
                      uint8_t* out_side, int64_t* out_calls, cudaStream_t st);

// csrc/boundary_graph.cu: boundary search by union-find / witness-path BFS for
// s-t connectivity and widest-path Phi (returns -1 when not applicable).
int boundary_graph_dispatch(const rsr_phi_desc& d, int threshold, const uint8_t* x0, int64_t B,
                            uint8_t* out_refs, uint8_t* out_side, int64_t* out_calls,
                            cudaStream_t st);

// Thermometer geometry (see include/rsr_b200.h).
inline int thermo_kdim(int n, int m) { return n * (m - 1); }
inline int thermo_bias_cols(int n, int m) { return (thermo_kdim(n, m) + 126) / 127; }
inline int thermo_kpad(int n, int m) {
  int need = thermo_kdim(n, m) + thermo_bias_cols(n, m);
  return (need + 31) / 32 * 32;
}

}  // namespace rsr

#define RSR_REQUIRE(cond, ...)        \
  do {                                \
    if (!(cond)) {                    \
      rsr::set_error(__VA_ARGS__);    \
      return RSR_EINVAL;              \
    }                                 \
  } while (0)

#define RSR_CUDA(call)                                                          \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                    \
      rsr::set_error("%s failed: %s", #call, cudaGetErrorString(e_));           \
      return RSR_ECUDA;                                                         \
    }                                                                           \
  } while (0)
