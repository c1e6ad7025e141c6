// Philox4x64-10 issue-rate probe: how close is the sampler (sample_rows_kernel,
// 1.37 ms per 2^20 x 295 draws) to the cost of the bit-exact generator alone?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/philox_rate tools/philox_rate.cu
// Variants: (0) compiler __umul64hi, (1) explicit 32-bit mad chains (PTX
// mad.lo/hi.cc), (2) (0) plus the M=2 threshold compare into shared memory,
// (3) four independent 32x32->64 products, (4) the independent device stream's
// Philox4x32-10 (same number of draws).
#include <cstdio>
#include <cstdint>

#include "../paper_2604_17066_b200/csrc/philox.cuh"

__device__ __forceinline__ void mulhilo_ptx(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint32_t r0, r1, r2, r3;
  asm("{\n\t"
      "mul.lo.u32 %0, %4, %6;\n\t"
      "mul.hi.u32 %1, %4, %6;\n\t"
      "mad.lo.cc.u32 %1, %4, %7, %1;\n\t"
      "madc.hi.u32 %2, %4, %7, 0;\n\t"
      "mad.lo.cc.u32 %1, %5, %6, %1;\n\t"
      "madc.hi.cc.u32 %2, %5, %6, %2;\n\t"
      "addc.u32 %3, 0, 0;\n\t"
      "mad.lo.cc.u32 %2, %5, %7, %2;\n\t"
      "madc.hi.u32 %3, %5, %7, %3;\n\t"
      "}"
      : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)
      : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
  lo = ((uint64_t)r1 << 32) | r0;
  hi = ((uint64_t)r3 << 32) | r2;
}

// four independent 32x32->64 products, carries on the integer ALU pipe
__device__ __forceinline__ void mulhilo_wide4(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  uint32_t a0 = (uint32_t)a, a1 = (uint32_t)(a >> 32), b0 = (uint32_t)b, b1 = (uint32_t)(b >> 32);
  uint32_t m, h0, h1;
  uint32_t l0;
  asm("{\n\t.reg .u64 p00, p01, p10, p11;\n\t.reg .u32 q0, q1, r0, r1, s0, s1, t0, t1, c;\n\t"
      "mul.wide.u32 p00, %4, %6;\n\t"
      "mul.wide.u32 p01, %4, %7;\n\t"
      "mul.wide.u32 p10, %5, %6;\n\t"
      "mul.wide.u32 p11, %5, %7;\n\t"
      "mov.b64 {q0, q1}, p00;\n\t"
      "mov.b64 {r0, r1}, p01;\n\t"
      "mov.b64 {s0, s1}, p10;\n\t"
      "mov.b64 {t0, t1}, p11;\n\t"
      "mov.b32 %0, q0;\n\t"
      "add.cc.u32 %1, r0, s0;\n\t"
      "addc.u32 c, 0, 0;\n\t"
      "add.cc.u32 %1, %1, q1;\n\t"
      "addc.u32 c, c, 0;\n\t"
      "add.cc.u32 %2, t0, r1;\n\t"
      "addc.u32 %3, t1, 0;\n\t"
      "add.cc.u32 %2, %2, s1;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "add.cc.u32 %2, %2, c;\n\t"
      "addc.u32 %3, %3, 0;\n\t"
      "}"
      : "=r"(l0), "=r"(m), "=r"(h0), "=r"(h1)
      : "r"(a0), "r"(a1), "r"(b0), "r"(b1));
  lo = ((uint64_t)m << 32) | l0;
  hi = ((uint64_t)h1 << 32) | h0;
}

template <bool W4>
__device__ __forceinline__ void philox_ptx(uint64_t ctr0, uint64_t key0, uint64_t key1,
                                           uint64_t out[4]) {
  const uint64_t M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
  const uint64_t W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      key0 += W0;
      key1 += W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    if (W4) {
      mulhilo_wide4(M0, c0, hi0, lo0);
      mulhilo_wide4(M1, c2, hi1, lo1);
    } else {
      mulhilo_ptx(M0, c0, hi0, lo0);
      mulhilo_ptx(M1, c2, hi1, lo1);
    }
    const uint64_t n0 = hi1 ^ c1 ^ key0, n2 = hi0 ^ c3 ^ key1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

template <int V>
__global__ void __launch_bounds__(256) probe(int64_t nblk, uint64_t seed, uint64_t gen,
                                             uint64_t* out, const unsigned long long* Tg) {
  __shared__ unsigned long long T[512];
  __shared__ uint8_t st[8192];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) T[i] = Tg[i];
  __syncthreads();
  uint64_t acc = 0;
  int n = threadIdx.x % 295;
  for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nblk;
       b += (int64_t)gridDim.x * blockDim.x) {
    uint64_t w[4];
    if (V == 4) {  // the independent device stream (Philox4x32-10): 4 x 32-bit draws
      uint32_t u[4];
      rsr::device_row_block((uint64_t)b / 74, (uint32_t)(b % 74), seed, gen, u);
      w[0] = u[0]; w[1] = u[1]; w[2] = u[2]; w[3] = u[3];
    } else if (V == 1)
      philox_ptx<false>((uint64_t)b + 1, seed, gen, w);
    else if (V == 3)
      philox_ptx<true>((uint64_t)b + 1, seed, gen, w);
    else
      rsr::philox4x64_10((uint64_t)b + 1, seed, gen, w);
    if (V == 2) {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        st[(threadIdx.x * 4 + j) & 8191] = (w[j] >> 11) >= T[n];
        if (++n == 295) n = 0;
      }
    } else {
      acc ^= w[0] ^ w[1] ^ w[2] ^ w[3];
    }
  }
  if (V == 2) {
    __syncthreads();
    acc = st[threadIdx.x];
  }
  out[(int64_t)blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  const int64_t draws = (int64_t)(1 << 20) * 295, nblk = draws / 4;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint64_t* out;
  unsigned long long* T;
  cudaMalloc(&out, (size_t)sms * 64 * 256 * 8);
  cudaMalloc(&T, 512 * 8);
  cudaMemset(T, 0x11, 512 * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  // correctness of variant 3 against the library generator
  {
    uint64_t *o0, *o3;
    cudaMalloc(&o0, (size_t)sms * 4 * 256 * 8);
    cudaMalloc(&o3, (size_t)sms * 4 * 256 * 8);
    probe<0><<<sms * 4, 256>>>(1 << 20, 7, 9, o0, T);
    probe<3><<<sms * 4, 256>>>(1 << 20, 7, 9, o3, T);
    static uint64_t h0[148 * 4 * 256], h3[148 * 4 * 256];
    cudaMemcpy(h0, o0, (size_t)sms * 4 * 256 * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(h3, o3, (size_t)sms * 4 * 256 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < sms * 4 * 256; ++i) bad += h0[i] != h3[i];
    printf("variant 3 mismatches vs variant 0: %d\n", bad);
  }
  for (int v = 0; v < 5; ++v) {
    for (int ctas_per_sm : {4, 8}) {
      const int grid = sms * ctas_per_sm;
      auto k = v == 0   ? probe<0>
               : v == 1 ? probe<1>
               : v == 2 ? probe<2>
               : v == 3 ? probe<3>
                        : probe<4>;
      k<<<grid, 256>>>(nblk, 123, 4, out, T);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) k<<<grid, 256>>>(nblk, 123, 4, out, T);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      ms /= 10;
      printf("variant %d ctas/sm %2d: %.3f ms per 2^20 x 295 draws = %.1f G draws/s\n", v,
             ctas_per_sm, ms, draws / ms / 1e6);
    }
  }
  cudaError_t err = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(err));
  return 0;
}
