// Microbenchmark: issue rate of tcgen05.mma.kind::i8 for candidate tile shapes.
// One CTA per SM, one thread issues `iters` MMAs from shared memory operands
// (contents irrelevant), commits, waits; reports cycles per MMA and TOPS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t s) {
  return (uint64_t)((s >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void commit(uint32_t b, int mode) {
  if (mode & 64)
    asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(b));
  else
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b));
}

template <int N, int KSTEPS>
__global__ void __launch_bounds__(384, 1) mma_loop(int iters, unsigned long long* cyc, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  uint8_t* A = base;              // mode&1: 6 tiles of 16 KB, else 1 tile
  uint8_t* B = base + ((mode & 1) ? 6 * 16384 : 16384);      // mode&1: 8 stages, else 1
  __shared__ uint64_t bar, bar2, bar3;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar2)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar3)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if ((mode & 64) ? (warp == 0) : (threadIdx.x == 0)) {
    long long t0 = clock64();
    const uint32_t id = idesc(128, N);
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tm + (uint32_t)((i & 1) * (512 / 2 >= N ? N : 0));
      const int stage = (mode & 1) ? (i & 3) : 0;
#pragma unroll
      for (int k = 0; k < KSTEPS; ++k) {
        const int at = (mode & 1) ? ((i & 1) * 3 + (k >> 2) % 3) : 0;
        const uint64_t a = desc(sa(A) + at * 16384 + (k & 3) * 32),
                       b = desc(sa(B) + stage * (N * 128) + (k & 3) * 32);
        if (mode & 64)
          asm volatile("{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                       "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a),
                       "l"(b), "r"(id), "r"(k));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                       "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(d), "l"(a),
                       "l"(b), "r"(id), "r"(k));
      }
      if (mode & 2)
        commit(sa(&bar2), mode);
      if (mode & 8) {  // wait on an already-completed phase (parity 1 of a fresh barrier)
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 1; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(sa(&bar3)));
      }
      if (mode & 16) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      if (mode & 32) {  // wait for this iteration's MMAs: commit + wait (full drain)
        commit(sa(&bar), mode);
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                       : "=r"(ok) : "r"(sa(&bar)), "r"(i & 1));
      }
    }
    if (!(mode & 32)) {
      commit(sa(&bar), mode);
      uint32_t done = 0;
      while (!done)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                     : "=r"(done) : "r"(sa(&bar)));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) {
      cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar3)));
    }
  } else if ((mode & 4) && warp >= 4) {
    uint32_t done = 0;
    while (!done)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(done) : "r"(sa(&bar3)));
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int KSTEPS>
void run(int sms, int mode) {
  const int iters = 4000;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  auto k = mma_loop<N, KSTEPS>;
  const int smem = 6 * 16384 + 4 * N * 128 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k<<<sms, 384, smem>>>(100, d, mode);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<sms, 384, smem>>>(iters, d, mode);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double mmas = (double)iters * KSTEPS;
  double ops = 2.0 * 128 * N * 32 * mmas * sms;
  printf("mode %d M=128 N=%3d ksteps/iter=%d: %.1f cycles/MMA (ideal %d), %.0f TOPS, err=%s\n", mode, N, KSTEPS,
         c / mmas, 128 * N / 256, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int mode : {0, 3, 64, 64 + 3, 64 + 24, 64 + 27, 64 + 32}) run<128, 8>(sms, mode);
  for (int mode : {64, 64 + 32}) run<128, 20>(sms, mode);
  for (int mode : {64, 64 + 27}) run<256, 4>(sms, mode);
  return 0;
}
