// TMEM -> register read bandwidth per SM for the tcgen05.ld shapes that move
// 32 registers per thread, with 4 / 8 / 16 reading warps per CTA (one CTA per SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define LD32(shape, addr, v)                                                                     \
  asm volatile("tcgen05.ld.sync.aligned." shape ".b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
               "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];" \
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),       \
                 "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),     \
                 "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), \
                 "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), \
                 "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), \
                 "=r"(v[30]), "=r"(v[31])                                                      \
               : "r"(addr))

template <int SHAPE>
__global__ void tmem_read(int iters, unsigned long long* cyc, uint32_t* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
  const uint32_t col0 = (uint32_t)(warp >> 2) * 32;
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    const uint32_t addr = tm + lane_base + ((col0 + (uint32_t)i * 128) & 255);
    if (SHAPE == 0) LD32("32x32b.x32", addr, v);
    if (SHAPE == 1) LD32("16x64b.x32", addr, v);
    if (SHAPE == 2) LD32("16x128b.x16", addr, v);
    if (SHAPE == 3) LD32("16x256b.x8", addr, v);
    if (SHAPE == 4) LD32("32x32b.x32.pack::16b", addr, v);
    if (SHAPE == 5) LD32("16x64b.x32.pack::16b", addr, v);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int k = 0; k < 32; ++k) acc ^= v[k];
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int SHAPE>
void run(const char* name, int sms, int warps) {
  const int iters = 20000;
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, sms * 8);
  cudaMalloc(&sink, sms * warps * 32 * 4);
  tmem_read<SHAPE><<<sms, warps * 32>>>(100, d, sink);
  tmem_read<SHAPE><<<sms, warps * 32>>>(iters, d, sink);
  cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  // 32 regs x 4 B per thread; pack::16b covers two 32-bit TMEM columns per register
  const double bytes = (double)iters * warps * 32 * 32 * 4 * (SHAPE >= 4 ? 2 : 1);
  printf("%-12s warps=%2d: %.1f B/clk per SM (%s)\n", name, warps, bytes / c,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8, 16}) {
    run<0>("32x32b.x32", sms, w);
    run<1>("16x64b.x32", sms, w);
    run<2>("16x128b.x16", sms, w);
    run<3>("16x256b.x8", sms, w);
    run<4>("32x32b.x64.p16", sms, w);
    run<5>("16x64b.x64.p16", sms, w);
  }
  return 0;
}
