// Which 16 bits of each 32-bit TMEM column does tcgen05.ld ... .pack::16b keep?
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__global__ void probe(uint32_t* out) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  if (warp == 0) {
    // column c of lane l holds 0xAAAA0000 | (l << 8) | c  (high half 0xAAAA)
    uint32_t v0 = 0xAAAA0000u | (lane << 8) | 0, v1 = 0xAAAA0000u | (lane << 8) | 1,
             v2 = 0xAAAA0000u | (lane << 8) | 2, v3 = 0xAAAA0000u | (lane << 8) | 3;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tm), "r"(v0), "r"(v1),
                 "r"(v2), "r"(v3));
    asm volatile("tcgen05.wait::st.sync.aligned;");
    uint32_t r0, r1;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.pack::16b.b32 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(tm));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    out[lane * 2] = r0;
    out[lane * 2 + 1] = r1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tm));
}
int main() {
  uint32_t* d;
  cudaMalloc(&d, 256);
  probe<<<1, 128>>>(d);
  uint32_t h[64];
  cudaMemcpy(h, d, 256, cudaMemcpyDeviceToHost);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  for (int l = 0; l < 3; ++l) printf("lane %d: r0=%08x r1=%08x\n", l, h[2 * l], h[2 * l + 1]);
  return 0;
}
