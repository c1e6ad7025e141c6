// Write bandwidth of the FP4 operand layout: 2^20 rows x 320 B written as
// 32-bit words (up half, lo half), vs cudaMemset, vs 16-byte stores.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
__global__ void words_kernel(uint8_t* out, int rows, int words) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= rows * words) return;
  int i = t / words, w = t - i * words;
  uint32_t* row = reinterpret_cast<uint32_t*>(out + (int64_t)i * 8 * words);
  row[w] = t;
  row[words + w] = ~t;
}
__global__ void vec_kernel(uint4* out, int64_t n) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = make_uint4(t, t, t, t);
}
int main() {
  const int rows = 1 << 20, words = 40;
  const size_t bytes = (size_t)rows * 8 * words;
  uint8_t* d;
  cudaMalloc(&d, bytes);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    cudaMemsetAsync(d, 1, bytes);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("memset %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a);
    words_kernel<<<(rows * words + 255) / 256, 256>>>(d, rows, words);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("word stores %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
    cudaEventRecord(a);
    vec_kernel<<<(bytes / 16 + 255) / 256, 256>>>((uint4*)d, bytes / 16);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("16B stores %.3f ms %.0f GB/s\n", ms, bytes / ms / 1e6);
  }
  return 0;
}
