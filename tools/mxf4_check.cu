// Probe of tcgen05.mma.kind::mxf4.block_scale (packed e2m1 operands, unit
// ue8m0 scales in TMEM) for the FP4 variant of the dominance classifier:
//   1. correctness: one CTA, M=128, N=NT, K=320 of random 0/1 operands laid out
//      K-major with the 128-byte swizzle; D (fp32) must equal the integer dot
//      products computed on the host;
//   2. issue rate: back-to-back MMAs on every SM, cycles per MMA and TOPS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mxf4_check mxf4_check.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t s) {
  return (uint64_t)((s >> 4) & 0x3FFF) | (1ull << 16) | (64ull << 32) | (1ull << 46) | (2ull << 61);
}
// block-scaled descriptor: a/b format E2M1 (=1 for kind::mxf4), scale ue8m0, K=64
__host__ __device__ constexpr uint32_t idesc_mxf4(int m, int n) {
  return (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (1u << 23) |
         ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void mma_mxf4(uint32_t d, uint64_t a, uint64_t b, uint32_t id,
                                         uint32_t sfa, uint32_t sfb, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc), "r"(sfa), "r"(sfb));
}

__device__ __forceinline__ void commit(uint32_t b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b));
}
__device__ __forceinline__ void wait0(uint32_t b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                 : "=r"(ok) : "r"(b), "r"(par));
}

// Fill TMEM columns [col0, col0+32) of all 128 lanes with unit ue8m0 scales.
__device__ __forceinline__ void fill_scales(uint32_t tm, int col0, uint32_t va = 0x7F7F7F7Fu,
                                            uint32_t vb = 0x7F7F7F7Fu) {
  const int warp = threadIdx.x / 32;
  const uint32_t v = va;
  uint32_t addr = tm + ((uint32_t)(warp * 32) << 16) + col0;
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,"
      "%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr),
      "r"(v));
  if (vb != va) {  // second 16 columns (SFB at col0 + 16) get vb
    addr += 16;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(addr),
        "r"(vb));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
}

// image: A tile (2 k-blocks x 128 rows x 128 B) then B tile (2 x NT x 128 B)
template <int NT>
__global__ void __launch_bounds__(128, 1) check_kernel(const uint8_t* img, int img_bytes, float* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < img_bytes / 16; i += blockDim.x)
    reinterpret_cast<uint4*>(base)[i] = reinterpret_cast<const uint4*>(img)[i];
  asm volatile("fence.proxy.async.shared::cta;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  fill_scales(tm, 480);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    const uint32_t A = sa(base), B = A + 2 * 128 * 128;
    for (int ks = 0; ks < 5; ++ks) {
      const int kb = ks / 4, off = (ks % 4) * 32;
      mma_mxf4(tm, desc(A + kb * 128 * 128 + off), desc(B + kb * NT * 128 + off), idesc_mxf4(128, NT),
               tm + 480, tm + 496, ks > 0);
    }
    commit(sa(&bar));
  }
  __syncwarp();
  wait0(sa(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = threadIdx.x;
  for (int c = 0; c < NT; c += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int i = 0; i < 8; ++i) out[row * NT + c + i] = __uint_as_float(v[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

__device__ __forceinline__ uint64_t desc32(uint32_t s);
template <int N, bool SW32>
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  fill_scales(tm, 480);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t A = sa(base), B = A + 16384;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tm + (uint32_t)((i & 1) * 240);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t a = SW32 ? desc32(A + k * 4096) : desc(A + k * 32),
                       b = SW32 ? desc32(B + k * 8192) : desc(B + k * 32);
        asm volatile(
            "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
            "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc_mxf4(128, N)), "r"(k), "r"(tm + 480), "r"(tm + 496));
      }
    }
    asm volatile("{.reg .pred e; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];}" ::"r"(sa(&bar)));
    wait0(sa(&bar), 0);
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static int swz(int r, int byte) {  // offset of (row r, byte) in a 128B-swizzled K-major k-block
  const int c = byte / 16, w = byte % 16;
  return (r / 8) * 1024 + (r % 8) * 128 + ((c ^ (r % 8)) * 16) + w;
}

template <int NT>
int check() {
  const int K = 320;
  static uint8_t a[128][K], b[NT][K];
  srand(7 + NT);
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < K; ++k) a[r][k] = (k < 295) ? (rand() % 3 == 0) : 0;
  for (int r = 0; r < NT; ++r)
    for (int k = 0; k < K; ++k) b[r][k] = (k < 295) ? (rand() % 3 != 0) : 0;
  const int abytes = 2 * 128 * 128, bbytes = 2 * NT * 128;
  uint8_t* img = (uint8_t*)calloc(abytes + bbytes, 1);
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < K; k += 2) {
      const int byte = k / 2, kb = byte / 128;
      img[kb * 128 * 128 + swz(r, byte % 128)] = (uint8_t)((a[r][k] ? 0x2 : 0) | (a[r][k + 1] ? 0x20 : 0));
    }
  for (int r = 0; r < NT; ++r)
    for (int k = 0; k < K; k += 2) {
      const int byte = k / 2, kb = byte / 128;
      img[abytes + kb * NT * 128 + swz(r, byte % 128)] =
          (uint8_t)((b[r][k] ? 0x2 : 0) | (b[r][k + 1] ? 0x20 : 0));
    }
  uint8_t* dimg;
  float* dout;
  cudaMalloc(&dimg, abytes + bbytes);
  cudaMalloc(&dout, 128 * NT * 4);
  cudaMemcpy(dimg, img, abytes + bbytes, cudaMemcpyHostToDevice);
  const int smem = abytes + bbytes + 1024;
  cudaFuncSetAttribute(check_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  check_kernel<NT><<<1, 128, smem>>>(dimg, abytes + bbytes, dout);
  cudaError_t e = cudaDeviceSynchronize();
  static float out[128 * NT];
  cudaMemcpy(out, dout, sizeof(out), cudaMemcpyDeviceToHost);
  int bad = 0, zeros = 0;
  for (int r = 0; r < 128; ++r)
    for (int n = 0; n < NT; ++n) {
      int s = 0;
      for (int k = 0; k < K; ++k) s += a[r][k] * b[n][k];
      zeros += s == 0;
      if (out[r * NT + n] != (float)s) {
        if (bad < 5) printf("  mismatch r=%d n=%d got %f want %d\n", r, n, out[r * NT + n], s);
        ++bad;
      }
    }
  printf("check N=%d: %s, %d mismatches of %d (exact zeros %d)\n", NT, cudaGetErrorString(e), bad, 128 * NT,
         zeros);
  cudaFree(dimg);
  cudaFree(dout);
  free(img);
  return bad;
}


// ---- 3. SW32 layout via one 3-D TMA box per operand (the classifier's layout):
// global rows of `rowb` bytes viewed as {32 B, rows, chunks} with strides
// {rowb, 32}; box {32, rows, chunks} lands as [chunk][row][32 B], 32-byte swizzle.
__device__ __forceinline__ uint64_t desc32(uint32_t s) {
  return (uint64_t)((s >> 4) & 0x3FFF) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) | (1ull << 46) |
         (6ull << 61);
}

template <int NT>
__global__ void __launch_bounds__(128, 1)
check_tma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb, float* out,
                 uint32_t sfa, uint32_t sfb) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t bar, tbar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  const uint32_t A = sa(base), B = A + 10 * 128 * 32;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&tbar)));
    if (sfa == 0xFFFFFFFFu) return;  // never
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  fill_scales(tm, 480, sfa, sfb);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&tbar)),
                 "r"(10 * 128 * 32 + 5 * NT * 32));
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(A), "l"((uint64_t)&ma), "r"(sa(&tbar)), "r"(0), "r"(0), "r"(0) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(B), "l"((uint64_t)&mb), "r"(sa(&tbar)), "r"(0), "r"(0), "r"(0) : "memory");
    wait0(sa(&tbar), 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int side = 0; side < 2; ++side)
      for (int ks = 0; ks < 5; ++ks)
        mma_mxf4(tm + side * 240, desc32(A + (side * 5 + ks) * 128 * 32), desc32(B + ks * NT * 32),
                 idesc_mxf4(128, NT), tm + 480, tm + 496, ks > 0);
    commit(sa(&bar));
  }
  __syncwarp();
  wait0(sa(&bar), 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = threadIdx.x;
  for (int side = 0; side < 2; ++side)
    for (int c = 0; c < NT; c += 8) {
      uint32_t v[8];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                     "=r"(v[7])
                   : "r"(tm + ((uint32_t)(warp * 32) << 16) + side * 240 + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      for (int i = 0; i < 8; ++i) out[(side * 128 + row) * NT + c + i] = __uint_as_float(v[i]);
    }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

static PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  void* ptr = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)ptr;
}

static int map3(CUtensorMap* m, void* base, int rows, int rowb, int box_rows) {
  cuuint64_t dims[3] = {32, (cuuint64_t)rows, (cuuint64_t)(rowb / 32)};
  cuuint64_t strides[2] = {(cuuint64_t)rowb, 32};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, (cuuint32_t)(rowb / 32)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = encoder()(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, base, dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                         CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r) printf("  cuTensorMapEncodeTiled failed %d\n", (int)r);
  return (int)r;
}

template <int NT>
int check_tma(uint32_t sfa = 0x7F7F7F7Fu, uint32_t sfb = 0x7F7F7F7Fu, bool denorm = false) {
  const int K = 320;  // 295 real + bias at 295 + zero pad
  static uint8_t a[128][K], b[NT][K];
  srand(11);
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < K; ++k) a[r][k] = (k < 295) ? (rand() % 8 == 0) : (k == 295);
  for (int r = 0; r < NT; ++r)
    for (int k = 0; k < K; ++k) b[r][k] = (k < 295) ? (rand() % 40 == 0) : (k == 295 && r % 7 == 0);
  // A rows: [A_up (160 B) | A_lo (160 B)], A_lo = complement of A_up on real columns
  static uint8_t ha[128 * 320], hb[NT * 160];
  memset(ha, 0, sizeof(ha));
  memset(hb, 0, sizeof(hb));
  for (int r = 0; r < 128; ++r)
    for (int k = 0; k < K; ++k) {
      const int up = a[r][k], lo = k < 295 ? !a[r][k] : (k == 295);
      ha[r * 320 + k / 2] |= (uint8_t)(up ? (k & 1 ? 0x20 : 0x2) : 0);
      ha[r * 320 + 160 + k / 2] |= (uint8_t)(lo ? (k & 1 ? 0x20 : 0x2) : 0);
    }
  for (int r = 0; r < NT; ++r)
    for (int k = 0; k < K; ++k) hb[r * 160 + k / 2] |= (uint8_t)(b[r][k] ? (k & 1 ? 0x20 : 0x2) : 0);
  uint8_t *da, *db;
  float* dout;
  cudaMalloc(&da, sizeof(ha));
  cudaMalloc(&db, sizeof(hb));
  cudaMalloc(&dout, 2 * 128 * NT * 4);
  cudaMemcpy(da, ha, sizeof(ha), cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb, sizeof(hb), cudaMemcpyHostToDevice);
  CUtensorMap ma, mb;
  if (map3(&ma, da, 128, 320, 128) || map3(&mb, db, NT, 160, NT)) return 1;
  const int smem = 10 * 128 * 32 + 5 * NT * 32 + 1024;
  cudaFuncSetAttribute(check_tma_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  check_tma_kernel<NT><<<1, 128, smem>>>(ma, mb, dout, sfa, sfb);
  cudaError_t e = cudaDeviceSynchronize();
  static float out[2 * 128 * NT];
  cudaMemcpy(out, dout, sizeof(out), cudaMemcpyDeviceToHost);
  int bad = 0, zeros = 0;
  for (int side = 0; side < 2; ++side)
    for (int r = 0; r < 128; ++r)
      for (int n = 0; n < NT; ++n) {
        int s = 0;
        for (int k = 0; k < K; ++k) {
          const int av = side == 0 ? a[r][k] : (k < 295 ? !a[r][k] : (k == 295));
          s += av * b[n][k];
        }
        zeros += s == 0;
        uint32_t bits;
        memcpy(&bits, &out[(side * 128 + r) * NT + n], 4);
        if (denorm ? bits != (uint32_t)s : out[(side * 128 + r) * NT + n] != (float)s) {
          if (bad < 5) printf("  tma mismatch side=%d r=%d n=%d got %f want %d\n", side, r, n,
                              out[(side * 128 + r) * NT + n], s);
          ++bad;
        }
      }
  printf("check TMA-SW32 N=%d scales %08x/%08x%s: %s, %d mismatches of %d (exact zeros %d)\n", NT, sfa, sfb,
         denorm ? " (denormal bits == count)" : "", cudaGetErrorString(e), bad, 2 * 128 * NT, zeros);
  return bad;
}

template <int N, bool SW32 = false>
void rate(int sms) {
  const int iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 4 * 8192 + 4 * 8192 + 1024;
  cudaFuncSetAttribute(rate_kernel<N, SW32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  rate_kernel<N, SW32><<<sms, 128, smem>>>(100, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  rate_kernel<N, SW32><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)iters * 4;
  const double ops = 2.0 * 128 * N * 64 * mmas * sms;
  printf("rate mxf4 %s M=128 N=%d K=64: %.1f cycles/MMA (ideal %d at 2x int8), %.0f TOPS, %s\n", SW32 ? "SW32" : "SW128", N, c / mmas,
         128 * N * 64 / 16384, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

// ---- 4. CTA-pair issue rate: leader issues M=256 N x K=64 (cta_group::2) MMAs,
// `per_commit` per commit (multicast to both CTAs' barrier), two accumulators.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
pair_rate_kernel(int iters, int per_commit, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (sa(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = slot;
  fill_scales(tm, 480);
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0 && rank == 0) {
    const uint32_t A = sa(base), B = A + 5 * 4096;
    long long t0 = clock64();
    int n = 0;
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = tm + (uint32_t)((i & 1) * 240);
      for (int k = 0; k < 5; ++k) {
        const uint64_t a = desc32(A + k * 4096), b = desc32(B + k * 4096);
        asm volatile(
            "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
            "@e tcgen05.mma.cta_group::2.kind::mxf4.block_scale.scale_vec::2X [%0], %1, %2, %3, [%5], [%6], p;\n}" ::"r"(d),
            "l"(a), "l"(b), "r"(idesc_mxf4(256, N)), "r"(k), "r"(tm + 480), "r"(tm + 496));
        if (++n == per_commit) {
          n = 0;
          asm volatile("{.reg .pred e; .reg .b16 m; mov.b16 m, 3; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;}" ::"r"(sa(&bar)));
        }
      }
    }
    asm volatile("{.reg .pred e; .reg .b16 m; mov.b16 m, 3; elect.sync _|e, 0xffffffff; @e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;}" ::"r"(sa(&bar)));
    // wait until the barrier has seen every commit: poll the phase count via try_wait on parity
    long long t1;
    {
      // the last commit completes after all MMAs; spin on any phase flip after it
      uint32_t ok = 0;
      const int commits = (iters * 5) / per_commit + 1;
      const uint32_t par = (commits - 1) & 1;
      while (!ok)
        asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}"
                     : "=r"(ok) : "r"(sa(&bar)), "r"(par));
      t1 = clock64();
    }
    if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N>
void pair_rate(int sms, int per_commit) {
  const int iters = 20000;
  unsigned long long* d;
  cudaMalloc(&d, sms * 8);
  const int smem = 10 * 4096 + 1024;
  cudaFuncSetAttribute(pair_rate_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  pair_rate_kernel<N><<<sms, 128, smem>>>(100, per_commit, d);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  pair_rate_kernel<N><<<sms, 128, smem>>>(iters, per_commit, d);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double mmas = (double)iters * 5;
  const double ops = 2.0 * 256 * N * 64 * mmas * (sms / 2);
  printf("pair mxf4 M=256 N=%d K=64 commit/%d: %.1f cycles/MMA (ideal %d), %.0f TOPS, %s\n", N, per_commit,
         c / mmas, 128 * N * 64 / 16384, ops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int bad = check<256>() + check<240>() + check_tma<240>();
  // D = count * 2^-127 * 2^-22 = count * 2^-149: fp32 denormal whose bits are the count
  check_tma<240>(0x00000000u, 0x69696969u, true);
  rate<256>(sms);
  rate<240>(sms);
  rate<224>(sms);
  rate<240, true>(sms);
  rate<256, true>(sms);
  pair_rate<240>(sms, 5);
  pair_rate<224>(sms, 5);
  pair_rate<208>(sms, 5);
  pair_rate<192>(sms, 5);
  pair_rate<176>(sms, 5);
  pair_rate<160>(sms, 5);
  pair_rate<128>(sms, 5);
  pair_rate<112>(sms, 5);
  pair_rate<96>(sms, 5);
  pair_rate<144>(sms, 5);
  return bad ? 1 : 0;
}
