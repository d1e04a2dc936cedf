// Micro-test: tcgen05.mma with the A operand in TMEM (copied there by
// tcgen05.cp from the same swizzled K-major smem image the SS form reads)
// gives the same D as the SS form.  One CTA, M = N = 128, K = 64 (SW128).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_a_test scripts/micro/tmem_a_test.cu
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
#include <vector>
#include <cmath>

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
// element (row, k) of a [rows, 64] bf16 K-major 128B-swizzled image
__device__ __forceinline__ int swz(int row, int k) { return row * 64 + ((((k >> 3) ^ (row & 7))) << 3) + (k & 7); }

__global__ void k_test(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D1, float* D2, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sb = sa + 128 * 64;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    sa[swz(r, k)] = A[i];
    sb[swz(r, k)] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = desc(s_u32(sa), 1024, 2), db = desc(s_u32(sb), 1024, 2);
  const uint32_t d1 = tb, d2 = tb + 128, ta = tb + 256;   // D1 128 cols, D2 128 cols, A 32 cols
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    for (int kk = 0; kk < 4; ++kk) {
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                   ::"r"(d1), "l"(da + kk * 2), "l"(db + kk * 2), "r"(idesc), "r"(kk) : "memory");
    }
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t col = mode == 0 ? kk * 8 : kk * 4;
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta + col), "l"(da + kk * 2) : "memory");
    }
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t col = mode == 0 ? kk * 8 : kk * 4;
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                   ::"r"(d2), "r"(ta + col), "l"(db + kk * 2), "r"(idesc), "r"(kk) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(s_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < 128; c += 16) {
      uint32_t v[16], w[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(d1 + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                     "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                   : "r"(d2 + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) {
        D1[row * 128 + c + i] = __uint_as_float(v[i]);
        D2[row * 128 + c + i] = __uint_as_float(w[i]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

int main() {
  const int n = 128 * 64;
  std::vector<__nv_bfloat16> hA(n), hB(n);
  for (int i = 0; i < n; ++i) {
    hA[i] = __float2bfloat16((float)((i * 37 % 17) - 8) / 8.f);
    hB[i] = __float2bfloat16((float)((i * 53 % 13) - 6) / 4.f);
  }
  // host reference D[i][j] = sum_k A[i][k] B[j][k]
  std::vector<float> ref(128 * 128);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += (double)__bfloat162float(hA[i * 64 + k]) * __bfloat162float(hB[j * 64 + k]);
      ref[i * 128 + j] = (float)s;
    }
  __nv_bfloat16 *A, *B;
  float *D1, *D2;
  cudaMalloc(&A, n * 2); cudaMalloc(&B, n * 2);
  cudaMalloc(&D1, 128 * 128 * 4); cudaMalloc(&D2, 128 * 128 * 4);
  cudaMemcpy(A, hA.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), n * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_test, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(D1, 0, 128 * 128 * 4); cudaMemset(D2, 0, 128 * 128 * 4);
    k_test<<<1, 128, 64 * 1024>>>(A, B, D1, D2, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: %s\n", mode, cudaGetErrorString(e)); return 1; }
    std::vector<float> h1(128 * 128), h2(128 * 128);
    cudaMemcpy(h1.data(), D1, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(h2.data(), D2, 128 * 128 * 4, cudaMemcpyDeviceToHost);
    double e1 = 0, e2 = 0;
    for (int i = 0; i < 128 * 128; ++i) { e1 = fmax(e1, fabs(h1[i] - ref[i])); e2 = fmax(e2, fabs(h2[i] - ref[i])); }
    printf("mode %d (A cols per K-step %d): SS max err %g, A-in-TMEM max err %g, sample ref %g ss %g tmem %g\n",
           mode, mode == 0 ? 8 : 4, e1, e2, ref[5 * 128 + 7], h1[5 * 128 + 7], h2[5 * 128 + 7]);
  }
  return 0;
}
