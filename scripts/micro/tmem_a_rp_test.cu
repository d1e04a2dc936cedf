// Micro-test 2: A operand in TMEM copied by tcgen05.cp.128x256b from the
// switch's pre-swizzled per-term slices ([128, rp] bf16, K-major, swizzle
// 32B / 64B / 128B for rp = 16 / 32 / 64), K = 64 total = 64/rp slices.
// Compares D = A B^T (A from TMEM) against the SS form and a host reference;
// D3: A written to TMEM by tcgen05.st from registers in natural K order (column
// c of a K-step = elements 2c (low half), 2c + 1), as the switch's TMEM fold does.
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
__device__ __forceinline__ int swz_off(int row, int k, int rp) {
  const int rb = 2 * rp;
  const int f = (row * rb / 128) & (rb / 16 - 1);
  return row * rp + (((k >> 3) ^ f) << 3) + (k & 7);
}

template <int RP>
__global__ void k_test(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D1, float* D2, float* D3) {
  extern __shared__ __align__(1024) uint8_t sm[];
  constexpr int NS = 64 / RP;                  // slices (terms)
  constexpr int TERM = 128 * RP;               // elements per slice
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sb = sa + NS * TERM;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64, j = k / RP, kk = k % RP;
    sa[j * TERM + swz_off(r, kk, RP)] = A[i];
    sb[j * TERM + swz_off(r, kk, RP)] = B[i];
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
  constexpr uint32_t LAY = RP == 16 ? 6 : RP == 32 ? 4 : 2;
  const uint64_t d0 = desc(0, 8 * RP * 2, LAY);
  const uint64_t da = d0 + (s_u32(sa) >> 4), db = d0 + (s_u32(sb) >> 4);
  const uint64_t term = (TERM * 2) >> 4;
  const uint32_t d1 = tb, d2 = tb + 128, ta = tb + 256, tst = tb + 288, d3 = tb + 384;
  if (warp < 4) {
    const int row = warp * 32 + (threadIdx.x & 31);
    const uint16_t* a16 = reinterpret_cast<const uint16_t*>(A);
    for (int n = 0; n < 4; ++n) {
      uint32_t w[8];
      for (int q = 0; q < 8; ++q)
        w[q] = (uint32_t)a16[row * 64 + 16 * n + 2 * q] | ((uint32_t)a16[row * 64 + 16 * n + 2 * q + 1] << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   ::"r"(tst + ((uint32_t)(warp * 32) << 16) + n * 8), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]),
                     "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]) : "memory");
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    for (int n = 0; n < 4; ++n) {
      const int j = n / (RP / 16), kk = n % (RP / 16);
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                   ::"r"(d3), "r"(tst + n * 8), "l"(db + j * term + kk * 2), "r"(idesc), "r"(n) : "memory");
    }
    int n = 0;
    for (int j = 0; j < NS; ++j)
      for (int kk = 0; kk < RP / 16; ++kk, ++n)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                     ::"r"(d1), "l"(da + j * term + kk * 2), "l"(db + j * term + kk * 2), "r"(idesc), "r"(n) : "memory");
    n = 0;
    for (int j = 0; j < NS; ++j)
      for (int kk = 0; kk < RP / 16; ++kk, ++n)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta + n * 8), "l"(da + j * term + kk * 2) : "memory");
    n = 0;
    for (int j = 0; j < NS; ++j)
      for (int kk = 0; kk < RP / 16; ++kk, ++n)
        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
                     ::"r"(d2), "r"(ta + n * 8), "l"(db + j * term + kk * 2), "r"(idesc), "r"(n) : "memory");
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
      uint32_t v[16], w[16], x[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(d1 + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
                     "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
                   : "r"(d2 + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
                     "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
                   : "r"(d3 + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) {
        D1[row * 128 + c + i] = __uint_as_float(v[i]);
        D2[row * 128 + c + i] = __uint_as_float(w[i]);
        D3[row * 128 + c + i] = __uint_as_float(x[i]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

template <int RP>
int run(__nv_bfloat16* A, __nv_bfloat16* B, float* D1, float* D2, float* D3, const std::vector<float>& ref) {
  cudaFuncSetAttribute(k_test<RP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  k_test<RP><<<1, 128, 64 * 1024>>>(A, B, D1, D2, D3);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("rp %d: %s\n", RP, cudaGetErrorString(e)); return 1; }
  std::vector<float> h1(128 * 128), h2(128 * 128), h3(128 * 128);
  cudaMemcpy(h1.data(), D1, 128 * 128 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), D2, 128 * 128 * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h3.data(), D3, 128 * 128 * 4, cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, e3 = 0;
  for (int i = 0; i < 128 * 128; ++i) {
    e1 = fmax(e1, fabs(h1[i] - ref[i])); e2 = fmax(e2, fabs(h2[i] - ref[i])); e3 = fmax(e3, fabs(h3[i] - ref[i]));
  }
  printf("rp %d: SS max err %g, A-in-TMEM (cp) max err %g, A-in-TMEM (st, natural order) max err %g\n", RP, e1, e2, e3);
  return 0;
}

int main() {
  const int n = 128 * 64;
  std::vector<__nv_bfloat16> hA(n), hB(n);
  for (int i = 0; i < n; ++i) {
    hA[i] = __float2bfloat16((float)((i * 37 % 17) - 8) / 8.f);
    hB[i] = __float2bfloat16((float)((i * 53 % 13) - 6) / 4.f);
  }
  std::vector<float> ref(128 * 128);
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += (double)__bfloat162float(hA[i * 64 + k]) * __bfloat162float(hB[j * 64 + k]);
      ref[i * 128 + j] = (float)s;
    }
  __nv_bfloat16 *A, *B;
  float *D1, *D2, *D3;
  cudaMalloc(&A, n * 2); cudaMalloc(&B, n * 2);
  cudaMalloc(&D1, 128 * 128 * 4); cudaMalloc(&D2, 128 * 128 * 4); cudaMalloc(&D3, 128 * 128 * 4);
  cudaMemcpy(A, hA.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), n * 2, cudaMemcpyHostToDevice);
  return run<16>(A, B, D1, D2, D3, ref) | run<32>(A, B, D1, D2, D3, ref) | run<64>(A, B, D1, D2, D3, ref);
}
