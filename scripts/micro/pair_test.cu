// Micro-test: a CTA pair (cluster of 2) computing D[256 x 256] = A[256 x 64] . B[256 x 64]^T
// with ONE tcgen05.mma.cta_group::2 chain issued by the leader CTA.  Each CTA
// holds 128 rows of A (its own M half) and, bmode 0, 128 rows of B (its N
// half) or, bmode 1, all 256 rows of B; alloc mode 0: both CTAs execute
// tcgen05.alloc.cta_group::2, 1: the leader only.  Bounded waits (no trap).
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
__device__ __forceinline__ int swz(int row, int k) { return row * 64 + ((((k >> 3) ^ (row & 7))) << 3) + (k & 7); }
__device__ __forceinline__ uint64_t gtime() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

__global__ void __cluster_dims__(2, 1, 1) k_pair(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D,
                                                int* status, int amode, int bmode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __nv_bfloat16* sa = reinterpret_cast<__nv_bfloat16*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __nv_bfloat16* sb = sa + 128 * 64;
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    sa[swz(r, k)] = A[(rank * 128 + r) * 64 + k];
  }
  const int brows = bmode == 0 ? 128 : 256;
  const int b0 = bmode == 0 ? rank * 128 : 0;
  for (int i = threadIdx.x; i < brows * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64;
    sb[swz(r, k)] = B[(b0 + r) * 64 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tbase = 0xffffffffu;
  __syncthreads();
  if (warp == 0 && (amode == 0 || rank == 0)) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(s_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tb = tbase;
  if (amode == 1 && rank == 1) {
    // read the leader's allocated address through DSMEM
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(s_u32(&tbase)));
    asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(tb) : "r"(remote) : "memory");
  }
  if (threadIdx.x == 0) status[rank * 4 + 0] = (int)tb;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((256u >> 4) << 24);
  const uint64_t da = desc(s_u32(sa), 1024, 2), db = desc(s_u32(sb), 1024, 2);
  if (rank == 0 && threadIdx.x == 0) {
    for (int kk = 0; kk < 4; ++kk)
      asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
                   ::"r"(tb), "l"(da + kk * 2), "l"(db + kk * 2), "r"(idesc), "r"(kk) : "memory");
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(s_u32(&bar)), "h"((uint16_t)3) : "memory");
  }
  {
    uint32_t ok = 0;
    const uint64_t t0 = gtime();
    while (!ok) {
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(s_u32(&bar)) : "memory");
      if (!ok && gtime() - t0 > 500000000ull) break;
    }
    if (threadIdx.x == 0) status[rank * 4 + 1] = (int)ok;
    if (!ok) return;
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    const int row = warp * 32 + (threadIdx.x & 31);
    for (int c = 0; c < 256; c += 16) {
      uint32_t v[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                     "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                   : "r"(tb + ((uint32_t)(warp * 32) << 16) + c));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int i = 0; i < 16; ++i) D[(rank * 128 + row) * 256 + c + i] = __uint_as_float(v[i]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0 && (amode == 0 || rank == 0))
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tb) : "memory");
}

int main() {
  const int nA = 256 * 64;
  std::vector<__nv_bfloat16> hA(nA), hB(nA);
  for (int i = 0; i < nA; ++i) {
    hA[i] = __float2bfloat16((float)((i * 37 % 17) - 8) / 8.f);
    hB[i] = __float2bfloat16((float)((i * 53 % 13) - 6) / 4.f);
  }
  std::vector<float> ref(256 * 256);
  for (int i = 0; i < 256; ++i)
    for (int j = 0; j < 256; ++j) {
      double s = 0;
      for (int k = 0; k < 64; ++k) s += (double)__bfloat162float(hA[i * 64 + k]) * __bfloat162float(hB[j * 64 + k]);
      ref[i * 256 + j] = (float)s;
    }
  __nv_bfloat16 *A, *B;
  float* D;
  int* st;
  cudaMalloc(&A, nA * 2); cudaMalloc(&B, nA * 2); cudaMalloc(&D, 256 * 256 * 4); cudaMalloc(&st, 64);
  cudaMemcpy(A, hA.data(), nA * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB.data(), nA * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int amode = 0; amode < 2; ++amode)
    for (int bmode = 0; bmode < 2; ++bmode) {
      cudaMemset(D, 0, 256 * 256 * 4);
      cudaMemset(st, 0xff, 64);
      k_pair<<<2, 128, 100 * 1024>>>(A, B, D, st, amode, bmode);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("amode %d bmode %d: %s\n", amode, bmode, cudaGetErrorString(e)); return 1; }
      std::vector<float> h(256 * 256);
      int hs[16];
      cudaMemcpy(h.data(), D, 256 * 256 * 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(hs, st, 64, cudaMemcpyDeviceToHost);
      double err = 0, err_top = 0, err_bot = 0;
      for (int i = 0; i < 256 * 256; ++i) {
        const double d = fabs(h[i] - ref[i]);
        err = fmax(err, d);
        if (i < 128 * 256) err_top = fmax(err_top, d); else err_bot = fmax(err_bot, d);
      }
      printf("alloc %s, B %s: tmem %d/%d done %d/%d  max err %g (rows 0-127 %g, 128-255 %g)  D[5][7]=%g ref %g D[200][201]=%g ref %g\n",
             amode ? "leader-only" : "both", bmode ? "full" : "split", hs[0], hs[4], hs[1], hs[5], err, err_top, err_bot,
             h[5 * 256 + 7], ref[5 * 256 + 7], h[200 * 256 + 201], ref[200 * 256 + 201]);
    }
  return 0;
}
