// mmabench2.cu -- do two MMA-issuing warps overlap their per-group latency?
// (tuning tool, not part of the product).  W issuer warps (1 or 2) each issue G
// groups of 4 tcgen05.mma (M=128, N=64, K=16, SS) + commit to their own
// mbarrier + wait, into disjoint TMEM columns; reports ns per group per warp and
// aggregate groups/us.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }
__device__ __forceinline__ uint64_t desc(uint32_t a, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((a >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)layout << 61);
}
__device__ __forceinline__ bool elect() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}" : "=r"(p));
  return p;
}

__global__ void __launch_bounds__(128, 1) k2(uint64_t* out, int groups, int nwarps) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (8u << 17) | (8u << 24);
  if (warp >= 1 && warp <= nwarps) {
    const int w = warp - 1;
    const uint64_t da = desc(su32(sm), 256, 6), db = desc(su32(sm + 32768), 256, 6);
    uint32_t phase = 0;
    const uint64_t t0 = gt();
    for (int g = 0; g < groups; ++g) {
      if (elect()) {
        for (int j = 0; j < 4; ++j)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tbase + w * 256 + j * 64), "l"(da + j * 256), "l"(db + j * 128), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[w])));
      }
      __syncwarp();
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                     : "=r"(ok) : "r"(su32(&bar[w])), "r"(phase));
      phase ^= 1;
    }
    if (lane == 0) atomicAdd((unsigned long long*)&out[w], (gt() - t0) / groups);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  for (int nw : {1, 2}) {
    cudaMemset(d, 0, 32);
    k2<<<148, 128, 96 * 1024>>>(d, 400, nw);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("issuer warps=%d: ns/group warp0 %.1f warp1 %.1f -> groups/us per SM %.2f %s\n", nw, h[0] / 148.0,
           h[1] / 148.0, nw * 1000.0 / (h[0] / 148.0), e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
