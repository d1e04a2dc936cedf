// mmabench3.cu -- tcgen05.mma issue / throughput microbenchmark (tuning tool,
// not part of the product).  One CTA per SM, one issuing warp.  For each
// variant (MMAs per group, N) it issues G groups back to back into rotating
// TMEM buffers, one commit per group, and waits only when the buffer about to
// be reused has not drained (depth D groups in flight).  Reports ns per group
// and ns per MMA, plus the cycles the issuing thread spends inside the MMA
// instructions themselves.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mmabench3 scripts/mmabench3.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

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
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                 : "=r"(ok) : "r"(bar), "r"(ph));
}

// nmma MMAs of width n per group; depth groups in flight (buffers of n*nmma columns)
__global__ void __launch_bounds__(64, 1) k(uint64_t* out, int groups, int nmma, int n, int depth) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | (8u << 24);
    const uint64_t da = desc(su32(sm), 256, 6), db = desc(su32(sm + 32768), 256, 6);
    const uint32_t bufcols = (uint32_t)(n * nmma);
    uint64_t issue_cycles = 0;
    uint32_t phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const uint64_t t0 = gt();
    for (int g = 0; g < groups; ++g) {
      const int b = g % depth;
      if (g >= depth) { wait(su32(&bar[b]), phase[b]); phase[b] ^= 1; }
      asm volatile("tcgen05.fence::after_thread_sync;");
      if (elect()) {
        const uint64_t c0 = clock64();
        for (int j = 0; j < nmma; ++j)
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                       ::"r"(tbase + b * bufcols + j * n), "l"(da + j * 256), "l"(db + j * 128), "r"(idesc), "r"(0u));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[b])));
        issue_cycles += clock64() - c0;
      }
      __syncwarp();
    }
    for (int b = 0; b < depth && b < groups; ++b) wait(su32(&bar[b]), phase[b]);
    const uint64_t t1 = gt();
    if (threadIdx.x == 0) {
      atomicAdd((unsigned long long*)&out[0], (t1 - t0));
      atomicAdd((unsigned long long*)&out[1], issue_cycles);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  struct V { int nmma, n, depth; } vs[] = {{1, 64, 2}, {2, 64, 2}, {4, 64, 2}, {8, 64, 1}, {4, 64, 1}, {2, 128, 2},
                                            {4, 128, 1}, {1, 128, 4}, {1, 256, 2}, {2, 256, 1}, {4, 64, 2}};
  const int G = 2000;
  for (const V& v : vs) {
    cudaMemset(d, 0, 16);
    k<<<148, 64, 96 * 1024>>>(d, G, v.nmma, v.n, v.depth);
    cudaError_t e = cudaDeviceSynchronize();
    uint64_t h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    const double ns_group = (double)h[0] / 148 / G;
    printf("mma/group %d  N %3d  depth %d : %7.1f ns/group  %6.1f ns/MMA  issue %6.1f cyc/group  %s\n", v.nmma, v.n,
           v.depth, ns_group, ns_group / v.nmma, (double)h[1] / 148 / G, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
