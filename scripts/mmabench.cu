// mmabench.cu -- tcgen05.mma issue-to-completion latency on B200 (tuning tool,
// not part of the product).  One CTA per SM; warp 1 issues G groups of
// `nmma` MMAs (kind::f16, M=128, N=64 or 128, K=16, SS operands) each followed by a
// commit to an mbarrier and a wait; measures ns per group with %globaltimer.
// Warps 2..9 optionally hammer shared memory (LDS/STS) to emulate an epilogue.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mmabench mmabench.cu
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

__global__ void __launch_bounds__(320, 1) mma_lat(uint64_t* out, int groups, int nmma, int N, int hammer, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    stop = 0;
  }
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24);
  if (warp == 1) {
    const uint64_t da = desc(su32(sm), 256, 6), db = desc(su32(sm + 32768), 256, 6);
    uint64_t t_sum = 0;
    uint32_t phase = 0;
    for (int g = 0; g < groups; ++g) {
      const uint64_t t0 = gt();
      if (mode == 1) {   // MMAs only timed: commit after the second timestamp
        if (elect())
          for (int j = 0; j < nmma; ++j) {
            const uint32_t d = tbase + (j % 4) * N;
            asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                         ::"r"(d), "l"(da + j * 256), "l"(db + j * 128), "r"(idesc), "r"(0u));
          }
        __syncwarp();
        const uint64_t tm = gt();
        if (elect()) asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
        __syncwarp();
        uint32_t ok = 0;
        while (!ok)
          asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                       : "=r"(ok) : "r"(su32(&bar)), "r"(phase));
        phase ^= 1;
        const uint64_t t2 = gt();
        if (g >= 10) t_sum += (t2 - t0);
        if (lane == 0 && blockIdx.x == 0 && g == groups - 1) { out[0] = tm - t0; out[1] = t2 - tm; }
        continue;
      }
      if (elect()) {
        for (int j = 0; j < nmma; ++j) {
          const uint32_t d = tbase + (j % 4) * N;
          asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
                       ::"r"(d), "l"(da + j * 256), "l"(db + j * 128), "r"(idesc), "r"(0u));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
      }
      __syncwarp();
      const uint64_t t1 = gt();
      uint32_t ok = 0;
      while (!ok)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                     : "=r"(ok) : "r"(su32(&bar)), "r"(phase));
      phase ^= 1;
      const uint64_t t2 = gt();
      if (g >= 10) t_sum += (t2 - t0);
      if (lane == 0 && blockIdx.x == 0 && g == groups - 1) { out[0] = t1 - t0; out[1] = t2 - t1; }
    }
    if (lane == 0) atomicAdd((unsigned long long*)&out[2], t_sum / (groups - 10));
    if (lane == 0) stop = 1;
  } else if (warp >= 2 && hammer) {
    // smem traffic: 16-B loads and stores over a 64 KB region, like an epilogue
    uint4* p = reinterpret_cast<uint4*>(sm + 65536);
    uint32_t acc = 0;
    int i = (warp - 2) * 32 + lane;
    while (!stop) {
      for (int k = 0; k < 64; ++k) {
        uint4 v = p[(i + k * 256) & 4095];
        acc += v.x;
        p[(i + k * 256 + 17) & 4095] = make_uint4(acc, v.y, v.z, v.w);
      }
    }
    if (acc == 0xdeadbeef) out[3] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 64);
  cudaFuncSetAttribute(mma_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  for (int mode : {0, 1})
  for (int hammer : {0})
    for (int N : {64, 128})
      for (int nmma : {1, 4, 8, 12}) {
        cudaMemset(d, 0, 64);
        mma_lat<<<148, 320, 160 * 1024>>>(d, 200, nmma, N, hammer, mode);
        cudaError_t e = cudaDeviceSynchronize();
        uint64_t h[4];
        cudaMemcpy(h, d, 32, cudaMemcpyDeviceToHost);
        printf("mode=%d hammer=%d N=%3d nmma=%2d: t1 %5llu ns, t2 %5llu ns, mean group %6.1f ns %s\n", mode, hammer, N, nmma,
               (unsigned long long)h[0], (unsigned long long)h[1], h[2] / 148.0,
               e == cudaSuccess ? "" : cudaGetErrorString(e));
      }
  return 0;
}
