// pingpong.cu -- mbarrier hand-off latency between two warps of one CTA on
// B200 (tuning tool, not part of the product): warp 0 arrives on bar[0], warp
// 1 waits then arrives on bar[1], warp 0 waits; 2*R hand-offs.  Waiting with
// mbarrier.try_wait (may suspend) vs spinning on mbarrier.test_wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pingpong pingpong.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t gt() { uint64_t t; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)); return t; }

template <bool kSpin>
__device__ __forceinline__ void wait(uint32_t bar, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    if (kSpin)
      asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                   : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    else
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0,1,0,p;\n}"
                   : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  }
}

template <bool kSpin>
__global__ void pp(uint64_t* out, int R) {
  __shared__ __align__(8) uint64_t bar[2];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[1])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  uint64_t t0 = gt();
  for (int r = 0; r < R; ++r) {
    const uint32_t ph = r & 1;
    if (warp == 0) {
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[0])) : "memory");
      wait<kSpin>(su32(&bar[1]), ph);
    } else if (warp == 1) {
      wait<kSpin>(su32(&bar[0]), ph);
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&bar[1])) : "memory");
    }
  }
  if (threadIdx.x == 0) atomicAdd((unsigned long long*)out, (gt() - t0) / (2 * R));
}

int main() {
  uint64_t* d;
  cudaMalloc(&d, 8);
  for (int spin : {0, 1}) {
    cudaMemset(d, 0, 8);
    if (spin) pp<true><<<148, 64>>>(d, 2000); else pp<false><<<148, 64>>>(d, 2000);
    cudaDeviceSynchronize();
    uint64_t h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%s: %.1f ns per hand-off (mean over 148 CTAs)\n", spin ? "test_wait spin" : "try_wait", h / 148.0);
  }
  return 0;
}
