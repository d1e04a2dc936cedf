// Micro-benchmark: tcgen05.ld / tcgen05.st throughput per SM (8 warps, two
// per lane quarter, 32x32b.x16 / .x32 shapes), and tcgen05.mma rate with the
// M-side operand in TMEM ([tmem]) vs in shared memory (descriptor), M = N = 128,
// kind::f16.  One CTA per SM over the whole GPU; cycles by clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_bw scripts/micro/tmem_bw.cu
#include <cstdio>
#include <cstdint>

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

__global__ void k_ld(unsigned long long* out, int iters, int wide) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t acc = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    if (wide) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(ta + (i & 1) * 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 32; ++q) acc += v[q];
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(ta + (i & 3) * 16));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      for (int q = 0; q < 16; ++q) acc += v[q];
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
    out[2 * blockIdx.x + 1] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

__global__ void k_st(unsigned long long* out, int iters) {
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t ta = tbase + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  __syncthreads();
  const long long t0 = clock64();
  uint32_t x = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 1664525u + 1013904223u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
        ::"r"(ta + (i & 3) * 16), "r"(x) : "memory");
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase) : "memory");
}

// MMA issue rate: n_mma MMAs of M = N = 128, K = 16, accumulating into one
// D, the M operand from TMEM (ts = 1) or shared memory (ts = 0); one commit.
__global__ void k_mma(unsigned long long* out, int n_mma, int ts) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* s = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 2 * 128 * 64; i += blockDim.x) reinterpret_cast<uint16_t*>(s)[i] = 0x3f80;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(s_u32(&tbase)) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tbase;
  const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
  const uint64_t da = desc(s_u32(s), 1024, 2), db = desc(s_u32(s + 128 * 128), 1024, 2);
  const uint32_t d = tb, ta = tb + 256;
  long long t0 = 0, t1 = 0;
  if (warp == 0 && (threadIdx.x & 31) == 0) {
    for (int kk = 0; kk < 4; ++kk)
      asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(ta + kk * 8), "l"(da + kk * 2) : "memory");
    t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int kk = i & 3;
      if (ts)
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, 1;"
                     ::"r"(d), "r"(ta + kk * 8), "l"(db + kk * 2), "r"(idesc) : "memory");
      else
        asm volatile("tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;"
                     ::"r"(d), "l"(da + kk * 2), "l"(db + kk * 2), "r"(idesc) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_u32(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}"
                   : "=r"(ok) : "r"(s_u32(&bar)) : "memory");
    t1 = clock64();
    out[2 * blockIdx.x] = (unsigned long long)(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb) : "memory");
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* out;
  cudaMalloc(&out, sms * 16);
  unsigned long long h[2];
  const int iters = 4096;
  for (int wide = 0; wide < 2; ++wide) {
    k_ld<<<sms, 256>>>(out, iters, wide);
    k_ld<<<sms, 256>>>(out, iters, wide);
    cudaDeviceSynchronize();
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    const double bytes = 8.0 * iters * 32 * (wide ? 32 : 16) * 4;
    printf("tcgen05.ld 32x32b.x%d, 8 warps: %llu cycles, %.1f B/cycle per SM\n", wide ? 32 : 16, h[0], bytes / h[0]);
  }
  k_st<<<sms, 256>>>(out, iters);
  k_st<<<sms, 256>>>(out, iters);
  cudaDeviceSynchronize();
  cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
  printf("tcgen05.st 32x32b.x16, 8 warps: %llu cycles, %.1f B/cycle per SM\n", h[0], 8.0 * iters * 32 * 16 * 4 / h[0]);
  cudaFuncSetAttribute(k_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  for (int ts = 0; ts < 2; ++ts) {
    const int n = 4096;
    k_mma<<<sms, 128, 80 * 1024>>>(out, n, ts);
    k_mma<<<sms, 128, 80 * 1024>>>(out, n, ts);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mma: %s\n", cudaGetErrorString(e)); return 1; }
    cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
    printf("tcgen05.mma M128 N128 K16 %s: %.1f cycles per MMA\n", ts ? "[tmem] A" : "smem A", (double)h[0] / n);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
