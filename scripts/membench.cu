// membench.cu -- B200 memory-pattern ceilings for the switch/GEMV design
// (tuning tool, not part of the product).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   copy       : out[i] = in[i]                     (cudaMemcpy-like, 2 streams)
//   rmw        : a[i] = a[i] + 0 in place           (read + write same lines)
//   read       : sum(a)
//   rmw_rows   : in-place RMW where each warp owns 128-B segments of R rows (strided)
// Each with U independent 16-B loads in flight per thread.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int U>
__global__ void copy_k(const uint4* __restrict__ in, uint4* __restrict__ out, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) v[u] = __ldcs(in + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) __stcs(out + i + u * blockDim.x, v[u]);
  }
}

template <int U>
__global__ void rmw_k(uint4* __restrict__ a, size_t n, uint32_t add) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) v[u] = __ldcs(a + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u].x += add;
      if (i + u * blockDim.x < n) __stcs(a + i + u * blockDim.x, v[u]);
    }
  }
}

template <int U>
__global__ void read_k(const uint4* __restrict__ a, size_t n, uint32_t* out) {
  size_t stride = (size_t)gridDim.x * blockDim.x * U;
  uint32_t s = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x * U + threadIdx.x; i < n; i += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) if (i + u * blockDim.x < n) v[u] = __ldcs(a + i + u * blockDim.x);
#pragma unroll
    for (int u = 0; u < U; ++u) s ^= v[u].x ^ v[u].w;
  }
  if (s == 0x12345678) out[0] = s;
}

// Row-strip pattern: matrix [rows, cols] of 16-B chunks; a CTA owns strips of
// 128 rows and walks column blocks of `cw` chunks (cw*16 B per row), the way a
// 128 x (cw*8 bf16) tile walk does.  Each warp handles 4 rows per step.
__global__ void rmw_strip_k(uint4* __restrict__ a, int rows, int cols_chunks, int cw, uint32_t add) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int strips = rows / 128;
  const int cblocks = cols_chunks / cw;
  const long tiles = (long)strips * cblocks;
  const long t0 = tiles * blockIdx.x / gridDim.x, t1 = tiles * (blockIdx.x + 1) / gridDim.x;
  for (long t = t0; t < t1; ++t) {
    const int s = (int)(t / cblocks), cb = (int)(t % cblocks);
    // 128 rows x cw chunks = 128*cw chunks; warps stride over (row, chunk)
    const int per = 128 * cw;
    for (int e = warp * 32 + lane; e < per; e += nw * 32 * 4) {
      uint4 v[4];
      long idx[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int ee = e + u * nw * 32;
        int r = ee / cw, c = ee % cw;
        idx[u] = (long)(s * 128 + r) * cols_chunks + cb * cw + c;
        if (ee < per) v[u] = __ldcs(a + idx[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        int ee = e + u * nw * 32;
        v[u].x += add;
        if (ee < per) __stcs(a + idx[u], v[u]);
      }
    }
  }
}


// 1-D bulk-copy (TMA engine) streaming read: per CTA a ring of S slots of B
// bytes; one producer thread issues cp.async.bulk, consumer warp 1 waits and
// releases (no compute).  Measures the bulk-copy read ceiling per SM.
__global__ void bulk_read_k(const uint8_t* __restrict__ a, size_t bytes, int S, int B) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[64], empty[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t nchunks = bytes / B;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  size_t i = 0;
  if (warp == 0 && lane == 0) {
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++i) {
      const int s = (int)(i % S);
      const uint32_t ph = (uint32_t)((i / S) & 1) ^ 1;
      uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty[s]), fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
      uint32_t ok = 0;
      while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(eb), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(B) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"((uint32_t)__cvta_generic_to_shared(sm + (size_t)s * B)), "l"(a + c * B), "r"(B), "r"(fb) : "memory");
    }
  } else if (warp == 1 && lane == 0) {
    for (size_t c = blockIdx.x; c < nchunks; c += gridDim.x, ++i) {
      const int s = (int)(i % S);
      const uint32_t ph = (uint32_t)((i / S) & 1);
      uint32_t eb = (uint32_t)__cvta_generic_to_shared(&empty[s]), fb = (uint32_t)__cvta_generic_to_shared(&full[s]);
      uint32_t ok = 0;
      while (!ok) asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p;}" : "=r"(ok) : "r"(fb), "r"(ph) : "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(eb) : "memory");
    }
  }
}

// LDGSTS (cp.async 16 B per thread) streaming read into a smem ring, all warps.
__global__ void ldgsts_read_k(const uint4* __restrict__ a, size_t n, int depth) {
  extern __shared__ __align__(128) uint4 sm4[];
  const size_t per_iter = (size_t)gridDim.x * blockDim.x;
  int it = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += per_iter, ++it) {
    uint4* dst = sm4 + (size_t)(it % depth) * blockDim.x + threadIdx.x;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(a + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 6;" ::: "memory");
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

int main() {
  const size_t bytes = (size_t)8 << 30;     // 8 GiB per buffer
  const size_t n = bytes / 16;
  uint4 *a, *b;
  uint32_t* o;
  CK(cudaMalloc(&a, bytes));
  CK(cudaMalloc(&b, bytes));
  CK(cudaMalloc(&o, 4));
  CK(cudaMemset(a, 0, bytes));
  CK(cudaMemset(b, 0, bytes));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto fn, double traffic, const char* name) {
    fn();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    cudaError_t err = cudaGetLastError();
    printf("%-40s %8.1f GB/s  (%.3f ms) %s\n", name, traffic / (best * 1e-3) / 1e9, best,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  timeit([&] { cudaMemcpy(b, a, bytes, cudaMemcpyDeviceToDevice); }, 2.0 * bytes, "cudaMemcpy D2D");
  for (int occ : {2, 4, 8}) {
    char nm[64];
    snprintf(nm, 64, "copy U=4 grid=%dx%d", sms, occ);
    timeit([&] { copy_k<4><<<sms * occ, 256>>>(a, b, n); }, 2.0 * bytes, nm);
    snprintf(nm, 64, "rmw U=4 grid=%dx%d", sms, occ);
    timeit([&] { rmw_k<4><<<sms * occ, 256>>>(a, n, 0); }, 2.0 * bytes, nm);
    snprintf(nm, 64, "rmw U=8 grid=%dx%d", sms, occ);
    timeit([&] { rmw_k<8><<<sms * occ, 256>>>(a, n, 0); }, 2.0 * bytes, nm);
    snprintf(nm, 64, "read U=8 grid=%dx%d", sms, occ);
    timeit([&] { read_k<8><<<sms * occ, 256>>>(a, n, o); }, 1.0 * bytes, nm);
  }
  for (int B : {4096, 8192, 16384, 32768}) {
    for (int occ : {1, 2}) {
      int S = (200 * 1024 / occ) / B;
      if (S > 64) S = 64;
      cudaFuncSetAttribute(bulk_read_k, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
      char nm[64];
      snprintf(nm, 64, "bulk_read B=%d S=%d grid=%dx%d", B, S, sms, occ);
      timeit([&] { bulk_read_k<<<sms * occ, 64, (size_t)S * B>>>((const uint8_t*)a, bytes, S, B); }, 1.0 * bytes, nm);
    }
  }
  for (int occ : {1, 2, 4}) {
    cudaFuncSetAttribute(ldgsts_read_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 512 * 16);
    char nm[64];
    snprintf(nm, 64, "ldgsts_read depth8 512thr grid=%dx%d", sms, occ);
    timeit([&] { ldgsts_read_k<<<sms * occ, 512, 8 * 512 * 16>>>(a, n, 8); }, 1.0 * bytes, nm);
  }
  // strip pattern over a [rows x 4096 bf16] matrix (512 chunks per row)
  const int cols_chunks = 512;
  const int rows = (int)(n / cols_chunks) / 128 * 128;
  for (int cw : {8, 16, 32, 64, 512}) {
    for (int occ : {1, 2, 4}) {
      char nm[64];
      snprintf(nm, 64, "rmw_strip 128x%d B grid=%dx%d", cw * 16, sms, occ);
      timeit([&] { rmw_strip_k<<<sms * occ, 512>>>(a, rows, cols_chunks, cw, 0); },
             2.0 * (double)rows * cols_chunks * 16, nm);
    }
  }
  return 0;
}
