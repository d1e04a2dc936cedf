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
