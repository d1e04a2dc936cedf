// gemv.cu -- K4: the batch-1 decode GEMV on the merged weights, Eq. 3.
//
// y = W* x for every site of a group (sites that share x: q|k|v, o, gate|up,
// down), one launch.  HBM-bound: each weight element is read once (2 B bf16).
// One warp per output row: lanes stream the row with 128-bit loads (8 bf16 /
// 4 fp32 per lane per step, coalesced 512 B per warp instruction), x is staged
// once per CTA in shared memory, products accumulate in fp32, and the row sum
// is a __shfl_xor_sync butterfly (north_star "warp-shuffle reductions").
// Persistent grid: a multiple of the SM count; warps stride over rows.
#include "lsw_internal.cuh"

namespace lsw {

constexpr int kGemvThreads = 512;
constexpr int kGemvMaxDin = 16384;    // shared x: 32 KB bf16 / 64 KB fp32
constexpr int kGemvUnroll = 4;        // independent 16-B loads in flight per lane

__device__ __forceinline__ void bf16x8_to_f32(const uint4 u, float* v) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    v[2 * i] = __uint_as_float(w[i] << 16);
    v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
  }
}

__device__ __forceinline__ uint4 ld_stream(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}

// bf16: a "chunk" is 8 elements (16 B).
__global__ void __launch_bounds__(kGemvThreads)
gemv_bf16_kernel(const GemvParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint4* xs = reinterpret_cast<uint4*>(smem_raw);
  const int64_t nchunk = p.d_in / 8;
  const uint4* xg = reinterpret_cast<const uint4*>(p.x);
  for (int64_t i = threadIdx.x; i < nchunk; i += blockDim.x) xs[i] = xg[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = warp; row < p.rows_total; row += nwarps) {
    int s = 0;
    while (s + 1 < p.n_sites && row >= p.site[s + 1].row_begin) ++s;
    const uint4* wr = reinterpret_cast<const uint4*>(p.site[s].W) + (row - p.site[s].row_begin) * nchunk;
    float acc = 0.f;
    int64_t c = lane;
    for (; c + 32 * (kGemvUnroll - 1) < nchunk; c += 32 * kGemvUnroll) {
      uint4 wv[kGemvUnroll];
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) wv[u] = ld_stream(wr + c + 32 * u);
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) {
        float w[8], x[8];
        bf16x8_to_f32(wv[u], w);
        bf16x8_to_f32(xs[c + 32 * u], x);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc = fmaf(w[q], x[q], acc);
      }
    }
    for (; c < nchunk; c += 32) {
      float w[8], x[8];
      bf16x8_to_f32(ld_stream(wr + c), w);
      bf16x8_to_f32(xs[c], x);
#pragma unroll
      for (int q = 0; q < 8; ++q) acc = fmaf(w[q], x[q], acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) p.y[row] = acc;
  }
}

// fp32: a "chunk" is 4 elements (16 B).
__global__ void __launch_bounds__(kGemvThreads)
gemv_f32_kernel(const GemvParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  float4* xs = reinterpret_cast<float4*>(smem_raw);
  const int64_t nchunk = p.d_in / 4;
  const float4* xg = reinterpret_cast<const float4*>(p.x);
  for (int64_t i = threadIdx.x; i < nchunk; i += blockDim.x) xs[i] = xg[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t row = warp; row < p.rows_total; row += nwarps) {
    int s = 0;
    while (s + 1 < p.n_sites && row >= p.site[s + 1].row_begin) ++s;
    const float4* wr = reinterpret_cast<const float4*>(p.site[s].W) + (row - p.site[s].row_begin) * nchunk;
    float acc = 0.f;
    for (int64_t c = lane; c < nchunk; c += 32) {
      const uint4 u = ld_stream(wr + c);
      const float4 x = xs[c];
      acc = fmaf(__uint_as_float(u.x), x.x, acc);
      acc = fmaf(__uint_as_float(u.y), x.y, acc);
      acc = fmaf(__uint_as_float(u.z), x.z, acc);
      acc = fmaf(__uint_as_float(u.w), x.w, acc);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) p.y[row] = acc;
  }
}

cudaError_t launch_gemv(const GemvParams& p, int32_t dtype, int num_sms, cudaStream_t s) {
  const size_t esz = dtype == LSW_BF16 ? 2 : 4;
  const size_t smem = (size_t)p.d_in * esz;
  const int warps_per_cta = kGemvThreads / 32;
  int64_t want = (p.rows_total + warps_per_cta - 1) / warps_per_cta;
  int64_t cap = (int64_t)num_sms * 4;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) grid = 1;
  if (dtype == LSW_BF16) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(gemv_bf16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gemv_bf16_kernel<<<grid, kGemvThreads, smem, s>>>(p);
  } else {
    if (smem > 48 * 1024) cudaFuncSetAttribute(gemv_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    gemv_f32_kernel<<<grid, kGemvThreads, smem, s>>>(p);
  }
  return cudaGetLastError();
}

}  // namespace lsw
