// prefill.cu -- the unmerged prefill of one GEMV group on CUDA cores (SURVEY
// 8f #4), for ctxs without a tensor-core plan (fp32 storage, or the
// SIMT switch forced): Eq. 2 as written,
//     Y[t] = W x_t + sum_j (alpha/r) g_tj B_{e_tj} (A_{e_tj} x_t),
// in two launches, fp32 accumulation in fixed orders (deterministic):
//   prefill_down_simt: U[t][q][j*r + rho] = A_q[e_tj][rho, :] . x_t  -- only the
//     k selected experts of each token, one warp per product;
//   prefill_rows_simt: one warp per (token, row): W[row, :] . x_t (lane-strided,
//     butterfly), then lane 0 adds sum_j (alpha/r) g_tj sum_rho B_q[e_tj][row, rho] U.
// The bf16 tensor-core path is prefill_tc.cu.
#include "lsw_internal.cuh"

namespace lsw {

template <bool kBf16>
__device__ __forceinline__ float ld_elem(const void* p, int64_t i) {
  if (kBf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}

template <typename T>
__device__ __forceinline__ T pick3(int q, T a, T b, T c) { return q == 0 ? a : q == 1 ? b : c; }

template <bool kBf16>
__device__ __forceinline__ float warp_dot(const void* a, const void* x, int64_t n, int lane) {
  float acc = 0.f;
  for (int64_t c = lane; c < n; c += 32) acc = fmaf(ld_elem<kBf16>(a, c), ld_elem<kBf16>(x, c), acc);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return acc;
}

template <bool kBf16>
__global__ void prefill_down_simt(const PrefillParams P) {
  const int lane = threadIdx.x & 31;
  const int kr = P.k * P.r;
  const int64_t n = P.T * P.n_sites * kr;
  const size_t es = kBf16 ? 2 : 4;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = w / (P.n_sites * kr);
    const int q = (int)((w / kr) % P.n_sites);
    const int j = (int)((w % kr) / P.r), rho = (int)(w % P.r);
    const int e = P.idx[t * P.k + j];
    float u = 0.f;
    if (e >= 0 && e < P.n_experts) {
      const uint8_t* a = reinterpret_cast<const uint8_t*>(pick3(q, P.A[0], P.A[1], P.A[2])) +
                         ((int64_t)e * P.r + rho) * P.d_in * es;
      u = warp_dot<kBf16>(a, reinterpret_cast<const uint8_t*>(P.X) + t * P.d_in * es, P.d_in, lane);
    }
    if (lane == 0) P.U[w] = u;
  }
}

template <bool kBf16>
__global__ void prefill_rows_simt(const PrefillParams P) {
  const int lane = threadIdx.x & 31;
  const int64_t n = P.T * P.rows;
  const size_t es = kBf16 ? 2 : 4;
  const int kr = P.k * P.r;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < n;
       w += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t t = w / P.rows, row = w - t * P.rows;
    const int q = (P.n_sites > 2 && row >= P.row_begin[2]) ? 2 : (P.n_sites > 1 && row >= P.row_begin[1]) ? 1 : 0;
    const int64_t rl = row - pick3(q, P.row_begin[0], P.row_begin[1], P.row_begin[2]);
    const int64_t dq = pick3(q, P.d_out[0], P.d_out[1], P.d_out[2]);
    const uint8_t* wr = reinterpret_cast<const uint8_t*>(pick3(q, P.W[0], P.W[1], P.W[2])) + rl * P.d_in * es;
    float y = warp_dot<kBf16>(wr, reinterpret_cast<const uint8_t*>(P.X) + t * P.d_in * es, P.d_in, lane);
    if (lane == 0) {
      const void* Bq = pick3(q, P.B[0], P.B[1], P.B[2]);
      const float* u = P.U + (t * P.n_sites + q) * kr;
      float lo = 0.f;
      for (int j = 0; j < P.k; ++j) {
        const int e = P.idx[t * P.k + j];
        if (e < 0 || e >= P.n_experts) continue;
        const float gj = P.scale * P.gate[t * P.k + j];
        float s = 0.f;
        for (int rho = 0; rho < P.r; ++rho) s = fmaf(ld_elem<kBf16>(Bq, ((int64_t)e * dq + rl) * P.r + rho), u[j * P.r + rho], s);
        lo = fmaf(gj, s, lo);
      }
      P.Y[w] = y + lo;
    }
  }
}

cudaError_t launch_prefill_simt(const PrefillParams& P, int32_t dtype, cudaStream_t s) {
  const bool bf16 = dtype == LSW_BF16;
  const int threads = 256;
  const int64_t w1 = P.T * P.n_sites * P.k * P.r;
  int blocks = (int)((w1 * 32 + threads - 1) / threads);
  if (blocks > 4096) blocks = 4096;
  if (bf16) prefill_down_simt<true><<<blocks, threads, 0, s>>>(P);
  else prefill_down_simt<false><<<blocks, threads, 0, s>>>(P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t w2 = P.T * P.rows;
  blocks = (int)((w2 * 32 + threads - 1) / threads);
  if (blocks > 8192) blocks = 8192;
  if (bf16) prefill_rows_simt<true><<<blocks, threads, 0, s>>>(P);
  else prefill_rows_simt<false><<<blocks, threads, 0, s>>>(P);
  return cudaGetLastError();
}

}  // namespace lsw
