// prefill.cu -- the unmerged prefill of one GEMV group for T prompt tokens
// ("For the prefilling phase, we have not implemented
// specific optimizations"): every token t carries its own pre-gated decision
// (idx[t], gate[t]), so the adapters cannot be merged and Eq. 2 is
// evaluated as written,
//     Y[t] = W x_t + sum_j (alpha/r) g_tj B_{e_tj} (A_{e_tj} x_t).
// The dense part is a plain library GEMM per site (cuBLAS, bf16/fp32 in, fp32
// accumulate and out); the LoRA parts are two small kernels:
//   lora_down_prefill: U[t][q][j*r + rho] = A_q[e_tj][rho, :] . x_t
//     (one CTA per (token, site), x_t staged in shared memory, one warp per
//     product, fixed-order warp reduction -- deterministic);
//   lora_up_prefill: Y[t][row] += sum_j s g_tj sum_rho B_q[e_tj][row, rho] U[...]
//     (one thread per (token, row)).
#include <cublas_v2.h>

#include "lsw_internal.cuh"

namespace lsw {

template <bool kBf16>
__device__ __forceinline__ float ld_elem(const void* p, int64_t i) {
  if (kBf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}

constexpr int kPrefillDownWarps = 8;

template <bool kBf16>
__global__ void __launch_bounds__(32 * kPrefillDownWarps)
lora_down_prefill(const PrefillParams P) {
  extern __shared__ float xs[];                       // x_t widened to fp32, [d_in]
  const int t = blockIdx.x, q = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t d_in = P.d_in;
  const uint8_t* xrow = reinterpret_cast<const uint8_t*>(P.X) + (int64_t)t * d_in * (kBf16 ? 2 : 4);
  for (int64_t c = threadIdx.x; c < d_in; c += blockDim.x) xs[c] = ld_elem<kBf16>(xrow, c);
  __syncthreads();
  const int kr = P.k * P.r;
  const void* Aq = q == 0 ? P.A[0] : q == 1 ? P.A[1] : P.A[2];
  for (int d = warp; d < kr; d += kPrefillDownWarps) {
    const int j = d / P.r, rho = d - j * P.r;
    const int e = P.idx[(int64_t)t * P.k + j];
    const int64_t base = ((int64_t)e * P.r + rho) * d_in;
    float acc = 0.f;
    for (int64_t c = lane; c < d_in; c += 32) acc = fmaf(ld_elem<kBf16>(Aq, base + c), xs[c], acc);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) P.U[((int64_t)t * 3 + q) * kr + d] = acc;
  }
}

template <bool kBf16>
__global__ void lora_up_prefill(const PrefillParams P) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P.T * P.rows) return;
  const int64_t t = i / P.rows, row = i - t * P.rows;
  const int q = (P.n_sites > 2 && row >= P.row_begin[2]) ? 2 : (P.n_sites > 1 && row >= P.row_begin[1]) ? 1 : 0;
  const int64_t rl = row - (q == 0 ? P.row_begin[0] : q == 1 ? P.row_begin[1] : P.row_begin[2]);
  const int64_t dq = q == 0 ? P.d_out[0] : q == 1 ? P.d_out[1] : P.d_out[2];
  const void* Bq = q == 0 ? P.B[0] : q == 1 ? P.B[1] : P.B[2];
  const int kr = P.k * P.r;
  const float* u = P.U + (t * 3 + q) * kr;
  float e = 0.f;
  for (int j = 0; j < P.k; ++j) {
    const int ej = P.idx[t * P.k + j];
    const float gj = P.scale * P.gate[t * P.k + j];
    const int64_t off = ((int64_t)ej * dq + rl) * P.r;
    for (int rho = 0; rho < P.r; ++rho) e = fmaf(gj * ld_elem<kBf16>(Bq, off + rho), u[j * P.r + rho], e);
  }
  P.Y[i] += e;
}

cudaError_t launch_prefill(const PrefillParams& P, int32_t dtype, void* cublas_handle, cudaStream_t s) {
  const bool bf16 = dtype == LSW_BF16;
  cublasHandle_t h = static_cast<cublasHandle_t>(cublas_handle);
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  // dense part, per site: Y[:, row_begin .. + d_out] = X W^T.  Column-major
  // view: C = Y^T block [d_out, T] (ldc = rows), A = W ([d_out, d_in] row-major
  // = [d_in, d_out] column-major, op T), B = X^T ([d_in, T], op N).
  const float one = 1.f, zero = 0.f;
  const cudaDataType_t ab = bf16 ? CUDA_R_16BF : CUDA_R_32F;
  for (int q = 0; q < P.n_sites; ++q) {
    const cublasStatus_t st =
        cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)P.d_out[q], (int)P.T, (int)P.d_in, &one, P.W[q], ab,
                     (int)P.d_in, P.X, ab, (int)P.d_in, &zero, P.Y + P.row_begin[q], CUDA_R_32F, (int)P.rows,
                     CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  }
  const size_t smem = (size_t)P.d_in * sizeof(float);
  auto fd = bf16 ? lora_down_prefill<true> : lora_down_prefill<false>;
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    cudaFuncSetAttribute(lora_down_prefill<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(lora_down_prefill<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = smem;
  }
  fd<<<dim3((unsigned)P.T, (unsigned)P.n_sites), 32 * kPrefillDownWarps, smem, s>>>(P);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  const int64_t n = P.T * P.rows;
  (bf16 ? lora_up_prefill<true> : lora_up_prefill<false>)<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t prefill_cublas_create(void** handle) {
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  *handle = h;
  return cudaSuccess;
}

void prefill_cublas_destroy(void* handle) {
  if (handle) cublasDestroy(static_cast<cublasHandle_t>(handle));
}

}  // namespace lsw
