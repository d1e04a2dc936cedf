// prefill.cu -- the unmerged prefill of one GEMV group for T prompt tokens
// ("For the prefilling phase, we have not implemented
// specific optimizations"): every token t carries its own pre-gated decision
// (idx[t], gate[t]), so the adapters cannot be merged and Eq. 2 is
// evaluated as written,
//     Y[t] = W x_t + sum_j (alpha/r) g_tj B_{e_tj} (A_{e_tj} x_t).
// The dense part and the LoRA-down products are plain library GEMMs per site
// (cuBLAS, bf16/fp32 in, fp32 accumulate and out): Y = X W^T and, for EVERY
// expert, U = X A^T (the bank A [N, r, d_in] is one [N*r, d_in] matrix).  The
// LoRA-up step: our kernel scales U by each token's gates at its selected
// experts (zero elsewhere, Z), then one fp32 GEMM per site adds Z B_cat^T
// against a packed fp32 copy of B ([d_out, N*r] per layer, built by the ctx on
// the first call).  Fallback (LSW_PREFILL_GATHER=1) -- a per-(token, row) gather:
//   lora_up_prefill: Y[t][row] += sum_j s g_tj sum_rho B_q[e_tj][row, rho] U[t][q][e_tj*r + rho]
//     (one thread per (token, row), 16-B loads of B).
// Measured (7B, 512 tokens, all groups of all layers): packed GEMM 15.6 ms
// (33K tokens/s), gather 20 ms (a shared-memory-staged gather 23 ms).
#include <cublas_v2.h>

#include "lsw_internal.cuh"

namespace lsw {

template <bool kBf16>
__device__ __forceinline__ float ld_elem(const void* p, int64_t i) {
  if (kBf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
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
  const int nr = P.n_experts * P.r;
  const float* u = P.U + (t * 3 + q) * nr;
  float e = 0.f;
  for (int j = 0; j < P.k; ++j) {
    const int ej = P.idx[t * P.k + j];
    const float gj = P.scale * P.gate[t * P.k + j];
    const int64_t off = ((int64_t)ej * dq + rl) * P.r;
    if (kBf16 && (P.r % 8) == 0) {
      const uint4* b4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(Bq) + off);
      for (int v = 0; v < P.r / 8; ++v) {
        const uint4 bb = __ldg(b4 + v);
        const uint32_t w[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          e = fmaf(gj * __uint_as_float(w[h] << 16), u[ej * P.r + 8 * v + 2 * h], e);
          e = fmaf(gj * __uint_as_float(w[h] & 0xffff0000u), u[ej * P.r + 8 * v + 2 * h + 1], e);
        }
      }
    } else {
      for (int rho = 0; rho < P.r; ++rho) e = fmaf(gj * ld_elem<kBf16>(Bq, off + rho), u[ej * P.r + rho], e);
    }
  }
  P.Y[i] += e;
}

// Z[t][q][e*r + rho] = (sum_j [e == e_tj] (alpha/r) g_tj) * U[t][q][e*r + rho]:
// the gate-scaled LoRA-down products of each token's selected experts, zero
// elsewhere, so that the LoRA-up step is one dense GEMM against the packed B.
__global__ void prefill_gate_u(const PrefillParams P) {
  const int nr = P.n_experts * P.r;
  const int64_t n = P.T * 3 * nr;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = i / (3 * nr);
    const int e = (int)((i % nr) / P.r);
    float c = 0.f;
    for (int j = 0; j < P.k; ++j)
      if (P.idx[t * P.k + j] == e) c += P.scale * P.gate[t * P.k + j];
    P.Z[i] = c * P.U[i];
  }
}

// B [N, d_out, r] (one layer of one kind) -> fp32 [d_out, N*r]
template <bool kBf16>
__global__ void pack_bcat(const void* B, float* out, int64_t d_out, int N, int r) {
  const int64_t n = d_out * N * r;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / (N * r);
    const int c = (int)(i % (N * r)), e = c / r, rho = c - e * r;
    out[i] = ld_elem<kBf16>(B, ((int64_t)e * d_out + row) * r + rho);
  }
}

cudaError_t launch_pack_bcat(const void* B, float* out, int64_t d_out, int N, int r, int32_t dtype, cudaStream_t s) {
  if (dtype == LSW_BF16) pack_bcat<true><<<1024, 256, 0, s>>>(B, out, d_out, N, r);
  else pack_bcat<false><<<1024, 256, 0, s>>>(B, out, d_out, N, r);
  return cudaGetLastError();
}

cudaError_t launch_prefill(const PrefillParams& P, int32_t dtype, void* cublas_handle, cudaStream_t s) {
  const bool bf16 = dtype == LSW_BF16;
  cublasHandle_t h = static_cast<cublasHandle_t>(cublas_handle);
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  cudaError_t e;
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
  // LoRA-down for every expert at once, also a library GEMM per site: the
  // bank A_q [N, r, d_in] is a [N*r, d_in] row-major matrix, so
  // U[t][q][e*r + rho] = A_q[e][rho, :] . x_t (N/k times the products a
  // per-token gather needs, on tensor cores, reading A once)
  const int nr = P.n_experts * P.r;
  for (int q = 0; q < P.n_sites; ++q) {
    const cublasStatus_t st =
        cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, nr, (int)P.T, (int)P.d_in, &one, P.A[q], ab, (int)P.d_in, P.X,
                     ab, (int)P.d_in, &zero, P.U + (int64_t)q * nr, CUDA_R_32F, 3 * nr, CUBLAS_COMPUTE_32F,
                     CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  }
  // LoRA-up: Y += Z B_cat^T per site, one fp32 GEMM (K = N*r) against the
  // ctx's packed fp32 copy of B, when it exists; else the per-(token, row) gather
  if (P.Bcat[0]) {
    prefill_gate_u<<<256, 256, 0, s>>>(P);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    for (int q = 0; q < P.n_sites; ++q) {
      const cublasStatus_t st =
          cublasGemmEx(h, CUBLAS_OP_T, CUBLAS_OP_N, (int)P.d_out[q], (int)P.T, nr, &one, P.Bcat[q], CUDA_R_32F, nr,
                       P.Z + (int64_t)q * nr, CUDA_R_32F, 3 * nr, &one, P.Y + P.row_begin[q], CUDA_R_32F,
                       (int)P.rows, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
      if (st != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    }
  } else {
    const int64_t n = P.T * P.rows;
    (bf16 ? lora_up_prefill<true> : lora_up_prefill<false>)<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(P);
  }
  e = cudaGetLastError();
  return e;
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
