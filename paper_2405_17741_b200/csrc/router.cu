// router.cu -- K2: the pre-gated top-k router, Eq. 2, G = Softmax(TopK(W_g x)).
//
// One CTA per token (the router runs once per token, not per layer: P:223,
// P:231).  Logits are accumulated in fp64: every bf16*bf16 (or fp32*fp32)
// product is exact in fp64, so the index decision is reproducible bit-for-bit
// against the fp64 oracle (R6).  Top-k by (z desc, index asc) (R5), softmax
// over the k selected logits only (R4), gates stored as fp32.
#include "lsw_internal.cuh"

namespace lsw {

template <typename T>
__device__ __forceinline__ double to_f64(T v);
template <>
__device__ __forceinline__ double to_f64<float>(float v) { return (double)v; }
template <>
__device__ __forceinline__ double to_f64<__nv_bfloat16>(__nv_bfloat16 v) { return (double)__bfloat162float(v); }

constexpr int kRouterThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kRouterThreads)
router_topk_kernel(const T* __restrict__ Wg, const T* __restrict__ x1, int32_t n_experts, int64_t d,
                   int32_t k, int32_t* __restrict__ idx, float* __restrict__ gate, DevState* state) {
  __shared__ double z[LSW_MAX_EXPERTS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = warp; e < n_experts; e += nwarps) {
    const T* row = Wg + (int64_t)e * d;
    double acc = 0.0;
    for (int64_t c = lane; c < d; c += 32) acc += to_f64(row[c]) * to_f64(x1[c]);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) z[e] = acc;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  bool finite = true;
  for (int e = 0; e < n_experts; ++e) finite &= isfinite(z[e]);
  if (!finite) {
    for (int j = 0; j < k; ++j) { idx[j] = -1; gate[j] = 0.f; }
    atomicCAS(&state->err, 0, LSW_DEV_NONFINITE_LOGITS);
    return;
  }
  // selection: repeatedly take the best remaining (z desc, e asc); k <= 8.
  int32_t sel[LSW_MAX_TOPK];
  uint64_t taken = 0;
  for (int j = 0; j < k; ++j) {
    int best = -1;
    for (int e = 0; e < n_experts; ++e) {
      if (taken & (1ull << e)) continue;
      if (best < 0 || z[e] > z[best]) best = e;   // strict '>' keeps the lower index on ties
    }
    sel[j] = best;
    taken |= 1ull << best;
  }
  const double m = z[sel[0]];
  double ex[LSW_MAX_TOPK], sum = 0.0;
  for (int j = 0; j < k; ++j) { ex[j] = exp(z[sel[j]] - m); sum += ex[j]; }
  for (int j = 0; j < k; ++j) {
    idx[j] = sel[j];
    gate[j] = (float)(ex[j] / sum);
  }
}

cudaError_t launch_router(const void* Wg, const void* x1, int32_t n_experts, int64_t d_model,
                          int32_t top_k, int32_t dtype, int32_t* idx, float* gate,
                          DevState* state, cudaStream_t s) {
  if (dtype == LSW_BF16)
    router_topk_kernel<__nv_bfloat16><<<1, kRouterThreads, 0, s>>>(
        (const __nv_bfloat16*)Wg, (const __nv_bfloat16*)x1, n_experts, d_model, top_k, idx, gate, state);
  else
    router_topk_kernel<float><<<1, kRouterThreads, 0, s>>>(
        (const float*)Wg, (const float*)x1, n_experts, d_model, top_k, idx, gate, state);
  return cudaGetLastError();
}

}  // namespace lsw
