// switch_simt.cu -- K1-simt: the all-layer in-place switch on CUDA cores.
//
// W <- RNE(W + sum_j c_j * B[e_j] @ A[e_j]) for every tile of every adapted
// matrix of every layer in ONE persistent launch (SGMM, Eq. 11, P:321-329;
// "a single CUDA kernel operation"; in place).  The coefficient
// list is Eq. 5/9/10 with Eq. 9's sign corrected (R1) and experts shared by
// both decisions compacted (lsw_internal.cuh build_coefs).
//
// Precision (R13/R14): each expert's B_e A_e product is accumulated in its own
// fp32 accumulator (rho ascending), combined with the fp32 coefficients
// (delta = sum_j c_j * acc_j, j in list order), added to W in fp32 and stored
// once with round-to-nearest-even.  This is the path used for fp32 storage
// (the toy config) and the correctness reference for the tensor-core kernel;
// at bf16 Llama shapes it is FFMA-bound, not HBM-bound.
#include "lsw_internal.cuh"

namespace lsw {

constexpr int kSimtThreads = 256;
constexpr int kSimtTM = 8;            // rows per tile (one warp per row)
constexpr int kSimtTN = 256;          // columns per tile (8 per lane)
constexpr int kSimtMaxK = kMaxTerms * 64;

template <typename T> struct Vec8;
template <> struct Vec8<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float* v) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      v[2 * i] = __uint_as_float(w[i] << 16);
      v[2 * i + 1] = __uint_as_float(w[i] & 0xffff0000u);
    }
  }
  __device__ static void store(__nv_bfloat16* p, const float* v) {
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);   // RNE
      w[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    *reinterpret_cast<uint4*>(p) = make_uint4(w[0], w[1], w[2], w[3]);
  }
};
template <> struct Vec8<float> {
  __device__ static void load(const float* p, float* v) {
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  __device__ static void store(float* p, const float* v) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
};

template <typename T> __device__ __forceinline__ float ld1(const T* p);
template <> __device__ __forceinline__ float ld1<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p) { return __bfloat162float(*p); }

template <typename T>
__global__ void __launch_bounds__(kSimtThreads)
switch_simt_kernel(const SwitchParams p) {
  __shared__ Coefs cf;
  __shared__ int32_t s_parity;
  __shared__ float Bs[kSimtTM * kSimtMaxK];      // [row][term*r + rho]
  if (threadIdx.x == 0) {
    const int32_t parity = *(volatile int32_t*)&p.state->parity;
    s_parity = parity;
    build_coefs(p, parity, cf);
    if (blockIdx.x == 0 && !cf.bad) stage_decision(p, parity);
  }
  __syncthreads();
  const int nt = cf.bad ? 0 : cf.n;
  const int r = p.rank;
  const int K = nt * r;
  if (nt > 0) {
    const int rl = threadIdx.x >> 5;              // row within the tile
    const int cl = (threadIdx.x & 31) * 8;        // first column within the tile
    for (int64_t t = blockIdx.x; t < p.tiles_total; t += gridDim.x) {
      int kd = 0;
      while (kd + 1 < LSW_NKIND && t >= p.kind[kd + 1].tile_begin) ++kd;
      const KindGeom& g = p.kind[kd];
      int64_t local = t - g.tile_begin;
      const int64_t per_layer = (int64_t)g.row_tiles * g.col_tiles;
      const int layer = (int)(local / per_layer);
      local -= (int64_t)layer * per_layer;
      const int rt = (int)(local / g.col_tiles);
      const int ct = (int)(local - (int64_t)rt * g.col_tiles);
      const int64_t row0 = (int64_t)rt * kSimtTM, col0 = (int64_t)ct * kSimtTN;
      const T* Bg = (const T*)g.B;
      const T* Ag = (const T*)g.A;
      __syncthreads();
      for (int i = threadIdx.x; i < kSimtTM * K; i += blockDim.x) {
        const int row = i / K, kk = i - row * K;
        const int j = kk / r, rho = kk - j * r;
        const int64_t grow = row0 + row;
        float v = 0.f;
        if (grow < g.d_out)
          v = ld1<T>(Bg + (((int64_t)layer * p.n_experts + cf.e[j]) * g.d_out + grow) * r + rho);
        Bs[i] = v;
      }
      __syncthreads();
      const int64_t row = row0 + rl, col = col0 + cl;
      if (row < g.d_out && col < g.d_in) {
        float delta[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) delta[q] = 0.f;
        for (int j = 0; j < nt; ++j) {
          float acc[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) acc[q] = 0.f;
          const T* Ap = Ag + (((int64_t)layer * p.n_experts + cf.e[j]) * r) * g.d_in + col;
          const float* bp = Bs + rl * K + j * r;
          for (int rho = 0; rho < r; ++rho) {
            float a[8];
            Vec8<T>::load(Ap + (int64_t)rho * g.d_in, a);
            const float b = bp[rho];
#pragma unroll
            for (int q = 0; q < 8; ++q) acc[q] = fmaf(b, a[q], acc[q]);
          }
          const float c = cf.c[j];
#pragma unroll
          for (int q = 0; q < 8; ++q) delta[q] = fmaf(c, acc[q], delta[q]);
        }
        T* Wp = (T*)g.W + ((int64_t)layer * g.d_out + row) * g.d_in + col;
        const T* Src = p.mode == MODE_RESTORE ? (const T*)g.P + ((int64_t)layer * g.d_out + row) * g.d_in + col : Wp;
        float w[8];
        Vec8<T>::load(Src, w);
#pragma unroll
        for (int q = 0; q < 8; ++q) w[q] = w[q] + delta[q];
        Vec8<T>::store(Wp, w);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) finish_pass(p, s_parity, cf);
}

cudaError_t launch_switch_simt(const SwitchParams& p, int32_t dtype, int grid, cudaStream_t s) {
  if (dtype == LSW_BF16)
    switch_simt_kernel<__nv_bfloat16><<<grid, kSimtThreads, 0, s>>>(p);
  else
    switch_simt_kernel<float><<<grid, kSimtThreads, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace lsw
