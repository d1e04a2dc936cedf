// gemv.cu -- K4: the batch-1 decode GEMV on the merged weights, Eq. 3.
//
// y = W* x for every site of a group (sites that share x: q|k|v, o, gate|up,
// down), one launch.  HBM-bound: each weight element is read once (2 B bf16).
// One warp per output row: lanes stream the row with 128-bit loads (8 bf16 /
// 4 fp32 per lane per step, 512 B per warp instruction, fully coalesced) with
// kUnroll independent loads in flight per lane; x is staged once per CTA in
// shared memory; products accumulate in fp32 and the row sum is a
// __shfl_xor_sync butterfly (north_star "warp-shuffle reductions").
// Persistent, co-resident grid (a multiple of the SM count); rows are dealt
// round-robin over CTAs first (row r -> CTA r % G), so every SM streams the
// same number of rows (+-1) and the last round is spread over all SMs.
#include <cstdlib>

#include "lsw_internal.cuh"

namespace lsw {

#ifdef LSW_TUNING
// tuning builds: per-CTA end time and SM of the last merged-GEMV launch
// (lsw_debug option gemv_trace_buf: device u32 [2][256])
__device__ uint32_t* g_gemv_trace = nullptr;
void gemv_set_trace(uint32_t* p) { cudaMemcpyToSymbol(g_gemv_trace, &p, sizeof(p)); }
#endif

constexpr int kGemvThreads = 512;
constexpr int kGemvUnroll = 8;        // independent 16-B loads in flight per lane

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

template <bool kBf16>
__device__ __forceinline__ float dot_chunk(const uint4 w, const uint4* xs, int64_t c);

template <>
__device__ __forceinline__ float dot_chunk<true>(const uint4 wv, const uint4* xs, int64_t c) {
  float w[8], x[8];
  bf16x8_to_f32(wv, w);
  bf16x8_to_f32(xs[c], x);
  float a = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) a = fmaf(w[q], x[q], a);
  return a;
}

template <>
__device__ __forceinline__ float dot_chunk<false>(const uint4 u, const uint4* xs, int64_t c) {
  const float4 x = reinterpret_cast<const float4*>(xs)[c];
  float a = __uint_as_float(u.x) * x.x;
  a = fmaf(__uint_as_float(u.y), x.y, a);
  a = fmaf(__uint_as_float(u.z), x.z, a);
  a = fmaf(__uint_as_float(u.w), x.w, a);
  return a;
}

__device__ __forceinline__ int site_of(const GemvParams& p, int64_t row) {
  return (p.n_sites > 2 && row >= p.site[2].row_begin) ? 2 : (p.n_sites > 1 && row >= p.site[1].row_begin) ? 1 : 0;
}

// site-indexed kernel parameters without dynamic indexing (which would copy the
// parameter struct to local memory)
template <typename T>
__device__ __forceinline__ T sel3(int q, T a, T b, T c) { return q == 0 ? a : q == 1 ? b : c; }

// Unmerged decode, the LoRA-up term of one row (Eq. 2):
// sum_j (alpha/r) g_j sum_rho B_q[e_j][row, rho] u_q[j][rho], in (j, rho) order;
// 16-B loads of B when a row's r elements are whole chunks.
template <bool kBf16>
__device__ __forceinline__ float lora_up_row(const GemvParams& p, const GemvLora& L, const float* us, int64_t row,
                                             int kr) {
  const int q = site_of(p, row);
  const int64_t rl = row - sel3(q, p.site[0].row_begin, p.site[1].row_begin, p.site[2].row_begin);
  const int64_t dq = sel3(q, p.site[0].d_out, p.site[1].d_out, p.site[2].d_out);
  const void* Bq = sel3(q, L.B[0], L.B[1], L.B[2]);
  float e = 0.f;
  for (int j = 0; j < L.k; ++j) {
    const int64_t off = ((int64_t)L.idx[j] * dq + rl) * L.r;
    const float gj = L.scale * L.gate[j];
    const float* uq = us + q * kr + j * L.r;
    if (kBf16 && (L.r % 8) == 0) {
      const uint4* b4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(Bq) + off);
      for (int v = 0; v < L.r / 8; ++v) {
        float b[8];
        bf16x8_to_f32(__ldg(b4 + v), b);
#pragma unroll
        for (int h = 0; h < 8; ++h) e = fmaf(gj * b[h], uq[8 * v + h], e);
      }
    } else {
      for (int rho = 0; rho < L.r; ++rho) {
        const float b = kBf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(Bq)[off + rho])
                              : reinterpret_cast<const float*>(Bq)[off + rho];
        e = fmaf(gj * b, uq[rho], e);
      }
    }
  }
  return e;
}

// L1 prefetch of the B rows lora_up_row will read for this row
template <bool kBf16>
__device__ __forceinline__ void lora_up_prefetch(const GemvParams& p, const GemvLora& L, int64_t row) {
  const int q = site_of(p, row);
  const int64_t rl = row - sel3(q, p.site[0].row_begin, p.site[1].row_begin, p.site[2].row_begin);
  const int64_t dq = sel3(q, p.site[0].d_out, p.site[1].d_out, p.site[2].d_out);
  const uint8_t* Bq = reinterpret_cast<const uint8_t*>(sel3(q, L.B[0], L.B[1], L.B[2]));
  const int64_t rbytes = (int64_t)L.r * (kBf16 ? 2 : 4);
  for (int j = 0; j < L.k; ++j) {
    const uint8_t* a = Bq + ((int64_t)L.idx[j] * dq + rl) * rbytes;
    for (int64_t o = 0; o < rbytes; o += 128) asm volatile("prefetch.global.L1 [%0];" ::"l"(a + o));
  }
}

// Both operands in registers (16 B each: 8 bf16 or 4 fp32), fp32 sum in order.
template <bool kBf16>
__device__ __forceinline__ float dot_chunk_vv(const uint4 a, const uint4 x) {
  float s;
  if (kBf16) {
    float av[8], xv[8];
    bf16x8_to_f32(a, av);
    bf16x8_to_f32(x, xv);
    s = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) s = fmaf(av[q], xv[q], s);
  } else {
    s = __uint_as_float(a.x) * __uint_as_float(x.x);
    s = fmaf(__uint_as_float(a.y), __uint_as_float(x.y), s);
    s = fmaf(__uint_as_float(a.z), __uint_as_float(x.z), s);
    s = fmaf(__uint_as_float(a.w), __uint_as_float(x.w), s);
  }
  return s;
}

// A "chunk" is 16 B: 8 bf16 or 4 fp32 elements.
template <bool kBf16>
__global__ void __launch_bounds__(kGemvThreads)
gemv_kernel(const GemvParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint4* xs = reinterpret_cast<uint4*>(smem_raw);
  const int64_t nchunk = p.d_in / (kBf16 ? 8 : 4);
  const uint4* xg = reinterpret_cast<const uint4*>(p.x);
  for (int64_t i = threadIdx.x; i < nchunk; i += blockDim.x) xs[i] = xg[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t G = gridDim.x;
  // row r -> CTA r % G, warp (r / G) % nw
  for (int64_t row = blockIdx.x + (int64_t)warp * G; row < p.rows_total; row += (int64_t)nw * G) {
    // select the site with constant indices (no local-memory copy of the params)
    const void* Wb = p.site[0].W;
    int64_t rb = 0;
    if (p.n_sites > 1 && row >= p.site[1].row_begin) { Wb = p.site[1].W; rb = p.site[1].row_begin; }
    if (p.n_sites > 2 && row >= p.site[2].row_begin) { Wb = p.site[2].W; rb = p.site[2].row_begin; }
    const uint4* wr = reinterpret_cast<const uint4*>(Wb) + (row - rb) * nchunk;
    float acc = 0.f;
    int64_t c = lane;
    for (; c + 32 * (kGemvUnroll - 1) < nchunk; c += 32 * kGemvUnroll) {
      uint4 wv[kGemvUnroll];
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) wv[u] = ld_stream(wr + c + 32 * u);
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u) acc += dot_chunk<kBf16>(wv[u], xs, c + 32 * u);
    }
    // ragged tail of the row: < kUnroll chunks per lane, still issued together
    {
      uint4 wv[kGemvUnroll];
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u)
        if (c + 32 * u < nchunk) wv[u] = ld_stream(wr + c + 32 * u);
#pragma unroll
      for (int u = 0; u < kGemvUnroll; ++u)
        if (c + 32 * u < nchunk) acc += dot_chunk<kBf16>(wv[u], xs, c + 32 * u);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (lane == 0) p.y[row] = acc;
  }
}

// ---------------------------------------------------------------------------
// Bulk-staged variant (default): one producer thread streams whole rows into a
// ring of shared-memory slots with 1-D cp.async.bulk copies (one per row,
// completion on an mbarrier), so ~200 KB per SM are in flight without any
// register cost; 8 consumer warps reduce rows from shared memory (512 B per
// warp instruction, conflict-free) against x (also in shared memory).
constexpr int kBulkConsumers = 16;   // measured (7B token of GEMVs): 8 warps 2.39 ms, 16 2.25, 24 2.24
constexpr int kBulkThreads = 32 * (1 + kBulkConsumers);
constexpr int kLoraWarps = 4;        // unmerged GEMV: extra warps computing the LoRA-down products
constexpr int kMaxDots = 3 * LSW_MAX_TOPK * 64;   // n_sites * k * r
constexpr int kMaxLocal = 1024;      // unmerged GEMV: row sums kept in shared memory up to this many rows per CTA
constexpr int kBulkMaxSlots = 32;

__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint32_t g_mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
               : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok;
}

__device__ __forceinline__ uint64_t g_globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Wait with a ~20 s watchdog (a protocol bug traps instead of hanging the GPU).
__device__ __forceinline__ void g_mbar_wait(uint32_t bar, uint32_t parity) {
  if (g_mbar_try(bar, parity)) return;
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (uint32_t n = 1; !g_mbar_try(bar, parity); ++n) {
    if ((n & 1023u) == 0) {
      asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();
    }
  }
}

// x as the consumer warps read it: bf16 x is widened once per GEMV into two
// fp32 planes (elements 0-3 and 4-7 of every 16-B chunk of the row, each plane
// read conflict-free with one LDS.128 per lane), so the inner loop is one
// LDS.128 of W, two of x, 8 bf16->fp32 unpacks and 4 packed FFMA2 per 8
// elements (measured: the unpack + scalar-FMA loop was the bottleneck of the
// bulk GEMV, 5.5 TB/s against 7.2 TB/s for the same stream without the math).
__host__ __device__ inline uint32_t x_stage_bytes(uint32_t row_bytes, bool bf16) {
  return ((bf16 ? 2 * row_bytes : row_bytes) + 127) & ~127u;
}

template <bool kBf16>
__device__ __forceinline__ void stage_x(const void* xg, uint8_t* xs, uint32_t row_bytes, int tid, int nthreads) {
  const uint4* src = reinterpret_cast<const uint4*>(xg);
  const int n16 = (int)(row_bytes / 16);
  if (kBf16) {
    float4* lo = reinterpret_cast<float4*>(xs);
    float4* hi = lo + n16;
    for (int i = tid; i < n16; i += nthreads) {
      const uint4 u = src[i];
      lo[i] = make_float4(__uint_as_float(u.x << 16), __uint_as_float(u.x & 0xffff0000u),
                          __uint_as_float(u.y << 16), __uint_as_float(u.y & 0xffff0000u));
      hi[i] = make_float4(__uint_as_float(u.z << 16), __uint_as_float(u.z & 0xffff0000u),
                          __uint_as_float(u.w << 16), __uint_as_float(u.w & 0xffff0000u));
    }
  } else {
    uint4* dst = reinterpret_cast<uint4*>(xs);
    for (int i = tid; i < n16; i += nthreads) dst[i] = src[i];
  }
}

__device__ __forceinline__ uint64_t g_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t g_ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float g_sum2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  return lo + hi;
}
// acc (fp32 pairs) += bf16 chunk w * x chunk (lo, hi planes)
__device__ __forceinline__ uint64_t dot8_f2(const uint4 w, const float4 lo, const float4 hi, uint64_t acc) {
  acc = g_ffma2(g_pack(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u)), g_pack(lo.x, lo.y), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u)), g_pack(lo.z, lo.w), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u)), g_pack(hi.x, hi.y), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u)), g_pack(hi.z, hi.w), acc);
  return acc;
}

// One 16-B chunk of a LoRA-down row against x as staged (raw bf16, fp32
// planes, or fp32), fp32 products summed in element order.
template <bool kBf16, bool kXB>
__device__ __forceinline__ float lora_chunk(const uint4 a, const uint8_t* xs, int64_t c, int64_t n16) {
  if (kBf16 && kXB) return dot_chunk<true>(a, reinterpret_cast<const uint4*>(xs), c);
  if (!kBf16) return dot_chunk<false>(a, reinterpret_cast<const uint4*>(xs), c);
  const float4 lo = reinterpret_cast<const float4*>(xs)[c], hi = reinterpret_cast<const float4*>(xs)[n16 + c];
  const float x[8] = {lo.x, lo.y, lo.z, lo.w, hi.x, hi.y, hi.z, hi.w};
  float w[8];
  bf16x8_to_f32(a, w);
  float s = 0.f;
#pragma unroll
  for (int q = 0; q < 8; ++q) s = fmaf(w[q], x[q], s);
  return s;
}

// acc (fp32 pairs) += bf16 chunk w * bf16 chunk x: the same element pairs and
// FFMA2 order as dot8_f2 (bitwise-identical results), x widened in registers
__device__ __forceinline__ uint64_t dot8_bb(const uint4 w, const uint4 x, uint64_t acc) {
  acc = g_ffma2(g_pack(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xffff0000u)),
                g_pack(__uint_as_float(x.x << 16), __uint_as_float(x.x & 0xffff0000u)), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.y << 16), __uint_as_float(w.y & 0xffff0000u)),
                g_pack(__uint_as_float(x.y << 16), __uint_as_float(x.y & 0xffff0000u)), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.z << 16), __uint_as_float(w.z & 0xffff0000u)),
                g_pack(__uint_as_float(x.z << 16), __uint_as_float(x.z & 0xffff0000u)), acc);
  acc = g_ffma2(g_pack(__uint_as_float(w.w << 16), __uint_as_float(w.w & 0xffff0000u)),
                g_pack(__uint_as_float(x.w << 16), __uint_as_float(x.w & 0xffff0000u)), acc);
  return acc;
}

// One row of W (in shared memory) against the staged x, reduced over the warp.
// kXB: x staged as raw bf16 (one LDS.128 of x per 8 elements instead of two of
// the fp32 planes: the consumers' shared-memory traffic per W byte drops from
// 3x to 2x, the ring fill adds 1x).
template <bool kBf16, bool kXB = false>
__device__ __forceinline__ float row_dot(const uint8_t* wrow, const uint8_t* xs, int64_t n16, int lane) {
  const uint4* w4 = reinterpret_cast<const uint4*>(wrow);
  float acc;
  if (kBf16 && kXB) {
    const uint4* x4 = reinterpret_cast<const uint4*>(xs);
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    int64_t c = lane;
    for (; c + 96 < n16; c += 128) {
      const uint4 w0 = w4[c], w1 = w4[c + 32], w2 = w4[c + 64], w3 = w4[c + 96];
      const uint4 x0 = x4[c], x1 = x4[c + 32], x2 = x4[c + 64], x3 = x4[c + 96];
      a0 = dot8_bb(w0, x0, a0);
      a1 = dot8_bb(w1, x1, a1);
      a2 = dot8_bb(w2, x2, a2);
      a3 = dot8_bb(w3, x3, a3);
    }
    for (; c < n16; c += 32) a0 = dot8_bb(w4[c], x4[c], a0);
    acc = (g_sum2(a0) + g_sum2(a1)) + (g_sum2(a2) + g_sum2(a3));
  } else if (kBf16) {
    const float4* lo = reinterpret_cast<const float4*>(xs);
    const float4* hi = lo + n16;
    uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;     // (+0.f, +0.f) pairs
    int64_t c = lane;
    for (; c + 96 < n16; c += 128) {              // 4 independent chunks per lane in flight
      const uint4 w0 = w4[c], w1 = w4[c + 32], w2 = w4[c + 64], w3 = w4[c + 96];
      a0 = dot8_f2(w0, lo[c], hi[c], a0);
      a1 = dot8_f2(w1, lo[c + 32], hi[c + 32], a1);
      a2 = dot8_f2(w2, lo[c + 64], hi[c + 64], a2);
      a3 = dot8_f2(w3, lo[c + 96], hi[c + 96], a3);
    }
    for (; c < n16; c += 32) a0 = dot8_f2(w4[c], lo[c], hi[c], a0);
    acc = (g_sum2(a0) + g_sum2(a1)) + (g_sum2(a2) + g_sum2(a3));
  } else {
    const uint4* x4 = reinterpret_cast<const uint4*>(xs);
    float acc0 = 0.f, acc1 = 0.f;
    int64_t c = lane;
    for (; c + 32 < n16; c += 64) {
      acc0 += dot_chunk<false>(w4[c], x4, c);
      acc1 += dot_chunk<false>(w4[c + 32], x4, c + 32);
    }
    if (c < n16) acc0 += dot_chunk<false>(w4[c], x4, c);
    acc = acc0 + acc1;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return acc;
}

// kSplit (merged form, rows over 24 KB -- the FFN down projection of
// Mistral-7B / Llama-2-13B): each row
// is reduced by TWO warps, one half of its columns each, the second to finish
// adding the halves in a fixed order (h0 + h1; deterministic) -- halves the
// per-row latency that the last rows of a launch expose before the CTA can
// leave (measured with the dot products off: down 14.4 vs 16.1 us per launch).
template <bool kBf16, bool kLora, bool kXB, bool kSplit = false>
__global__ void __launch_bounds__(kLora ? kBulkThreads + 32 * kLoraWarps : kBulkThreads, 1)
gemv_bulk_kernel(const GemvParams p, int32_t slots, int32_t R, int32_t early_w, const GemvLora L) {
  static_assert(!(kSplit && kLora), "split rows: merged form only");
  constexpr int UH = kSplit ? 2 : 1;            // units (warps) per row
  extern __shared__ __align__(128) uint8_t smem_raw[];
  __shared__ __align__(8) uint64_t full[kBulkMaxSlots], empty[kBulkMaxSlots];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t row_bytes = (uint32_t)(p.d_in * (kBf16 ? 2 : 4));
  const uint32_t x_bytes = x_stage_bytes(row_bytes, kBf16 && !kXB);
  const size_t slot_bytes = (size_t)R * row_bytes;
  uint8_t* xs = smem_raw;
  uint8_t* ring = smem_raw + x_bytes;
  const int64_t G = gridDim.x;
  const int64_t n_chunks = (p.rows_total + R - 1) / R;            // chunk c = rows [c*R, c*R + R)
  const int64_t my_chunks = n_chunks > blockIdx.x ? (n_chunks - blockIdx.x + G - 1) / G : 0;
  // Chunks issued so far.  A consumer warp takes only every 16th row, so it can
  // reach a slot's NEXT-but-one fill while the next fill is not yet issued; the
  // full barrier's parity would then alias an already completed phase.  Waiting
  // for the ticket first makes the parity wait unambiguous.  Written with
  // st.release and read with ld.acquire (CTA scope, morally strong -- not a
  // data race, though racecheck reports it): the consumer's parity wait then
  // sees at least the producer's expect_tx of that chunk.
  __shared__ int64_t issued;
  if (threadIdx.x == 0) {
    for (int s = 0; s < slots; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(&full[s])), "r"(1));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(&empty[s])), "r"(R * UH));
    }
    issued = 0;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();                                  // barrier inits visible
  // Programmatic dependent launch: W may be prefetched before the previous
  // grid completes only when the caller says so (early_w: the previous launch
  // was a GEMV that itself waited for whatever wrote W).  Everything else
  // (x, y) is touched only after griddepcontrol.wait.
  if (!(early_w & 1)) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (warp == 0) {
    // producer: one bulk copy per contiguous run of a chunk's rows (a chunk is
    // split only where it crosses from one site's matrix into the next);
    // starts at once -- x is staged by the consumer warps in parallel
    if (lane == 0) {
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      for (int64_t i = 0; i < my_chunks; ++i) {
        const int s = (int)(i % slots);
        g_mbar_wait(s_u32(&empty[s]), (uint32_t)((i / slots) & 1) ^ 1);
        const int64_t r0 = (blockIdx.x + i * G) * R;
        const int64_t r1 = r0 + R < p.rows_total ? r0 + R : p.rows_total;
        const uint32_t bar = s_u32(&full[s]);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)((r1 - r0) * row_bytes)) : "memory");
        int64_t r = r0;
        while (r < r1) {
          const void* Wb = p.site[0].W;
          int64_t rb = 0, re = p.n_sites > 1 ? p.site[1].row_begin : p.rows_total;
          if (p.n_sites > 1 && r >= p.site[1].row_begin) {
            Wb = p.site[1].W; rb = p.site[1].row_begin; re = p.n_sites > 2 ? p.site[2].row_begin : p.rows_total;
          }
          if (p.n_sites > 2 && r >= p.site[2].row_begin) { Wb = p.site[2].W; rb = p.site[2].row_begin; re = p.rows_total; }
          const int64_t run_end = r1 < re ? r1 : re;
          const uint8_t* src = reinterpret_cast<const uint8_t*>(Wb) + (r - rb) * (int64_t)row_bytes;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
              ::"r"(s_u32(ring + s * slot_bytes + (r - r0) * (size_t)row_bytes)), "l"(src),
                "r"((uint32_t)((run_end - r) * row_bytes)), "r"(bar), "l"(pol)
              : "memory");
          r = run_end;
        }
        asm volatile("st.release.cta.shared::cta.b64 [%0], %1;" ::"r"(s_u32(&issued)), "l"(i + 1) : "memory");
      }
    }
    return;
  }
  if (early_w & 1) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // after our wait: see above
  // unmerged form: the decision is validated by every CTA alike (indices in
  // [0, N) and distinct, gates finite -- as the switch's build_coefs); an
  // invalid one drops the LoRA terms (y = W x) and latches the error.  Only
  // the LoRA warps look at it (the consumers start streaming at once: the
  // check's dependent global loads cost 5 % of the token when every warp ran
  // it); the consumers read the verdict after their final barrier with them.
  __shared__ int32_t s_lora_ok;
  bool lora_ok = false;
  if (kLora && warp > kBulkConsumers) {
    int bad = 0;
    for (int j = 0; j < L.k; ++j) {
      const int32_t e = L.idx[j];
      if (e < 0 || e >= L.n_experts) bad = LSW_DEV_BAD_INDEX;
      for (int i = 0; i < j; ++i) if (L.idx[i] == e) bad = LSW_DEV_BAD_INDEX;
      if (!bad && !isfinite(L.gate[j])) bad = LSW_DEV_BAD_GATE;
    }
    lora_ok = bad == 0;
    if (threadIdx.x == 32 * (1 + kBulkConsumers)) {
      s_lora_ok = lora_ok;
      if (bad && blockIdx.x == 0) atomicCAS(L.err, 0, bad);
    }
  }
  const int kr = lora_ok ? L.k * L.r : 0;
  const int n_dots = kLora ? p.n_sites * kr : 0;
  // unmerged form: u (all LoRA-down products of the group), staged by the
  // LoRA-down warps once every CTA has published its share
  __shared__ float us[kLora ? kMaxDots : 1];
  __shared__ float acc_s[kLora ? kMaxLocal : 1], e_s[kLora ? kMaxLocal : 1];   // this CTA's rows (if they fit)
  const int64_t n_local = my_chunks * R;
  if (kLora && warp > kBulkConsumers) {
    // LoRA-down (Eq. 2, A_{e_j} x) by the kLoraWarps extra warps, while the
    // consumers stream W: the group's n_sites * k * r dot products are dealt
    // over the grid (dot d -> CTA d % G), each split over the dot warps' K
    // ranges (x read from global, L2-hot), partial sums added in warp order
    // (deterministic), published as u[d] and a release increment of the
    // arrival counter.  Then these warps wait for every CTA's products, stage
    // u in shared memory and compute the LoRA-up terms of the CTA's rows.
    __shared__ float part[kLoraWarps];
    const int dw = warp - 1 - kBulkConsumers;
    const int64_t n16 = row_bytes / 16;
    const int64_t per = (n16 + kLoraWarps - 1) / kLoraWarps;
    const uint4* x4 = reinterpret_cast<const uint4*>(p.x);
    for (int d = blockIdx.x; d < n_dots; d += (int)G) {
      const int q = d / kr, j = (d - q * kr) / L.r, rho = d - q * kr - j * L.r;
      const uint4* a4 = reinterpret_cast<const uint4*>(reinterpret_cast<const uint8_t*>(sel3(q, L.A[0], L.A[1], L.A[2])) +
                                                       ((int64_t)L.idx[j] * L.r + rho) * row_bytes);
      const int64_t c0 = dw * per, c1 = c0 + per < n16 ? c0 + per : n16;
      float acc = 0.f;
      for (int64_t c = c0 + lane; c < c1; c += 32 * 8) {
        uint4 a[8], x[8];
#pragma unroll
        for (int v = 0; v < 8; ++v) {
          const bool in = c + 32 * v < c1;
          a[v] = in ? __ldg(a4 + c + 32 * v) : make_uint4(0, 0, 0, 0);
          x[v] = in ? __ldg(x4 + c + 32 * v) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int v = 0; v < 8; ++v) acc += dot_chunk_vv<kBf16>(a[v], x[v]);
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
      if (lane == 0) part[dw] = acc;
      __syncwarp();
      asm volatile("bar.sync 2, %0;" ::"r"(32 * kLoraWarps) : "memory");
      if (dw == 0 && lane == 0) {
        float u = 0.f;
        for (int w = 0; w < kLoraWarps; ++w) u += part[w];
        L.u[d] = u;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(L.arrive) : "memory");
      }
      __syncwarp();
      asm volatile("bar.sync 2, %0;" ::"r"(32 * kLoraWarps) : "memory");   // part[] reusable
    }
    // the LoRA-up operands of this CTA's rows (B rows of the selected
    // experts) requested into L1 while the other CTAs' products arrive
    if (n_local <= kMaxLocal && lora_ok)
      for (int64_t t = threadIdx.x - 32 * (1 + kBulkConsumers); t < n_local; t += 32 * kLoraWarps) {
        const int64_t row = (blockIdx.x + (t / R) * G) * R + t % R;
        if (row < p.rows_total) lora_up_prefetch<kBf16>(p, L, row);
      }
    if (dw == 0 && lane == 0) {
      uint32_t v;
      const uint64_t t0 = g_globaltimer();
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(L.arrive) : "memory");
        if (v >= (uint32_t)n_dots) break;
        __nanosleep(64);
        if (g_globaltimer() - t0 > 20000000000ull) __trap();
      }
    }
    __syncwarp();
    asm volatile("bar.sync 2, %0;" ::"r"(32 * kLoraWarps) : "memory");
    for (int d = threadIdx.x - 32 * (1 + kBulkConsumers); d < n_dots; d += 32 * kLoraWarps) us[d] = __ldcg(L.u + d);
    __syncwarp();
    asm volatile("bar.sync 2, %0;" ::"r"(32 * kLoraWarps) : "memory");
    // every CTA's products read: this CTA is done with the counters; the last
    // one resets both for the next launch (which publishes its products only
    // after this grid has completed: griddepcontrol.wait).  Here, not at the
    // CTA's end: the atomic's round trip stays off the path to the CTA's exit
    // (the next launch's CTA on this SM starts only then).
    if (dw == 0 && lane == 0) {
      uint32_t prev;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(L.depart) : "memory");
      if (prev == gridDim.x - 1) {
        *reinterpret_cast<volatile uint32_t*>(L.arrive) = 0;
        *reinterpret_cast<volatile uint32_t*>(L.depart) = 0;
        __threadfence();
      }
    }
    // LoRA-up terms of this CTA's rows, one lane per row, while the consumers
    // still stream (their row sums wait in acc_s; joined at the end)
    if (n_local <= kMaxLocal && !(L.flags & 4) && lora_ok)
      for (int64_t t = threadIdx.x - 32 * (1 + kBulkConsumers); t < n_local; t += 32 * kLoraWarps) {
        const int64_t row = (blockIdx.x + (t / R) * G) * R + t % R;
        e_s[t] = row < p.rows_total ? lora_up_row<kBf16>(p, L, us, row, kr) : 0.f;
      }
    __syncwarp();
    asm volatile("barrier.sync 3, %0;" ::"r"(32 * (kBulkConsumers + kLoraWarps)) : "memory");   // two code sites: not .aligned
    return;
  }
  // x -> shared (consumer warps), then a named barrier among the consumers only
  stage_x<kBf16 && !kXB>(p.x, xs, row_bytes, threadIdx.x - 32, 32 * kBulkConsumers);
  __syncwarp();
  asm volatile("bar.sync 1, %0;" ::"r"(32 * kBulkConsumers) : "memory");
  // consumers: unit u = (local chunk i, row k in chunk); warp cw takes u = cw mod 16
  const int cw = warp - 1;
  const int64_t nchunk16 = row_bytes / 16;
  const bool in_smem = kLora && n_local <= kMaxLocal;
  // kSplit: the halves' partial sums of a slot's rows, and how many halves are in
  __shared__ float part[kSplit ? kBulkMaxSlots : 1][kSplit ? 16 : 1][2];
  __shared__ uint32_t part_n[kSplit ? kBulkMaxSlots : 1][kSplit ? 16 : 1];
  if (kSplit)
    for (int t = threadIdx.x - 32; t < kBulkMaxSlots * 16; t += 32 * kBulkConsumers) part_n[t / 16][t % 16] = 0;
  if (kSplit) {
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kBulkConsumers) : "memory");
  }
  for (int64_t u = cw; u < my_chunks * R * UH; u += kBulkConsumers) {
    const int64_t i = u / (R * UH);
    const int64_t rem = u - i * R * UH;
    const int k = (int)(rem / UH), h = (int)(rem - (rem / UH) * UH);
    const int s = (int)(i % slots);
    const int64_t row = (blockIdx.x + i * G) * R + k;
    for (;;) {                                    // ticket: chunk i's fill is armed
      int64_t v;
      asm volatile("ld.acquire.cta.shared::cta.b64 %0, [%1];" : "=l"(v) : "r"(s_u32(&issued)) : "memory");
      if (v > i) break;
      __nanosleep(64);
    }
    g_mbar_wait(s_u32(&full[s]), (uint32_t)((i / slots) & 1));
    if (kSplit && row < p.rows_total && !(early_w & 2)) {
      const int64_t c0 = h ? nchunk16 / 2 : 0, c1 = h ? nchunk16 : nchunk16 / 2;
      const float acc = row_dot<kBf16, kXB>(ring + s * slot_bytes + (size_t)k * row_bytes + c0 * 16, xs + c0 * 16,
                                            c1 - c0, lane);
      if (lane == 0) {
        part[s][k][h] = acc;
        uint32_t old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(s_u32(&part_n[s][k]))
                     : "memory");
        if (old == 1) {                            // the second half in: y = h0 + h1
          p.y[row] = part[s][k][0] + part[s][k][1];
          part_n[s][k] = 0;                        // (reused only after this slot's next fill)
        }
      }
    } else if (row < p.rows_total && !(early_w & 2)) {    // early_w bit 1: tuning probe, stream only
      const float acc = row_dot<kBf16, kXB>(ring + s * slot_bytes + (size_t)k * row_bytes, xs, nchunk16, lane);
      if (lane == 0) {
        if (in_smem) acc_s[u] = acc;
        else p.y[row] = acc;
      }
    }
    // (the slot's reads have returned before the release arrive; the producer's
    // acquire wait orders the next bulk copy after them -- no proxy fence, as in
    // TMA pipelines: measured, one per row costs 5 % of the unmerged decode)
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[s])) : "memory");
  }
#ifdef LSW_TUNING
  if (!kLora && g_gemv_trace) {
    __syncwarp();
    asm volatile("bar.sync 1, %0;" ::"r"(32 * kBulkConsumers) : "memory");
    if (cw == 0 && lane == 0 && blockIdx.x < 256) {
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_gemv_trace[blockIdx.x] = (uint32_t)g_globaltimer();
      g_gemv_trace[256 + blockIdx.x] = smid + 1;
    }
  }
#endif
  if (kLora) {
    // Eq. 2: y = (W x) + LoRA-up term, one rounding of the sum per row
    __syncwarp();
    asm volatile("barrier.sync 3, %0;" ::"r"(32 * (kBulkConsumers + kLoraWarps)) : "memory");   // two code sites: not .aligned   // e_s / us ready
    lora_ok = s_lora_ok != 0;                      // written by the LoRA warps before the barrier
    const bool up = !(L.flags & 4) && !(early_w & 2) && lora_ok;
    if (in_smem) {
      for (int64_t t = threadIdx.x - 32; t < n_local; t += 32 * kBulkConsumers) {
        const int64_t row = (blockIdx.x + (t / R) * G) * R + t % R;
        if (row < p.rows_total && !(early_w & 2)) p.y[row] = up ? acc_s[t] + e_s[t] : acc_s[t];
      }
    } else if (up) {
      // many rows per CTA (small grids): the terms now, one lane per row
      for (int64_t t = threadIdx.x - 32; t < n_local; t += 32 * kBulkConsumers) {
        const int64_t row = (blockIdx.x + (t / R) * G) * R + t % R;
        if (row < p.rows_total) p.y[row] = p.y[row] + lora_up_row<kBf16>(p, L, us, row, kr);
      }
    }
  }
}

cudaError_t launch_gemv(const GemvParams& p, int32_t dtype, const GemvTune& t, cudaStream_t s, bool early_w,
                        GemvLora* lora) {
  const bool bf16 = dtype == LSW_BF16;
  const int num_sms = t.grid_cap;
  if (!t.ldg) {
    // bulk-copy throughput grows with bytes per operation (scripts/membench.cu:
    // 4 KB ops 2.6 TB/s ... 32 KB ops 7.3 TB/s): move R >= 1 rows per op, ~32 KB;
    // x staged in shared memory as raw bf16 / fp32
    const uint32_t row_bytes = (uint32_t)(p.d_in * (bf16 ? 2 : 4));
    const uint32_t x_bytes = x_stage_bytes(row_bytes, false);
    const size_t budget = lora ? t.budget_lora : t.budget;
    // rows per op: of the R with op_min <= R * row_bytes <= op_bytes (R = 1
    // when one row is already larger), the one that puts the most bytes in
    // flight (slots * R * row_bytes), ties to the smaller op.  Measured (r02,
    // 7B, groups of every layer back to back): 8 KB rows R = 3 (24 KB ops,
    // 7 slots) vs R = 4 (32 KB, 5 slots): q|k|v 6.14 vs 5.81 TB/s, o 4.40 vs
    // 3.07, gate|up 6.68 vs 6.34; 16 KB ops (R = 2) 4.7-5.0 -- token 2.12-2.14
    // vs 2.19 ms; 13B (10 KB rows) keeps R = 3 (R = 2, 20 KB ops: 4.40 vs 4.27)
    int R = 1;
    {
      size_t best = 0;
      for (int r = 1; r <= 16; ++r) {
        const size_t op = (size_t)r * row_bytes;
        if (op > t.op_bytes && r > 1) break;
        if (op < t.op_min && (size_t)(r + 1) * row_bytes <= t.op_bytes) continue;
        const size_t sl = budget > x_bytes ? (budget - x_bytes) / op : 0;
        const size_t fly = (sl > (size_t)kBulkMaxSlots ? (size_t)kBulkMaxSlots : sl) * op;
        if (sl >= 2 && fly > best) { best = fly; R = r; }
      }
    }
    const size_t slot_bytes = (size_t)R * row_bytes;
    // Ring budget.  Measured (7B token of GEMVs): 220 KB 2.37 ms, 110 KB 2.59 ms,
    // 72 KB 3.49 ms -- a deep ring per SM beats letting the next GEMV's CTA
    // co-reside under PDL; with the bf16 x staging (same box, 2 runs each):
    // 220 KB 2.172, 176 KB 2.164, 144 KB 2.32, 112 KB 2.53 ms -- five 32-KB
    // slots in flight rather than six.  Two CTAs per SM (8 consumer warps and
    // a half ring each, so that the next launch's CTA streams before this
    // one's last CTA on the SM ends; r02, same box): 104 KB 2.42, 110 KB 2.36,
    // 80 KB 2.60 ms vs 2.19 for one CTA with 176 KB -- dropped.
    // (the unmerged form keeps ~12 KB of static shared memory: u, row sums, terms)
    int slots = budget > x_bytes ? (int)((budget - x_bytes) / slot_bytes) : 0;
    if (slots > kBulkMaxSlots) slots = kBulkMaxSlots;
    if (slots >= 2) {
      const size_t smem = x_bytes + (size_t)slots * slot_bytes;
      // rows over 24 KB (at most 16 per chunk): each reduced by two warps.
      // Measured (down, us per launch, same box): Mistral-7B (28 KB rows)
      // 19.6 vs 20.8, Llama-2-13B (27 KB) 23.4 vs 24.9, but Llama-2-7B (22 KB,
      // 7 ring slots instead of 5) 17.1 vs 16.1
      const bool split = !lora && R <= 16 && (t.split_rows == 2 || (t.split_rows == 1 && row_bytes > 24576));
      auto fn = lora ? (bf16 ? gemv_bulk_kernel<true, true, true> : gemv_bulk_kernel<false, true, false>)
              : split ? (bf16 ? gemv_bulk_kernel<true, false, true, true> : gemv_bulk_kernel<false, false, false, true>)
                      : (bf16 ? gemv_bulk_kernel<true, false, true> : gemv_bulk_kernel<false, false, false>);
      static size_t smem_set[3][2] = {{0, 0}, {0, 0}, {0, 0}};   // attribute set once per kernel (not per launch)
      const int fi = lora ? 1 : split ? 2 : 0;
      if (smem > smem_set[fi][bf16]) {
        cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        smem_set[fi][bf16] = smem;
      }
      const int64_t n_chunks = (p.rows_total + R - 1) / R;
      int grid = (int)(n_chunks < num_sms ? n_chunks : num_sms);
      if (grid < 1) grid = 1;
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(grid);
      lc.blockDim = dim3(kBulkThreads + (lora ? 32 * kLoraWarps : 0));
      lc.dynamicSmemBytes = smem;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      const GemvLora none{};
      return cudaLaunchKernelEx(&lc, fn, p, slots, R,
                                (int32_t)((early_w || lora ? 1 : 0) | (t.probe ? 2 : 0)),
                                lora ? *lora : none);
    }
  }
  if (lora) return cudaErrorNotSupported;   // the LDG variant has no unmerged form
  const size_t smem = (size_t)p.d_in * (bf16 ? 2 : 4);
  auto fn = bf16 ? gemv_kernel<true> : gemv_kernel<false>;
  static int occ_cache[2][8] = {};          // [dtype][smem bucket of 16 KB] -> CTAs per SM
  const int bucket = (int)(smem >> 14) < 8 ? (int)(smem >> 14) : 7;
  int& occ = occ_cache[bf16][bucket];
  static size_t smem_set[2] = {0, 0};
  if (smem > 48 * 1024 && smem > smem_set[bf16]) {
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set[bf16] = smem;
  }
  if (occ == 0) {
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, kGemvThreads, ((size_t)bucket + 1) << 14);
    if (occ < 1) occ = 1;
  }
  const int warps_per_cta = kGemvThreads / 32;
  int64_t want = (p.rows_total + warps_per_cta - 1) / warps_per_cta;
  int64_t cap = (int64_t)num_sms * occ;
  int grid = (int)(want < cap ? want : cap);
  if (grid < 1) grid = 1;
  fn<<<grid, kGemvThreads, smem, s>>>(p);
  return cudaGetLastError();
}

}  // namespace lsw
