// tc_common.cuh -- PTX wrappers (mbarrier, TMA, bulk copies, tcgen05 MMA /
// commit / TMEM loads, UMMA descriptors), the switch's tile walk and the
// pre-swizzled operand packing; shared by the tensor-core switch
// (switch_tc_fc.cu) and the tensor-core prefill (prefill_tc.cu).  Internal.
#pragma once

#include <cuda.h>
#include <cudaTypedefs.h>

#include "lsw_internal.cuh"

namespace lsw {
namespace tcx {

// ------------------------------------------------------------------ PTX helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ bool mbar_try(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// Wait for the phase with parity `parity` to complete.  A watchdog traps after
// ~20 s so a protocol bug fails the launch instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  if (mbar_try(bar, parity)) return;
  const uint64_t t0 = globaltimer();
  uint32_t n = 0;
  while (!mbar_try(bar, parity)) {
    if ((++n & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) __trap();
  }
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1,
                                             int32_t c2, int32_t c3, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3, %4}], [%5], %6;"
      ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(src), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1,
                                             int32_t c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
      ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(src), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1-D bulk copy global -> shared, completion on an mbarrier (transaction bytes)
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                          uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(policy)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

// UMMA shared-memory descriptor (K-major, swizzled): start>>4 [0,14), LBO>>4
// [16,30) (unused for swizzled K-major; 1), SBO>>4 [32,46) = 8 rows * row
// bytes, version 1 at [46,48), layout type [61,64).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t sbo_bytes, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

__device__ __forceinline__ void umma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}"
      ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// the M-side operand from TMEM: a_tmem = [lane 0, column] of a [128, K] bf16
// operand, column c of a 16-wide K step = elements 2c (low half), 2c + 1
// (scripts/micro/tmem_a_rp_test.cu)
__device__ __forceinline__ void umma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}"
      ::"r"(d_tmem), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

// elect.sync: true in exactly one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// N consecutive 32-bit columns of this warp's 32 lanes (one register per column)
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t* r);
template <>
__device__ __forceinline__ void tmem_st<8>(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
template <>
__device__ __forceinline__ void tmem_st<16>(uint32_t taddr, const uint32_t* r) {
  tmem_st<8>(taddr, r);
  tmem_st<8>(taddr + 8, r + 8);
}
template <>
__device__ __forceinline__ void tmem_st<32>(uint32_t taddr, const uint32_t* r) {
  tmem_st<16>(taddr, r);
  tmem_st<16>(taddr + 16, r + 16);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ------------------------------------------------------------------ fp32x2 / bf16 helpers

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ uint32_t f2_to_bf16x2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);     // RNE, lo -> low half
  return *reinterpret_cast<uint32_t*>(&b2);
}

// ------------------------------------------------------------------ tile walk

// Per-CTA tile sequence over the global (kind, layer, row block, column block)
// order: chunks of `chunk` consecutive tiles dealt round-robin to the CTAs, so a
// CTA walks along 128-row strips while all CTAs sweep ~one matrix at a time.
struct Cursor {
  int64_t t;             // global tile index, -1 when done
  int32_t kd, layer, rb, cb;
  int32_t left;          // tiles of the current chunk after this one (no per-tile division)
  int32_t k;             // dynamic chunks: ordinal of the current chunk in this CTA's walk
};

struct TileSeq {
  int64_t T, t0;         // T tiles of this launch, starting at global tile t0
  int32_t chunk, G, b;
  uint32_t wlo, whi;     // fused decode, adaptive split: this CTA's range bounds (2^-24 units of a segment)
  int32_t adapt;         // 0: uniform split
  // plain sweep, dynamic chunks (dyn): chunk n -> the CTA that claims it from
  // the device counter ctr (in claim order, so the CTAs still sweep about one
  // region at a time, and a faster SM takes more chunks); ring = this CTA's
  // shared [claimed, claimer, id[16]]: every role reads its k-th chunk from it
  int32_t dyn;
  uint32_t* ctr;
  int32_t* ring;
};

struct TileKinds {
  int64_t tile_begin[LSW_NKIND];
  int32_t row_tiles[LSW_NKIND], col_tiles[LSW_NKIND];
  int32_t n_layers;
};

__device__ __forceinline__ void cursor_set(const TileKinds& g, Cursor& c, int64_t t) {
  c.t = t;
  if (t < 0) return;
  int kd = 0;
  while (kd + 1 < LSW_NKIND && t >= g.tile_begin[kd + 1]) ++kd;
  int64_t local = t - g.tile_begin[kd];
  const int64_t per_layer = (int64_t)g.row_tiles[kd] * g.col_tiles[kd];
  c.kd = kd;
  c.layer = (int)(local / per_layer);
  local -= (int64_t)c.layer * per_layer;
  c.rb = (int)(local / g.col_tiles[kd]);
  c.cb = (int)(local - (int64_t)c.rb * g.col_tiles[kd]);
}

// start of chunk number n of the launch: its first tile and length
__device__ __forceinline__ void cursor_chunk(const TileKinds& g, const TileSeq& q, Cursor& c, int64_t n) {
  const int64_t r0 = n * q.chunk;
  if (n < 0 || r0 >= q.T) { c.t = -1; return; }
  const int64_t len = q.T - r0 < q.chunk ? q.T - r0 : q.chunk;
  cursor_set(g, c, q.t0 + r0);
  c.left = (int32_t)len - 1;
}

// dynamic chunks: the chunk of ordinal k of this CTA's walk (-1: none left).
// The first role of the CTA to need ordinal k claims it (election on
// ring[1]); the others wait for it (ring[0] > k).  Ring slot k & 15 is reused
// 16 chunks later -- the CTA's roles run within ~12 tiles of each other (their
// stage rings), and dyn needs chunks of >= 2 tiles.
__device__ __forceinline__ int64_t seq_claim(const TileSeq& q, int32_t k) {
  int32_t* claimed = q.ring;
  int32_t* claimer = q.ring + 1;
  volatile int32_t* ids = q.ring + 2;
  for (;;) {
    int32_t cl;
    asm volatile("ld.acquire.cta.b32 %0, [%1];" : "=r"(cl) : "l"(claimed) : "memory");
    if (cl > k) return ids[k & 15];
    if (atomicCAS(claimer, k, k + 1) == k) {
      const uint32_t id = atomicAdd(q.ctr, 1u);
      const int64_t n_chunks = (q.T + q.chunk - 1) / q.chunk;
      ids[k & 15] = (int64_t)id < n_chunks ? (int32_t)id : -1;
      asm volatile("st.release.cta.b32 [%0], %1;" ::"l"(claimed), "r"(k + 1) : "memory");
      return ids[k & 15];
    }
  }
}

__device__ __forceinline__ Cursor cursor_first(const TileKinds& g, const TileSeq& q) {
  Cursor c;
  c.k = 0;
  cursor_chunk(g, q, c, q.dyn ? seq_claim(q, 0) : q.b);
  return c;
}

__device__ __forceinline__ void cursor_next(const TileKinds& g, const TileSeq& q, Cursor& c) {
  if (c.left > 0) {
    --c.left;
    ++c.t;
    if (++c.cb == g.col_tiles[c.kd]) {
      c.cb = 0;
      if (++c.rb == g.row_tiles[c.kd]) {
        c.rb = 0;
        if (++c.layer == g.n_layers) { c.layer = 0; ++c.kd; }
      }
    }
    return;
  }
  if (q.dyn) {
    ++c.k;
    cursor_chunk(g, q, c, seq_claim(q, c.k));
  } else {
    cursor_chunk(g, q, c, (c.t - q.t0) / q.chunk + q.G);   // once per chunk
  }
}

__device__ __forceinline__ int64_t strip_id(const Cursor& c) { return c.t - c.cb; }

// ring position: stage index + phase bit, advanced without division
struct Ring {
  uint32_t i, phase, n;
  __device__ __forceinline__ void next() { if (++i == n) { i = 0; phase ^= 1u; } }
};

// ------------------------------------------------------------------ operand packing

// Pre-swizzled K-major operand image: element (row, k) of a [rows, rp] operand
// goes to 16-byte chunk (k/8) ^ f(row) of its row, f = the TMA/UMMA swizzle of
// row-byte width RB = 2*rp (32B: (row>>2)&1, 64B: (row>>1)&3, 128B: row&7), so
// a 1-D bulk copy of 128 rows to a 1 KB-aligned shared address reproduces what a
// swizzled TMA load would have written.  Rows >= n_rows and ranks >= r are 0.
__device__ __forceinline__ int64_t swz_off(int64_t row, int k, int rp) {
  const int rb = 2 * rp;
  const int f = (int)((row * rb / 128) & (rb / 16 - 1));
  return row * rp + (((k >> 3) ^ f) << 3) + (k & 7);
}

// A [L, N, r, d_in] -> A^T blocks [L, col_tiles, N, tc, rp] (tc = tile columns):
// block (l, cb) holds, expert after expert, the pre-swizzled [tc, rp] slice
// A_{l,e}^T[cb*tc : cb*tc + tc, :] (zero beyond d_in / r).
static __global__ void pack_At_kernel(const __nv_bfloat16* __restrict__ A, __nv_bfloat16* __restrict__ At,
                                      int64_t L, int N, int r, int rp, int64_t d_in, int64_t col_tiles, int tc) {
  const int64_t din_pad = col_tiles * tc;
  const int64_t total = L * N * din_pad * rp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % rp);
    const int64_t c = (i / rp) % din_pad;
    const int64_t m = i / ((int64_t)rp * din_pad);       // l * N + e
    const int64_t l = m / N, e = m % N;
    const __nv_bfloat16 v = (k < r && c < d_in) ? A[(m * r + k) * d_in + c] : __float2bfloat16(0.f);
    const int64_t blk = (l * col_tiles + c / tc) * N + e;
    At[blk * tc * rp + swz_off(c % tc, k, rp)] = v;
  }
}

// B [M, d_out, r] -> [M, dout_pad, rp]
static __global__ void pack_B_kernel(const __nv_bfloat16* __restrict__ B, __nv_bfloat16* __restrict__ Bp, int64_t M,
                                     int r, int rp, int64_t d_out, int64_t dout_pad) {
  const int64_t total = M * dout_pad * rp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(i % rp);
    const int64_t row = (i / rp) % dout_pad;
    const int64_t m = i / ((int64_t)rp * dout_pad);
    const __nv_bfloat16 v = (k < r && row < d_out) ? B[(m * d_out + row) * r + k] : __float2bfloat16(0.f);
    Bp[m * dout_pad * rp + swz_off(row, k, rp)] = v;
  }
}

}  // namespace tcx
}  // namespace lsw
