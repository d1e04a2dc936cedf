// switch_tc.cu -- K1-tc: the all-layer in-place switch on the 5th-gen tensor cores.
//
// What it computes (identical to K1-simt): for every adapted matrix m of every
// layer, in ONE persistent launch (SGMM Eq. 11; in place P:328):
//     W_m <- RNE( W_m + sum_j c_j * B_{m,e_j} @ A_{m,e_j} )
// with the Eq. 5/9/10 coefficient list (Eq. 9 sign corrected, R1; compacted,
// lsw_internal.cuh build_coefs).
//
// How:
//  * A W tile is 128 rows x (64*nsub) columns (nsub = 2 by default, i.e. 256 B
//    of each row per tile: B200's in-place read-modify-write stream loses ~20%
//    of its bandwidth at 128-B row segments, scripts/membench.cu).  It is loaded
//    by nsub 64-column TMA boxes (128B swizzle) into one ring stage, updated in
//    place in shared memory and written back by nsub TMA bulk tensor stores.
//    3-D tensor maps [L, d_out, d_in] zero-fill / clip ragged tiles and never
//    spill into the next layer.
//  * The tile sequence (kind, layer, row block, column block) is cut into chunks
//    of 32 consecutive tiles dealt round-robin to the persistent CTAs (grid =
//    #SMs): a CTA walks ALONG a 128-row strip within its chunk, so the strip's B
//    slices (UMMA operand A: 128 x r per expert, K-major) stay resident in
//    shared memory, while all CTAs together sweep one matrix at a time, so the
//    A slices (UMMA operand B: A^T, 64*nsub x r per expert, K-major), re-read by
//    every row strip, stay L2-resident.  Both come from ctx-owned copies packed
//    at create time PRE-SWIZZLED into the exact shared-memory image the UMMA
//    descriptors expect (B: one cp.async.bulk per slice; A: cp.async, below).
//  * One tcgen05.mma (kind::f16, bf16 in, fp32 accumulate, M=128, N=64, K=16)
//    per expert per 16 of r per 64-column sub-tile, each expert into ITS OWN
//    TMEM accumulator, double-buffered across sub-tiles: the gate coefficients
//    c_j are applied in fp32 in the epilogue (R13: exact fp32 coefficients, not
//    Eq. 5's bf16-rounded g*DOWN).
//  * Epilogue (8 warps, 2 per TMEM lane quarter): tcgen05.ld the accumulators,
//    W + sum_j c_j acc_j with packed fp32x2 FMAs (FFMA2), RNE to bf16, in place
//    in the (conflict-free, 128B-swizzled) stage.
//  * Warp roles: 0 = W producer (TMA), 1 = TMEM allocator + MMA issuer,
//    2 = store warp (TMA stores, frees W stages as soon as they are read),
//    3 = operand producer (B strips by bulk copy; per-tile A slices by cp.async
//    on the LSU path, so they do not queue behind W tiles in the TMA engine),
//    4..11 = epilogue.
//    W prefetch depth is therefore set by the W ring alone, not by the
//    operand ring that the MMA releases.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "lsw_internal.cuh"
#include "switch_tc_impl.cuh"

// This file is compiled twice: as lsw::v1 (the switch kernel) and, from
// switch_tc_fused.cu with LSW_TC_FUSED=1, as lsw::v1f (the same kernel with the
// fused switch + decode epilogue).  Keeping the fused code out of
// the plain build leaves the switch kernel's code generation untouched
// (measured: one binary with both epilogues made the switch 4-12 % slower).
#ifndef LSW_TC_FUSED
#define LSW_TC_FUSED 0
#endif

namespace lsw {
#if LSW_TC_FUSED
namespace v1f {
#else
namespace v1 {
#endif

constexpr int kTcTM = 128;                 // tile rows = UMMA M = TMEM lanes
constexpr int kTcTN = 64;                  // sub-tile columns = UMMA N
constexpr int kSubBytes = kTcTM * kTcTN * 2;   // 16 KB: one swizzled W sub-tile
constexpr int kTcEpiWarps = 8;
constexpr int kTcFirstEpiWarp = 4;
constexpr int kTcThreads = 32 * (kTcFirstEpiWarp + kTcEpiWarps);
constexpr int kTcMaxStages = 8;
constexpr int kTcMaxAccBufs = 4;           // TMEM accumulator buffers (mbarrier pairs)

enum { ORDER_STRIP = 0, ORDER_SWEEP = 1 };

struct TcMaps {
  CUtensorMap w[LSW_NKIND];   // W [L, d_out, d_in], box {64, 128, 1}, 128B swizzle
  CUtensorMap p[LSW_NKIND];   // pristine copies (RESTORE source), same geometry
};

struct TcKind {
  int64_t tile_begin;
  int32_t row_tiles, col_tiles;
  __nv_bfloat16* W;           // [L, d_out, d_in] (written back by the epilogue in STG mode)
  int64_t d_out, d_in;
  int64_t din_pad, dout_pad;  // packed-operand row counts (multiples of 128)
  const __nv_bfloat16* At;    // packed A^T [L, col_tiles, N, tile_cols, rp], pre-swizzled:
                              // one tile's slices of all N experts are one contiguous block
  const __nv_bfloat16* Bp;    // packed B   [L*N, dout_pad, rp], pre-swizzled
};

struct TcGeom {
  TcKind kind[LSW_NKIND];
  int64_t tiles_total;
  int32_t n_layers, n_experts, rp;        // rp: rank padded to a multiple of 16
  int32_t nsub;                           // 64-column sub-tiles per W tile (1 or 2)
  int32_t w_stages, a_stages, b_bufs, acc_bufs;
  int32_t max_terms;                      // 2k
  uint32_t tmem_cols;
  uint32_t a_bytes_per_term;              // 64*nsub * rp * 2
  uint32_t b_bytes_per_term;              // 128 * rp * 2
  uint32_t a_stage_bytes, b_buf_bytes, w_stage_bytes;
  int32_t a_all;                          // 1: one bulk op fetches all N experts' A slices of a tile
  int32_t split;                          // 1: "split mode" -- c_j*B_j folded into B as 3 bf16 parts
                                          //    (hi+mid+lo == the fp32 product), ONE accumulator per tile
                                          //    (N = tile width), one MMA group per tile, 4 TMEM buffers;
                                          // 0: one accumulator per expert term, c_j applied in the epilogue
  int32_t w4d;                            // 1: W moved by ONE 4-D TMA op per tile (LSW_TC_W4D)
  int32_t w_policy;                       // W loads/stores L2 policy: 0 evict_first, 1 evict_normal
  int32_t store_stg;                      // 1: epilogue writes W back with coalesced STG.128 (LSU);
                                          // 0: the store warp issues TMA bulk tensor stores
  uint32_t swz_mode;                      // UMMA layout type of the r-wide operands
  uint32_t smem_bytes;
};

// Fused switch + decode: tiles walked in decoder order, one
// segment per (layer, GEMV group); every tile's freshly rounded W also feeds
// y_seg += W_tile x_seg in the epilogue.  Segment s's epilogue work starts only
// after every tile of segment s-1 is done (its y final), as a decoder needs.
struct FusedSeg {
  int64_t tile_begin, tile_count;   // fused-order tiles of this segment
  int32_t layer, n_kinds;
  int32_t kinds[3];                 // kind ids in group order
  int32_t pad;
  int64_t x_off;                    // elements into xs of this segment's input
  int64_t y_off[3];                 // elements into ys of each kind's row 0
};

struct TcPlan {
  TcMaps maps;
  TcGeom geom;
  FusedSeg* d_segs = nullptr;       // fused mode: device table (tc_plan_set_fused)
  int32_t n_segs = 0;
  int64_t fused_tiles = 0;
  unsigned long long* d_seg_done = nullptr;
  // Tile order (measured, 7B shape, same run): strip 4.60-4.67 TB/s, sweep with
  // 32-tile chunks 5.02-5.03 TB/s.  With strip order the 148 CTAs work on ~148
  // different matrices, so the per-tile A^T slices (re-read once per row strip)
  // fall out of L2; the chunked sweep keeps all CTAs on ~one matrix.
  int32_t order = ORDER_SWEEP, chunk = 48, probe = 0;   // chunk 24/32/48/64: 5317/5183/5358/5286 GB/s
  uint64_t* trace = nullptr;  // LSW_TC_TRACE: [kTraceCtas][kTraceTiles][kTraceEvents] device timestamps
  void* packed_At[LSW_NKIND] = {};
  void* packed_B[LSW_NKIND] = {};
  int64_t bytes = 0;
  int grid = 0;
};

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

// Tuning trace (LSW_TC_TRACE): %globaltimer stamps of pipeline events for the
// first kTraceTiles tiles of kTraceCtas CTAs spread over the grid
// (CTA b is traced as slot b / kTraceStride when b % kTraceStride == 0),
// layout [slot][tile][event].
constexpr int kTraceTiles = 2048, kTraceEvents = 16, kTraceCtas = 4, kTraceStride = 49;
enum { EV_W_ISSUED = 0, EV_A_ISSUED, EV_A_FULL, EV_MMA_START, EV_MMA_DONE, EV_EPI_WFULL, EV_EPI_ACC0,
       EV_STAGE_FREE, EV_EPI_DONE, EV_MMA_ACC0, EV_MMA_ISSUED0, EV_EPI_SUB0_DONE };
__device__ __forceinline__ void trace_ev(uint64_t* tr, uint32_t it, int ev) {
  if (tr && blockIdx.x % kTraceStride == 0 && it < (uint32_t)kTraceTiles) {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    tr[((size_t)(blockIdx.x / kTraceStride) * kTraceTiles + it) * kTraceEvents + ev] = t;
  }
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

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int32_t c0, int32_t c1,
                                             int32_t c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group.L2::cache_hint [%0, {%1, %2, %3}], [%4], %5;"
      ::"l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(src), "l"(policy)
      : "memory");
}

// 4-D view [L, col block, d_out, 64] of W: ONE op moves a whole 128 x 128 tile
// (both 64-column sub-tiles, in the same smem order as two 3-D boxes)
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

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// elect.sync: true in exactly one lane of the (converged) warp
__device__ __forceinline__ bool elect_one() {
  uint32_t p;
  asm volatile("{\n .reg .pred P;\n elect.sync _|P, 0xffffffff;\n selp.u32 %0, 1, 0, P;\n}" : "=r"(p));
  return p != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// ------------------------------------------------------------------ tile walk

// Per-CTA tile sequence over the global (kind, layer, row block, column block)
// order.  ORDER_STRIP: one contiguous range per CTA.  ORDER_SWEEP (default,
// measured best): chunks of consecutive tiles dealt round-robin to the CTAs.
// ORDER_SWEEP: chunks of `chunk` consecutive tiles dealt round-robin.

struct Cursor {
  int64_t t;             // global tile index, -1 when done
  int32_t kd, layer, rb, cb;
#if LSW_TC_FUSED
  int32_t seg, kidx;     // fused order: segment and kind index within its group
#endif
};

struct TileSeq {
  int64_t T, t_begin, t_end;   // T tiles of this launch, starting at global tile t0
  int64_t t0;
  int32_t order, chunk, G, b;
#if LSW_TC_FUSED
  const FusedSeg* segs;        // fused (decoder) tile order
  int32_t n_seg;
#endif
};

#if LSW_TC_FUSED
// fused order: segment (binary search), then kind within the group, rb, cb
__device__ __forceinline__ void cursor_set_fused(const TcGeom& g, const TileSeq& q, Cursor& c, int64_t t) {
  c.t = t;
  if (t < 0) return;
  int lo = 0, hi = q.n_seg - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (q.segs[mid].tile_begin <= t) lo = mid; else hi = mid - 1;
  }
  const FusedSeg& S = q.segs[lo];
  int64_t off = t - S.tile_begin;
  int ki = 0, kd = S.kinds[0];
  for (; ki < S.n_kinds; ++ki) {
    kd = S.kinds[ki];
    const int64_t per = (int64_t)g.kind[kd].row_tiles * g.kind[kd].col_tiles;
    if (off < per) break;
    off -= per;
  }
  c.seg = lo;
  c.kidx = ki;
  c.kd = kd;
  c.layer = S.layer;
  c.rb = (int)(off / g.kind[kd].col_tiles);
  c.cb = (int)(off - (int64_t)c.rb * g.kind[kd].col_tiles);
}

__device__ __forceinline__ void cursor_step_fused(const TcGeom& g, const TileSeq& q, Cursor& c) {
  if (++c.cb == g.kind[c.kd].col_tiles) {
    c.cb = 0;
    if (++c.rb == g.kind[c.kd].row_tiles) {
      c.rb = 0;
      if (++c.kidx == q.segs[c.seg].n_kinds) {
        c.kidx = 0;
        ++c.seg;
        c.layer = q.segs[c.seg].layer;
      }
      c.kd = q.segs[c.seg].kinds[c.kidx];
    }
  }
}
#endif

__device__ __forceinline__ void cursor_set(const TcGeom& g, Cursor& c, int64_t t) {
  c.t = t;
  if (t < 0) return;
  int kd = 0;
  while (kd + 1 < LSW_NKIND && t >= g.kind[kd + 1].tile_begin) ++kd;
  const TcKind& k = g.kind[kd];
  int64_t local = t - k.tile_begin;
  const int64_t per_layer = (int64_t)k.row_tiles * k.col_tiles;
  c.kd = kd;
  c.layer = (int)(local / per_layer);
  local -= (int64_t)c.layer * per_layer;
  c.rb = (int)(local / k.col_tiles);
  c.cb = (int)(local - (int64_t)c.rb * k.col_tiles);
}

__device__ __forceinline__ Cursor cursor_first(const TcGeom& g, const TileSeq& q) {
  Cursor c;
  int64_t t = q.order == ORDER_STRIP ? (q.t_begin < q.t_end ? q.t_begin : -1)
                                     : ((int64_t)q.b * q.chunk < q.T ? (int64_t)q.b * q.chunk : -1);
#if LSW_TC_FUSED
  cursor_set_fused(g, q, c, t < 0 ? -1 : q.t0 + t);
#else
  cursor_set(g, c, t < 0 ? -1 : q.t0 + t);
#endif
  return c;
}

// Advance to the CTA's next tile: +1 inside a range/chunk (no division), a
// jump (one division) between sweep chunks.
__device__ __forceinline__ void cursor_next(const TcGeom& g, const TileSeq& q, Cursor& c) {
  const int64_t t1 = c.t + 1, r1 = t1 - q.t0;          // r: position within this launch's range
  const bool step = q.order == ORDER_STRIP ? (r1 < q.t_end) : (r1 % q.chunk != 0 && r1 < q.T);
#if LSW_TC_FUSED
  if (step) {
    c.t = t1;
    cursor_step_fused(g, q, c);
    return;
  }
#endif
  if (step) {
    c.t = t1;
    if (++c.cb == g.kind[c.kd].col_tiles) {
      c.cb = 0;
      if (++c.rb == g.kind[c.kd].row_tiles) {
        c.rb = 0;
        if (++c.layer == g.n_layers) { c.layer = 0; ++c.kd; }
      }
    }
    return;
  }
  if (q.order == ORDER_STRIP) { c.t = -1; return; }
  const int64_t nq = (c.t - q.t0) / q.chunk + q.G;
#if LSW_TC_FUSED
  cursor_set_fused(g, q, c, nq * q.chunk < q.T ? q.t0 + nq * q.chunk : -1);
#else
  cursor_set(g, c, nq * q.chunk < q.T ? q.t0 + nq * q.chunk : -1);
#endif
}

__device__ __forceinline__ int64_t strip_id(const Cursor& c) { return c.t - c.cb; }

// ring position: stage index + phase bit, advanced without division
struct Ring {
  uint32_t i, phase, n;
  __device__ __forceinline__ void next() { if (++i == n) { i = 0; phase ^= 1u; } }
};

// ------------------------------------------------------------------ epilogue math

__device__ __forceinline__ uint64_t f2_pack(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint32_t f2_to_bf16x2(uint64_t v) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
  __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);     // RNE, lo -> low half
  return *reinterpret_cast<uint32_t*>(&b2);
}

// One 16-column chunk of one row: W (two swizzled 16-B smem chunks) <-
// RNE(W + sum_j c_j acc_j), with the sum in fp32 pairs (FFMA2), W as the first
// addend.  NT = number of accumulators (compile-time).
template <int NT>
__device__ __forceinline__ void epi_chunk(uint32_t tm_addr, const uint64_t* c2, uint8_t* wrow, int row, int col16) {
  uint32_t acc[NT][16];
#pragma unroll
  for (int j = 0; j < NT; ++j) tmem_ld16(tm_addr + j * kTcTN, acc[j]);
  uint4* p0 = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + 0) ^ (row & 7)) << 4));
  uint4* p1 = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + 1) ^ (row & 7)) << 4));
  const uint4 u0 = *p0, u1 = *p1;
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  tmem_wait_ld();
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    uint64_t v = f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u));
#pragma unroll
    for (int j = 0; j < NT; ++j)
      v = ffma2(f2_pack(__uint_as_float(acc[j][2 * q]), __uint_as_float(acc[j][2 * q + 1])), c2[j], v);
    o[q] = f2_to_bf16x2(v);
  }
  *p0 = make_uint4(o[0], o[1], o[2], o[3]);
  *p1 = make_uint4(o[4], o[5], o[6], o[7]);
}

#if LSW_TC_FUSED
// epi_chunk, then the GEMV on the stored (rounded) weights: ydot += this row's
// 16 new W values x x (16 bf16 in x16[0..1])
template <int NT>
__device__ __forceinline__ void epi_chunk_fused(uint32_t tm_addr, const uint64_t* c2, uint8_t* wrow, int row,
                                                int col16, const uint4* x16, float* ydot) {
  epi_chunk<NT>(tm_addr, c2, wrow, row, col16);
  const uint4 u0 = *reinterpret_cast<const uint4*>(wrow + (((col16 * 2 + 0) ^ (row & 7)) << 4));
  const uint4 u1 = *reinterpret_cast<const uint4*>(wrow + (((col16 * 2 + 1) ^ (row & 7)) << 4));
  const uint32_t o[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  const uint32_t xw[8] = {x16[0].x, x16[0].y, x16[0].z, x16[0].w, x16[1].x, x16[1].y, x16[1].z, x16[1].w};
  uint64_t a = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q)
    a = ffma2(f2_pack(__uint_as_float(o[q] << 16), __uint_as_float(o[q] & 0xffff0000u)),
              f2_pack(__uint_as_float(xw[q] << 16), __uint_as_float(xw[q] & 0xffff0000u)), a);
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  *ydot += lo + hi;
}
#endif

// General term count (> 4): groups of 4 accumulators.
__device__ __forceinline__ void epi_chunk_many(uint32_t tm_addr, const float* cs, int nt, uint8_t* wrow, int row,
                                               int col16) {
  uint4* p0 = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + 0) ^ (row & 7)) << 4));
  uint4* p1 = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + 1) ^ (row & 7)) << 4));
  const uint4 u0 = *p0, u1 = *p1;
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  uint64_t v[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u));
  for (int j0 = 0; j0 < nt; j0 += 4) {
    uint32_t acc[4][16];
    const int nj = nt - j0 < 4 ? nt - j0 : 4;
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (jj < nj) tmem_ld16(tm_addr + (j0 + jj) * kTcTN, acc[jj]);
    tmem_wait_ld();
#pragma unroll
    for (int jj = 0; jj < 4; ++jj)
      if (jj < nj) {
        const uint64_t c2 = f2_pack(cs[j0 + jj], cs[j0 + jj]);
#pragma unroll
        for (int q = 0; q < 8; ++q)
          v[q] = ffma2(f2_pack(__uint_as_float(acc[jj][2 * q]), __uint_as_float(acc[jj][2 * q + 1])), c2, v[q]);
      }
  }
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = f2_to_bf16x2(v[q]);
  *p0 = make_uint4(o[0], o[1], o[2], o[3]);
  *p1 = make_uint4(o[4], o[5], o[6], o[7]);
}

// ------------------------------------------------------------------ epilogue loop

struct TcArgs {
  TcGeom g;
  int32_t order, chunk, probe;
  uint64_t* trace;            // tuning: per-tile event timestamps of CTAs 0,1 (LSW_TC_TRACE), or null
  // coefficient inputs (same as SwitchParams)
  int32_t mode, top_k, n_experts;
  float scale;
  const int32_t* cur_idx;
  const float* cur_g;
  DevState* state;
  int64_t t0, t_count;        // tile range of this launch (t_count = 0: all tiles)
#if LSW_TC_FUSED
  const FusedSeg* segs;       // decoder-order segment table
  int32_t n_seg;
  const __nv_bfloat16* xs;    // packed GEMV inputs (lsw_decode_token layout)
  float* ys;                  // packed outputs, zeroed before the launch (accumulated)
  unsigned long long* seg_done;   // [n_seg], zeroed before the launch
#endif
};

struct EpiCtx {
  const TcGeom& g;
  uint8_t* wst0;
  uint32_t tmem_base;
  int warp, lane;
  bool probe;
  bool skip_math;
  uint64_t* bar_wfull;
  uint64_t* bar_wdone;
  uint64_t* bar_wempty;
  uint64_t* bar_accfull;
  uint64_t* bar_accempty;
  uint64_t* trace;
#if LSW_TC_FUSED
  const TcArgs* args;          // segs, xs, ys, seg_done
#endif
};

#if LSW_TC_FUSED
// Spin (with a ~20 s watchdog) until a device-wide counter reaches target.
__device__ __forceinline__ void wait_count(const unsigned long long* p, unsigned long long target) {
  auto load = [&]() {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
  };
  if (load() >= target) return;
  const uint64_t t0 = globaltimer();
  for (uint32_t n = 1; load() < target; ++n) {
    __nanosleep(64);
    if ((n & 1023u) == 0 && globaltimer() - t0 > 20000000000ull) __trap();
  }
}
#endif

// The epilogue warps' tile loop, specialised on the term count (NT = -1: any;
// NT = kSplitNT: split mode, one pre-scaled accumulator per tile).
constexpr int kSplitNT = 100;
template <int NT>
__device__ __forceinline__ void epilogue_loop(const EpiCtx& e, const TileSeq& seq, const Coefs& cf) {
  constexpr bool SPLIT = NT == kSplitNT;
  const TcGeom& g = e.g;
  const int ew = e.warp - kTcFirstEpiWarp;     // 0..7
  const int quarter = e.warp & 3;              // TMEM lane quarter this warp may access
  const int half = ew >> 2;                    // which 32 of a sub-tile's 64 columns
  const int row = quarter * 32 + e.lane;       // tile-local row == TMEM lane
  uint64_t c2[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) c2[j] = (!SPLIT && NT > j) ? f2_pack(cf.c[j], cf.c[j]) : 0ull;
  if (SPLIT) c2[0] = f2_pack(1.f, 1.f);        // W + acc (coefficients are already in the MMA)
  const int nt = cf.n;
  // per-term mode: one TMEM buffer (max_terms x 64 columns) per sub-tile;
  // split mode: one buffer (64*nsub columns) per tile
  const uint32_t buf_cols = SPLIT ? kTcTN * g.nsub : g.max_terms * kTcTN;
  Ring wring{0, 0, (uint32_t)g.w_stages};
  Ring acc{0, 0, (uint32_t)g.acc_bufs};
  uint64_t* tr = (ew == 0 && e.lane == 0) ? e.trace : nullptr;
  uint32_t it = 0;
#if LSW_TC_FUSED
  int cur_seg = -1;
  int64_t seg_mine = 0;                        // tiles of cur_seg this CTA finished
  const bool leader = ew == 0 && e.lane == 0;
#endif
  for (Cursor c = cursor_first(g, seq); c.t >= 0; cursor_next(g, seq, c), ++it) {
#if LSW_TC_FUSED
    float ydot = 0.f;                          // this thread's part of y[row] for the tile
    const __nv_bfloat16* xt;
    int64_t x_lim;
    {
      const TcArgs& A = *e.args;
      if (c.seg != cur_seg) {
        // decoder order: x of segment s is final only once every tile of
        // segment s-1 is done.  One thread per CTA publishes the CTA's count of
        // the segment it leaves (after all 8 epilogue warps issued their y
        // atomics) and waits for the previous segment's total (one counter
        // update per CTA and segment -- per tile and warp, the single hot
        // address serialised: 14.4 ms per 7B token instead of 8.4)
        named_bar(3, 32 * kTcEpiWarps);
        if (leader) {
          if (cur_seg >= 0) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(A.seg_done + cur_seg),
                         "l"((unsigned long long)seg_mine) : "memory");
          }
          if (c.seg > 0) wait_count(&A.seg_done[c.seg - 1], (unsigned long long)A.segs[c.seg - 1].tile_count);
        }
        named_bar(3, 32 * kTcEpiWarps);
        cur_seg = c.seg;
        seg_mine = 0;
      }
      const int64_t col0 = (int64_t)c.cb * kTcTN * g.nsub;
      xt = A.xs + A.segs[c.seg].x_off + col0;
      x_lim = g.kind[c.kd].d_in - col0;        // columns of this tile inside d_in
    }
#endif
    mbar_wait(smem_u32(&e.bar_wfull[wring.i]), wring.phase);            // W tile landed (acquire)
    trace_ev(tr, it, EV_EPI_WFULL);
    uint8_t* wt = e.wst0 + (size_t)wring.i * g.w_stage_bytes;
    for (int sb = 0; sb < g.nsub; ++sb) {
#if LSW_TC_FUSED
      uint4 xq[2][2];
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int cl = sb * kTcTN + (half * 2 + q2) * 16 + h * 8;     // 8 columns (16 B) of x
          xq[q2][h] = cl < x_lim ? *reinterpret_cast<const uint4*>(xt + cl) : make_uint4(0, 0, 0, 0);
        }
#endif
      if (!e.probe && (!SPLIT || sb == 0))
        mbar_wait(smem_u32(&e.bar_accfull[acc.i]), acc.phase);          // accumulators ready
      if (sb == 0) trace_ev(tr, it, EV_EPI_ACC0);
      tc_fence_after();
      uint8_t* wrow = wt + sb * kSubBytes + row * 128;
      const uint32_t tm_row = e.tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * buf_cols +
                              (SPLIT ? sb * kTcTN : 0);
#pragma unroll
      for (int q2 = 0; q2 < 2; ++q2) {
        const int col16 = half * 2 + q2;       // 16-column chunk 0..3 of the sub-tile
        const uint32_t ta = tm_row + col16 * 16;
#if LSW_TC_FUSED
        if constexpr (NT > 0 && !SPLIT) epi_chunk_fused<NT>(ta, c2, wrow, row, col16, xq[q2], &ydot);
#else
        if constexpr (SPLIT) { if (!e.skip_math) epi_chunk<1>(ta, c2, wrow, row, col16); }
        else if constexpr (NT > 0) epi_chunk<NT>(ta, c2, wrow, row, col16);
#endif
        else if constexpr (NT < 0) epi_chunk_many(ta, cf.c, nt, wrow, row, col16);
      }
      if (!SPLIT || sb == g.nsub - 1) {
        // accumulators consumed -> MMA may reuse this TMEM buffer
        tc_fence_before();
        __syncwarp();
        if (e.lane == 0 && !e.probe) mbar_arrive(smem_u32(&e.bar_accempty[acc.i]));
        acc.next();
      }
      if (sb == 0) trace_ev(tr, it, EV_EPI_SUB0_DONE);
    }
    if (g.store_stg) {
      // Copy-out through the LSU path, per warp (no cross-warp barrier): this
      // warp computed rows 32*quarter.. +31, columns 32*half.. +31 of every
      // sub-tile; re-read them from shared memory so that 4 lanes write one
      // row's 64 contiguous bytes (two full 32-B sectors) per STG.128.
      __syncwarp();
      const TcKind& K = g.kind[c.kd];
      const int64_t row0 = (int64_t)c.rb * kTcTM + quarter * 32, col0 = (int64_t)c.cb * kTcTN * g.nsub;
      __nv_bfloat16* Wl = K.W + (int64_t)c.layer * K.d_out * K.d_in;
      const int sub_r = e.lane >> 2, ch4 = e.lane & 3;   // 8 rows x 4 chunks per instruction
      for (int sb = 0; sb < g.nsub; ++sb) {
#pragma unroll
        for (int rr = 0; rr < 32; rr += 8) {
          const int r = quarter * 32 + rr + sub_r;       // tile-local row
          const int ch = half * 4 + ch4;                 // 16-B chunk within the 128-B sub-tile row
          const uint4 v = *reinterpret_cast<const uint4*>(wt + sb * kSubBytes + r * 128 + ((ch ^ (r & 7)) << 4));
          const int64_t gr = row0 + rr + sub_r, gc = col0 + sb * kTcTN + ch * 8;
          if (gr < K.d_out && gc < K.d_in) __stcs(reinterpret_cast<uint4*>(Wl + gr * K.d_in + gc), v);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (e.lane == 0) mbar_arrive(smem_u32(&e.bar_wempty[wring.i]));   // stage reusable
    } else {
      // generic-proxy smem writes -> visible to the TMA store (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (e.lane == 0) mbar_arrive(smem_u32(&e.bar_wdone[wring.i]));
    }
#if LSW_TC_FUSED
    {
      const TcArgs& A = *e.args;
      const int64_t grow = (int64_t)c.rb * kTcTM + row;
      if (grow < g.kind[c.kd].d_out) atomicAdd(A.ys + A.segs[c.seg].y_off[c.kidx] + grow, ydot);
      ++seg_mine;
    }
#endif
    trace_ev(tr, it, EV_EPI_DONE);
    wring.next();
  }
#if LSW_TC_FUSED
  if (cur_seg >= 0) {                          // publish the last segment this CTA worked on
    named_bar(3, 32 * kTcEpiWarps);
    if (leader) {
      __threadfence();
      asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(e.args->seg_done + cur_seg),
                   "l"((unsigned long long)seg_mine) : "memory");
    }
  }
#endif
}

// ------------------------------------------------------------------ the kernel


__global__ void __launch_bounds__(kTcThreads, 1)
switch_tc_kernel(const __grid_constant__ TcMaps maps, const __grid_constant__ TcArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ Coefs cf;
  __shared__ int32_t s_parity;
  __shared__ uint32_t s_tmem_base;
  __shared__ __align__(8) uint64_t bar_wfull[kTcMaxStages], bar_wempty[kTcMaxStages], bar_wdone[kTcMaxStages];
  __shared__ __align__(8) uint64_t bar_afull[4], bar_aempty[4];
  __shared__ __align__(8) uint64_t bar_bfull[2], bar_bempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[kTcMaxAccBufs], bar_accempty[kTcMaxAccBufs];

  const TcGeom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // shared layout (1 KB aligned): [w_stages x W tile][a_stages x A slices][b_bufs x B strip slices]
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* wst0 = base;
  uint8_t* ast0 = wst0 + (size_t)g.w_stages * g.w_stage_bytes;
  uint8_t* bst0 = ast0 + (size_t)g.a_stages * g.a_stage_bytes;

  if (threadIdx.x == 0) {
    SwitchParams p{};
    p.mode = args.mode;
    p.top_k = args.top_k;
    p.n_experts = args.n_experts;
    p.scale = args.scale;
    p.cur_idx = args.cur_idx;
    p.cur_g = args.cur_g;
    p.state = args.state;
    const int32_t parity = *(volatile int32_t*)&args.state->parity;
    s_parity = parity;
    build_coefs(p, parity, cf);
    if (blockIdx.x == 0 && !cf.bad) stage_decision(p, parity);
    for (int s = 0; s < g.w_stages; ++s) {
      mbar_init(smem_u32(&bar_wfull[s]), 1);
      mbar_init(smem_u32(&bar_wempty[s]), g.store_stg ? kTcEpiWarps : 1);
      mbar_init(smem_u32(&bar_wdone[s]), kTcEpiWarps);
    }
    for (int s = 0; s < g.a_stages; ++s) {
      mbar_init(smem_u32(&bar_afull[s]), 32);             // one arrival per operand-warp lane
      mbar_init(smem_u32(&bar_aempty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&bar_bfull[s]), 1);
      mbar_init(smem_u32(&bar_bempty[s]), 1);
    }
    for (int s = 0; s < g.acc_bufs; ++s) {
      mbar_init(smem_u32(&bar_accfull[s]), 1);
      mbar_init(smem_u32(&bar_accempty[s]), kTcEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0)
    for (int k = 0; k < LSW_NKIND; ++k) prefetch_map(args.mode == MODE_RESTORE ? &maps.p[k] : &maps.w[k]);
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&s_tmem_base)), "r"(g.tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const int nt = cf.bad ? 0 : cf.n;
  // Tuning-only diagnostic levels (results are NOT the switch; never default):
  //   probe=1: W stream only (no slices, no MMA, epilogue writes W back);
  //   probe=2: full pipeline but the epilogue skips the TMEM reads / math.
  const bool probe = args.probe == 1;
  const bool skip_math = args.probe == 2;
  const int nsub = g.nsub;
  TileSeq seq;
  seq.T = args.t_count > 0 ? args.t_count : g.tiles_total;   // ablation: one matrix per launch
  seq.t0 = args.t0;
  seq.order = args.order;
  seq.chunk = args.chunk < 1 ? 1 : args.chunk;
  seq.G = gridDim.x;
  seq.b = blockIdx.x;
  seq.t_begin = seq.T * blockIdx.x / gridDim.x;
  seq.t_end = seq.T * (blockIdx.x + 1) / gridDim.x;
#if LSW_TC_FUSED
  seq.segs = args.segs;
  seq.n_seg = args.n_seg;
#endif
  const uint32_t tmem_base = s_tmem_base;
  const int tile_cols = kTcTN * nsub;

  if (nt > 0) {
    if (warp == 0) {
      // ============================ W producer =============================
      if (lane == 0) {
        const uint64_t pol_stream = g.w_policy ? policy_evict_normal() : policy_evict_first();
        const bool restore = args.mode == MODE_RESTORE;      // load from the pristine copy
        Ring wring{0, 0, (uint32_t)g.w_stages};
        uint32_t it = 0;
        for (Cursor c = cursor_first(g, seq); c.t >= 0; cursor_next(g, seq, c), ++it) {
          mbar_wait(smem_u32(&bar_wempty[wring.i]), wring.phase ^ 1);
          const uint32_t wbar = smem_u32(&bar_wfull[wring.i]);
          mbar_expect_tx(wbar, nsub * kSubBytes);
          uint8_t* wdst = wst0 + (size_t)wring.i * g.w_stage_bytes;
          if (g.w4d)
            tma_load_4d(smem_u32(wdst), restore ? &maps.p[c.kd] : &maps.w[c.kd], 0, c.rb * kTcTM, c.cb * nsub,
                        c.layer, wbar, pol_stream);
          else
            for (int sb = 0; sb < nsub; ++sb)
              tma_load_3d(smem_u32(wdst + sb * kSubBytes), restore ? &maps.p[c.kd] : &maps.w[c.kd],
                          c.cb * tile_cols + sb * kTcTN, c.rb * kTcTM, c.layer, wbar, pol_stream);
          trace_ev(args.trace, it, EV_W_ISSUED);
          wring.next();
        }
      }
    } else if (warp == 3) {
      // ============================ operand producer ========================
      if (!probe) {
        const uint64_t pol_keep = policy_evict_last();
        int64_t strip_prev = -1;
        Ring bring{0, 0, (uint32_t)g.b_bufs};
        Ring aring{0, 0, (uint32_t)g.a_stages};
        const size_t rpe = (size_t)g.rp;                   // elements per packed row
        uint64_t* tr = lane == 0 ? args.trace : nullptr;
        uint32_t it = 0;
        for (Cursor c = cursor_first(g, seq); c.t >= 0; cursor_next(g, seq, c), ++it) {
          const TcKind& K = g.kind[c.kd];
          if (strip_id(c) != strip_prev && g.split) {
            // Split mode: B slices of a new 128-row strip, scaled by their fp32
            // coefficient and split exactly into hi + mid + lo bf16 parts
            // (v = fl32(c_j b); hi = rne(v); mid = rne(v - hi); lo = v - hi - mid),
            // written at the same (pre-swizzled) positions of 3 part arrays.
            if (strip_prev >= 0) bring.next();
            strip_prev = strip_id(c);
            mbar_wait(smem_u32(&bar_bempty[bring.i]), bring.phase ^ 1);   // MMAs of the old strip done
            uint8_t* dst = bst0 + (size_t)bring.i * g.b_buf_bytes;
            const uint32_t chunks = g.b_bytes_per_term / 16;
            for (int j = 0; j < nt; ++j) {
              const uint4* src = reinterpret_cast<const uint4*>(
                  K.Bp + (((size_t)c.layer * g.n_experts + cf.e[j]) * K.dout_pad + (size_t)c.rb * kTcTM) * rpe);
              const float cj = cf.c[j];
              uint8_t* p0 = dst + (size_t)(3 * j + 0) * g.b_bytes_per_term;
              for (uint32_t q = lane; q < chunks; q += 32) {
                const uint4 u = __ldg(src + q);
                const uint32_t w[4] = {u.x, u.y, u.z, u.w};
                uint32_t hi[4], mid[4], lo[4];
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                  float v[2] = {__uint_as_float(w[i] << 16) * cj, __uint_as_float(w[i] & 0xffff0000u) * cj};
                  __nv_bfloat162 h = __floats2bfloat162_rn(v[0], v[1]);
                  const float r0 = v[0] - __low2float(h), r1 = v[1] - __high2float(h);
                  __nv_bfloat162 m = __floats2bfloat162_rn(r0, r1);
                  __nv_bfloat162 l = __floats2bfloat162_rn(r0 - __low2float(m), r1 - __high2float(m));
                  hi[i] = *reinterpret_cast<uint32_t*>(&h);
                  mid[i] = *reinterpret_cast<uint32_t*>(&m);
                  lo[i] = *reinterpret_cast<uint32_t*>(&l);
                }
                reinterpret_cast<uint4*>(p0)[q] = make_uint4(hi[0], hi[1], hi[2], hi[3]);
                reinterpret_cast<uint4*>(p0 + g.b_bytes_per_term)[q] = make_uint4(mid[0], mid[1], mid[2], mid[3]);
                reinterpret_cast<uint4*>(p0 + 2 * g.b_bytes_per_term)[q] = make_uint4(lo[0], lo[1], lo[2], lo[3]);
              }
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> MMA (async)
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_bfull[bring.i]));
          } else if (strip_id(c) != strip_prev) {          // B slices of a new 128-row strip (bulk, rare)
            if (strip_prev >= 0) bring.next();
            strip_prev = strip_id(c);
            if (lane == 0) {
              mbar_wait(smem_u32(&bar_bempty[bring.i]), bring.phase ^ 1);
              const uint32_t bar = smem_u32(&bar_bfull[bring.i]);
              mbar_expect_tx(bar, nt * g.b_bytes_per_term);
              uint8_t* dst = bst0 + (size_t)bring.i * g.b_buf_bytes;
              for (int j = 0; j < nt; ++j) {
                const __nv_bfloat16* src =
                    K.Bp + (((size_t)c.layer * g.n_experts + cf.e[j]) * K.dout_pad + (size_t)c.rb * kTcTM) * rpe;
                bulk_load(smem_u32(dst + j * g.b_bytes_per_term), src, g.b_bytes_per_term, bar, pol_keep);
              }
            }
            __syncwarp();
          }
          // A^T slices of this tile's columns, through the LSU (cp.async, 16 B per
          // lane) rather than the TMA engine: 4-KB bulk ops would queue behind
          // the W tiles already in the SM's TMA queue and arrive microseconds late.
          mbar_wait(smem_u32(&bar_aempty[aring.i]), aring.phase ^ 1);
          uint8_t* adst = ast0 + (size_t)aring.i * g.a_stage_bytes;
          const __nv_bfloat16* blk =
              K.At + (((size_t)c.layer * K.col_tiles + c.cb) * g.n_experts) * (size_t)tile_cols * rpe;
          for (int j = 0; j < nt; ++j) {
            const uint8_t* src = reinterpret_cast<const uint8_t*>(blk + (size_t)cf.e[j] * tile_cols * rpe);
            const uint32_t dst = smem_u32(adst + j * g.a_bytes_per_term);
            for (uint32_t off = lane * 16; off < g.a_bytes_per_term; off += 32 * 16)
              asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;"
                           ::"r"(dst + off), "l"(src + off), "l"(pol_keep) : "memory");
          }
          // the A stage's mbarrier tracks these copies asynchronously (one
          // arrival per lane when its copies land); the MMA thread issues the
          // generic->async proxy fence after its wait
          asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar_afull[aring.i]))
                       : "memory");
          trace_ev(tr, it, EV_A_ISSUED);
          aring.next();
        }
      }
    } else if (warp == 1) {
      // ============================ MMA issuer ==============================
      // The whole warp runs the loop (all values warp-uniform, so operands stay
      // in uniform registers); one elected lane issues each tcgen05 instruction.
      if (!probe) {
        // instruction descriptor: D f32, A/B bf16, both K-major, N = 64, M = 128
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcTN >> 3) << 17) |
                               ((uint32_t)(kTcTM >> 4) << 24);
        const uint32_t row_bytes = g.rp * 2;
        const uint32_t sbo = 8 * row_bytes;
        const int ksteps = g.rp / 16;
        // smem descriptors advance linearly with the start address (>> 4, no carry
        // out of the 14-bit field: addresses < 256 KB)
        const uint64_t desc0 = umma_desc(0, sbo, g.swz_mode);
        const uint64_t b_term = g.b_bytes_per_term >> 4, a_term = g.a_bytes_per_term >> 4;
        uint64_t* tr = lane == 0 ? args.trace : nullptr;
        Ring bring{0, 0, (uint32_t)g.b_bufs};
        Ring aring{0, 0, (uint32_t)g.a_stages};
        Ring acc{0, 0, (uint32_t)g.acc_bufs};
        Cursor c = cursor_first(g, seq);
        int64_t strip_prev = -1;
        uint32_t it = 0;
        while (c.t >= 0) {
          const int64_t strip = strip_id(c);
          if (strip != strip_prev) {
            if (strip_prev >= 0) bring.next();
            strip_prev = strip;
            mbar_wait(smem_u32(&bar_bfull[bring.i]), bring.phase);
          }
          mbar_wait(smem_u32(&bar_afull[aring.i]), aring.phase);
          // A slices were written by cp.async (generic proxy); order them before
          // the tensor core's (async-proxy) operand reads
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          trace_ev(tr, it, EV_MMA_START);
          const uint64_t a_desc = desc0 + (smem_u32(ast0 + (size_t)aring.i * g.a_stage_bytes) >> 4);
          const uint64_t b_desc = desc0 + (smem_u32(bst0 + (size_t)bring.i * g.b_buf_bytes) >> 4);
          if (g.split) {
            // ONE group per tile: N = 64*nsub columns, all terms x 3 parts into one accumulator
            mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
            trace_ev(tr, it, EV_MMA_ACC0);
            tc_fence_after();
            const uint32_t idesc_t = (idesc & ~(0x3Fu << 17)) | ((uint32_t)((kTcTN * nsub) >> 3) << 17);
            const uint32_t d = tmem_base + acc.i * (kTcTN * nsub);
            if (elect_one()) {
              uint32_t accum = 0;
              for (int j = 0; j < nt; ++j)
                for (int p = 0; p < 3; ++p)
                  for (int kk = 0; kk < ksteps; ++kk) {
                    umma_f16(d, b_desc + (3 * j + p) * b_term + kk * 2, a_desc + j * a_term + kk * 2, idesc_t, accum);
                    accum = 1;
                  }
              umma_commit(smem_u32(&bar_accfull[acc.i]));
            }
            __syncwarp();
            trace_ev(tr, it, EV_MMA_ISSUED0);
            acc.next();
          }
          for (int sb = 0; sb < nsub && !g.split; ++sb) {
            mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
            if (sb == 0) trace_ev(tr, it, EV_MMA_ACC0);
            tc_fence_after();
            const uint32_t d0 = tmem_base + acc.i * g.max_terms * kTcTN;
            const uint64_t a_sub = a_desc + ((sb * kTcTN * row_bytes) >> 4);
            if (elect_one()) {
              for (int j = 0; j < nt; ++j)
                for (int kk = 0; kk < ksteps; ++kk)
                  umma_f16(d0 + j * kTcTN, b_desc + j * b_term + kk * 2, a_sub + j * a_term + kk * 2, idesc,
                           kk > 0 ? 1u : 0u);
              umma_commit(smem_u32(&bar_accfull[acc.i]));
            }
            __syncwarp();
            if (sb == 0) trace_ev(tr, it, EV_MMA_ISSUED0);
            acc.next();
          }
          // B strip no longer needed once this CTA's next tile is in another strip
          cursor_next(g, seq, c);
          const bool strip_ends = c.t < 0 || strip_id(c) != strip;
          if (elect_one()) {
            umma_commit(smem_u32(&bar_aempty[aring.i]));     // A slices consumed
            if (strip_ends) umma_commit(smem_u32(&bar_bempty[bring.i]));
          }
          __syncwarp();
          trace_ev(tr, it, EV_MMA_DONE);
          ++it;
          aring.next();
        }
      }
    } else if (warp == 2 && !g.store_stg) {
      // ============================ store warp ==============================
      if (lane == 0) {
        const uint64_t pol_stream = g.w_policy ? policy_evict_normal() : policy_evict_first();
        Ring wring{0, 0, (uint32_t)g.w_stages};
        uint32_t it = 0;
        for (Cursor c = cursor_first(g, seq); c.t >= 0; cursor_next(g, seq, c), ++it) {
          mbar_wait(smem_u32(&bar_wdone[wring.i]), wring.phase);     // epilogue wrote the tile
          uint8_t* wsrc = wst0 + (size_t)wring.i * g.w_stage_bytes;
          if (g.w4d)
            tma_store_4d(&maps.w[c.kd], smem_u32(wsrc), 0, c.rb * kTcTM, c.cb * nsub, c.layer, pol_stream);
          else
            for (int sb = 0; sb < nsub; ++sb)
              tma_store_3d(&maps.w[c.kd], smem_u32(wsrc + sb * kSubBytes), c.cb * tile_cols + sb * kTcTN,
                           c.rb * kTcTM, c.layer, pol_stream);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read -> stage reusable
          mbar_arrive(smem_u32(&bar_wempty[wring.i]));
          trace_ev(args.trace, it, EV_STAGE_FREE);
          wring.next();
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    } else if (warp >= kTcFirstEpiWarp) {
      // ============================ epilogue ================================
      const int ntc = (probe || skip_math) ? 0 : nt;
      EpiCtx ec{g, wst0, tmem_base, warp, lane, probe, skip_math, bar_wfull, bar_wdone, bar_wempty, bar_accfull,
                bar_accempty, args.trace
#if LSW_TC_FUSED
                , &args
#endif
      };
      // split mode always runs the split loop (its TMEM buffer protocol differs);
      // with probe/skip_math it only skips the math
      switch (g.split && nt > 0 && !probe ? kSplitNT : ntc) {
        case kSplitNT: epilogue_loop<kSplitNT>(ec, seq, cf); break;
        case 0: epilogue_loop<0>(ec, seq, cf); break;
        case 1: epilogue_loop<1>(ec, seq, cf); break;
        case 2: epilogue_loop<2>(ec, seq, cf); break;
        case 3: epilogue_loop<3>(ec, seq, cf); break;
        case 4: epilogue_loop<4>(ec, seq, cf); break;
        default: epilogue_loop<-1>(ec, seq, cf); break;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(g.tmem_cols)
                 : "memory");
  }
  if (threadIdx.x == 0) {
    SwitchParams p{};
    p.mode = args.mode;
    p.state = args.state;
    finish_pass(p, s_parity, cf);
  }
}

#if LSW_TC_FUSED
// ------------------------------------------------------------------ fused launcher (v1f)

// Launch the fused kernel with the plain build's plan data (v1 and v1f TcMaps /
// TcGeom are the same source, hence the same layout).
cudaError_t launch_fused_raw(const void* maps, const void* geom, int grid, uint32_t smem, int32_t order_chunk,
                             const SwitchParams& p, cudaStream_t s, const void* segs, int32_t n_seg, int64_t tiles,
                             const void* xs, float* ys, unsigned long long* seg_done, uint64_t* trace) {
  static uint32_t smem_set = 0;
  if (smem > smem_set) {
    cudaError_t e = cudaFuncSetAttribute(switch_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    smem_set = smem;
  }
  TcArgs a;
  a.g = *reinterpret_cast<const TcGeom*>(geom);
  a.order = ORDER_SWEEP;
  a.chunk = order_chunk;
  a.probe = 0;
  a.trace = trace;
  a.mode = p.mode;
  a.top_k = p.top_k;
  a.n_experts = p.n_experts;
  a.scale = p.scale;
  a.cur_idx = p.cur_idx;
  a.cur_g = p.cur_g;
  a.state = p.state;
  a.t0 = 0;
  a.t_count = tiles;
  a.segs = reinterpret_cast<const FusedSeg*>(segs);
  a.n_seg = n_seg;
  a.xs = reinterpret_cast<const __nv_bfloat16*>(xs);
  a.ys = ys;
  a.seg_done = seg_done;
  switch_tc_kernel<<<grid, kTcThreads, smem, s>>>(*reinterpret_cast<const TcMaps*>(maps), a);
  return cudaGetLastError();
}

#else   // the plain build: packing, planning, launches

// ------------------------------------------------------------------ packing

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
__global__ void pack_At_kernel(const __nv_bfloat16* __restrict__ A, __nv_bfloat16* __restrict__ At, int64_t L,
                               int N, int r, int rp, int64_t d_in, int64_t col_tiles, int tc) {
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
__global__ void pack_B_kernel(const __nv_bfloat16* __restrict__ B, __nv_bfloat16* __restrict__ Bp, int64_t M,
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

// ------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 4-D view (w4d): dims {64, d_out, d_in / 64, L}, box {64, 128, nsub, 1} -- one
// TMA op per W tile.  Needs d_in % 64 == 0.
// tuning knob LSW_TC_L2PROMO = 0 (none) / 64 / 128 / 256 (default) bytes
static CUtensorMapL2promotion l2_promotion() {
  const char* v = getenv("LSW_TC_L2PROMO");
  const int x = v ? atoi(v) : 256;
  return x == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE : x == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
         : x == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

static bool encode_w4(CUtensorMap* m, const void* base, uint64_t d_in, uint64_t d_out, uint64_t L, int nsub) {
  auto enc = get_encode();
  if (!enc || d_in % 64) return false;
  cuuint64_t dims[4] = {64, d_out, d_in / 64, L};
  cuuint64_t strides[3] = {d_in * 2, 128, d_in * d_out * 2};
  cuuint32_t box[4] = {(cuuint32_t)kTcTN, (cuuint32_t)kTcTM, (cuuint32_t)nsub, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool encode_w(CUtensorMap* m, const void* base, uint64_t d_in, uint64_t d_out, uint64_t L) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d_in, d_out, L};
  cuuint64_t strides[2] = {d_in * 2, d_in * d_out * 2};
  cuuint32_t box[3] = {(cuuint32_t)kTcTN, (cuuint32_t)kTcTM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, l2_promotion(),
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static uint32_t align1k(uint32_t x) { return (x + 1023) & ~1023u; }

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& sp, int num_sms, const char** why, bool strict) {
  *out = nullptr;
  int dev = 0, major = 0, minor = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) { *why = "needs an sm_100 (B200) device"; return cudaErrorNotSupported; }
  // r padded with zeros to a K-major row of 32, 64 or 128 bytes (one swizzle
  // atom width: SW32 / SW64 / SW128); e.g. r = 48 runs as 64
  const int r = sp.rank, rp = r <= 16 ? 16 : r <= 32 ? 32 : 64;
  if (rp > 64) { *why = "rank > 64"; return cudaErrorNotSupported; }
  TcPlan* plan = new TcPlan();
  TcGeom& g = plan->geom;
  memset(&g, 0, sizeof(g));
  g.n_layers = sp.n_layers;
  g.n_experts = sp.n_experts;
  g.rp = rp;
  g.max_terms = 2 * sp.top_k;
  g.swz_mode = rp == 16 ? 6u : rp == 32 ? 4u : 2u;        // SWIZZLE_32B / 64B / 128B (UMMA encoding)
  // Shared-memory / TMEM plan.  Candidates in order of preference:
  //   split mode, 128-column tiles (one accumulator of 128 columns per tile, 4 TMEM
  //     buffers; B strip holds 3 parts per term, single-buffered);
  //   per-term mode, 128-column tiles (max_terms x 64 TMEM columns per sub-tile);
  //   per-term mode, 64-column tiles.
  // Each needs >= 2 A stages and enough W stages (4 for 128-column tiles).
  const uint32_t budget = 227 * 1024 - 1024 /*align*/ - 2048 /*static*/;
  g.b_bytes_per_term = kTcTM * rp * 2;
  bool ok = false;
  int nsub_env = 0, split_env = -1;
  if (const char* v = getenv("LSW_TC_NSUB")) nsub_env = atoi(v);
  if (const char* v = getenv("LSW_TC_SPLIT")) split_env = atoi(v);
  int a_max = 3;                                         // A-slice ring depth (tuning: LSW_TC_ASTAGES)
  if (const char* v = getenv("LSW_TC_ASTAGES")) { int x = atoi(v); if (x >= 1 && x <= 4) a_max = x; }
  // measured (scripts/tune_switch.py, 7B shape): per-term 4583 GB/s vs split 3756 GB/s --
  // split mode triples the MMAs and the SS operand reads; it is opt-in (LSW_TC_SPLIT=1)
  if (split_env < 0) split_env = 0;
  for (int cand = 0; cand < 3 && !ok; ++cand) {
    const int split = cand == 0 ? 1 : 0;
    const int nsub = cand < 2 ? 2 : 1;
    if (nsub_env && nsub != nsub_env) continue;
    if (split_env >= 0 && split != split_env) continue;
    // TMEM
    const uint32_t buf_cols = split ? kTcTN * nsub : (uint32_t)g.max_terms * kTcTN;
    if (buf_cols > 512) continue;
    const int acc_bufs = split ? (int)(512 / buf_cols < 4 ? 512 / buf_cols : 4) : (buf_cols * 2 <= 512 ? 2 : 1);
    // shared memory
    const uint32_t a_term = kTcTN * nsub * rp * 2;
    const uint32_t a_stage = align1k(g.max_terms * a_term);
    const uint32_t b_buf = align1k(g.max_terms * (split ? 3 : 1) * g.b_bytes_per_term);
    const uint32_t w_stage = nsub * kSubBytes;
    for (int bbufs = split ? 1 : 2; bbufs >= 1 && !ok; --bbufs)
      for (int astages = a_max; astages >= 2 && !ok; --astages) {
        int ws = (int)((budget - (int64_t)bbufs * b_buf - (int64_t)astages * a_stage) / w_stage);
        if ((int64_t)budget < (int64_t)bbufs * b_buf + (int64_t)astages * a_stage) ws = 0;
        if (ws > kTcMaxStages) ws = kTcMaxStages;
        int min_ws = nsub == 2 ? 4 : 2;
        if (split)
          if (const char* v = getenv("LSW_TC_SPLIT_MINWS")) { int x = atoi(v); if (x >= 2 && x <= 4) min_ws = x; }
        if (ws >= min_ws) {
          ok = true;
          g.split = split;
          g.nsub = nsub;
          g.w_stages = ws;
          g.a_stages = astages;
          g.b_bufs = bbufs;
          g.acc_bufs = acc_bufs;
          g.a_bytes_per_term = a_term;
          g.a_stage_bytes = a_stage;
          g.a_all = 0;
          g.b_buf_bytes = b_buf;
          g.w_stage_bytes = w_stage;
          uint32_t cols = 32;
          while (cols < buf_cols * acc_bufs) cols <<= 1;
          g.tmem_cols = cols;
        }
      }
  }
  if (!ok) { delete plan; *why = "shared memory / TMEM: rank * top_k too large"; return cudaErrorNotSupported; }
  if (strict && (g.split || g.nsub != 2 || g.acc_bufs < 2)) {
    // degraded plan: the term-group kernel (switch_tc_tg.cu) serves this shape
    delete plan;
    *why = "v1: no double-buffered 128-column plan";
    return cudaErrorNotSupported;
  }
  // tuning knobs (defaults are the measured best)
  if (const char* v = getenv("LSW_TC_STAGES")) { int x = atoi(v); if (x >= 2 && x < g.w_stages) g.w_stages = x; }
  if (const char* v = getenv("LSW_TC_ORDER")) plan->order = strcmp(v, "sweep") == 0 ? ORDER_SWEEP : ORDER_STRIP;
  if (const char* v = getenv("LSW_TC_CHUNK")) { int x = atoi(v); if (x >= 1) plan->chunk = x; }
  if (const char* v = getenv("LSW_TC_PROBE")) plan->probe = atoi(v);
  if (getenv("LSW_TC_TRACE")) {
    const size_t tb = sizeof(uint64_t) * kTraceCtas * kTraceTiles * kTraceEvents;
    if (cudaMalloc(&plan->trace, tb) == cudaSuccess) cudaMemset(plan->trace, 0, tb);
    else plan->trace = nullptr;
  }
  g.w4d = 0;
  if (const char* v = getenv("LSW_TC_W4D")) g.w4d = atoi(v) != 0;
  g.w_policy = 0;
  if (const char* v = getenv("LSW_TC_WPOLICY")) g.w_policy = strcmp(v, "normal") == 0;
  for (int k = 0; k < LSW_NKIND; ++k) if (sp.kind[k].d_in % 64) g.w4d = 0;
  if (g.nsub != 2 || g.split) g.w4d = 0;
  g.store_stg = 0;                                       // measured: TMA store 4466 vs STG 4222 GB/s
  if (const char* v = getenv("LSW_TC_STORE")) g.store_stg = strcmp(v, "stg") == 0;
  // tuning probe (W stream only): all of shared memory as W stages
  if (plan->probe == 1 && getenv("LSW_TC_PROBE_WSTAGES")) {
    const int x = atoi(getenv("LSW_TC_PROBE_WSTAGES"));
    if (x >= 2 && x <= kTcMaxStages) { g.w_stages = x; g.a_stages = 0; g.b_bufs = 0; }
  }
  g.smem_bytes = g.w_stages * g.w_stage_bytes + g.a_stages * g.a_stage_bytes + g.b_bufs * g.b_buf_bytes + 1024;
  // tiles
  const int tile_cols = kTcTN * g.nsub;
  int64_t t = 0;
  for (int k = 0; k < LSW_NKIND; ++k) {
    const KindGeom& kg = sp.kind[k];
    g.kind[k].row_tiles = (int32_t)((kg.d_out + kTcTM - 1) / kTcTM);
    g.kind[k].col_tiles = (int32_t)((kg.d_in + tile_cols - 1) / tile_cols);
    g.kind[k].din_pad = (int64_t)g.kind[k].col_tiles * tile_cols;
    g.kind[k].dout_pad = (int64_t)g.kind[k].row_tiles * kTcTM;
    g.kind[k].tile_begin = t;
    t += (int64_t)sp.n_layers * g.kind[k].row_tiles * g.kind[k].col_tiles;
  }
  g.tiles_total = t;
  plan->grid = (int)(t < num_sms ? t : num_sms);
  // testing knob: fewer CTAs -> many tiles per CTA even for small shapes (ring wrap-around)
  if (const char* v = getenv("LSW_TC_GRID")) { int x = atoi(v); if (x >= 1 && x < plan->grid) plan->grid = x; }
  if (plan->grid < 1) plan->grid = 1;
  // pack operands + encode maps
  const int64_t M = (int64_t)sp.n_layers * sp.n_experts;
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < LSW_NKIND && e == cudaSuccess; ++k) {
    const KindGeom& kg = sp.kind[k];
    const size_t at_bytes = (size_t)M * g.kind[k].din_pad * rp * 2;
    const size_t b_bytes = (size_t)M * g.kind[k].dout_pad * rp * 2;
    e = cudaMalloc(&plan->packed_At[k], at_bytes);
    if (e != cudaSuccess) break;
    e = cudaMalloc(&plan->packed_B[k], b_bytes);
    if (e != cudaSuccess) break;
    plan->bytes += at_bytes + b_bytes;
    pack_At_kernel<<<2048, 256>>>((const __nv_bfloat16*)kg.A, (__nv_bfloat16*)plan->packed_At[k], sp.n_layers,
                                  sp.n_experts, r, rp, kg.d_in, g.kind[k].col_tiles, tile_cols);
    pack_B_kernel<<<2048, 256>>>((const __nv_bfloat16*)kg.B, (__nv_bfloat16*)plan->packed_B[k], M, r, rp,
                                 kg.d_out, g.kind[k].dout_pad);
    g.kind[k].At = (const __nv_bfloat16*)plan->packed_At[k];
    g.kind[k].Bp = (const __nv_bfloat16*)plan->packed_B[k];
    g.kind[k].W = (__nv_bfloat16*)kg.W;
    g.kind[k].d_out = kg.d_out;
    g.kind[k].d_in = kg.d_in;
    if (!(g.w4d ? encode_w4(&plan->maps.w[k], kg.W, kg.d_in, kg.d_out, sp.n_layers, g.nsub)
                : encode_w(&plan->maps.w[k], kg.W, kg.d_in, kg.d_out, sp.n_layers))) {
      *why = "cuTensorMapEncodeTiled failed";
      e = cudaErrorInvalidValue;
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(switch_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem_bytes);
  if (e != cudaSuccess) {
    if (!*why || !**why) *why = cudaGetErrorString(e);
    tc_plan_destroy(plan);
    return e;
  }
  *out = plan;
  return cudaSuccess;
}

void tc_plan_destroy(TcPlan* plan) {
  if (!plan) return;
  cudaFree(plan->d_segs);
  cudaFree(plan->d_seg_done);
  for (int k = 0; k < LSW_NKIND; ++k) {
    cudaFree(plan->packed_At[k]);
    cudaFree(plan->packed_B[k]);
  }
  cudaFree(plan->trace);
  delete plan;
}

int64_t tc_plan_bytes(const TcPlan* plan) { return plan ? plan->bytes : 0; }
int tc_plan_grid(const TcPlan* plan) { return plan ? plan->grid : 0; }
int tc_plan_tile_n(const TcPlan* plan) { return plan ? kTcTN * plan->geom.nsub : 0; }
int64_t tc_plan_tiles(const TcPlan* plan) { return plan ? plan->geom.tiles_total : 0; }

int64_t tc_plan_trace(const TcPlan* plan, uint64_t* host, int64_t n) {
  if (!plan || !plan->trace) return 0;
  const int64_t total = (int64_t)kTraceCtas * kTraceTiles * kTraceEvents;
  if (n > total) n = total;
  if (cudaMemcpy(host, plan->trace, n * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess) return 0;
  return n;
}

cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& sp) {
  for (int k = 0; k < LSW_NKIND; ++k)
    if (!sp.kind[k].P ||
        !(plan->geom.w4d ? encode_w4(&plan->maps.p[k], sp.kind[k].P, sp.kind[k].d_in, sp.kind[k].d_out, sp.n_layers,
                                     plan->geom.nsub)
                         : encode_w(&plan->maps.p[k], sp.kind[k].P, sp.kind[k].d_in, sp.kind[k].d_out, sp.n_layers)))
      return cudaErrorInvalidValue;
  return cudaSuccess;
}

int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0) {
  const TcKind& k = plan->geom.kind[kind];
  const int64_t per = (int64_t)k.row_tiles * k.col_tiles;
  *t0 = k.tile_begin + (int64_t)layer * per;
  return per;
}

cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0,
                             int64_t t_count) {
  TcArgs a;
  a.t0 = t0;
  a.t_count = t_count;
  a.g = plan->geom;
  a.order = plan->order;
  a.chunk = plan->chunk;
  a.probe = plan->probe;
  a.trace = plan->trace;
  a.mode = p.mode;
  a.top_k = p.top_k;
  a.n_experts = p.n_experts;
  a.scale = p.scale;
  a.cur_idx = p.cur_idx;
  a.cur_g = p.cur_g;
  a.state = p.state;
  switch_tc_kernel<<<plan->grid, kTcThreads, plan->geom.smem_bytes, s>>>(plan->maps, a);
  return cudaGetLastError();
}

// ------------------------------------------------------------------ fused switch + decode (host)

cudaError_t tc_plan_set_fused(TcPlan* plan, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]) {
  const TcGeom& g = plan->geom;
  if (g.split || g.max_terms > 4) return cudaErrorNotSupported;
  const int n = 4 * n_layers;
  FusedSeg* h = new FusedSeg[n];
  int64_t t = 0;
  for (int l = 0; l < n_layers; ++l)
    for (int gi = 0; gi < 4; ++gi) {
      FusedSeg& S = h[l * 4 + gi];
      memset(&S, 0, sizeof(S));
      S.tile_begin = t;
      S.layer = l;
      S.n_kinds = nk[gi];
      S.x_off = l * x_per_layer + x_off[gi];
      int64_t yo = l * y_per_layer + y_off[gi];
      for (int i = 0; i < nk[gi]; ++i) {
        const int kd = kinds[gi][i];
        S.kinds[i] = kd;
        S.y_off[i] = yo;
        yo += g.kind[kd].d_out;
        S.tile_count += (int64_t)g.kind[kd].row_tiles * g.kind[kd].col_tiles;
      }
      t += S.tile_count;
    }
  cudaError_t e = cudaSuccess;
  if (!plan->d_segs) e = cudaMalloc(&plan->d_segs, sizeof(FusedSeg) * n);
  if (e == cudaSuccess && !plan->d_seg_done) e = cudaMalloc(&plan->d_seg_done, sizeof(unsigned long long) * n);
  if (e == cudaSuccess) e = cudaMemcpy(plan->d_segs, h, sizeof(FusedSeg) * n, cudaMemcpyHostToDevice);
  delete[] h;
  if (e != cudaSuccess) return e;
  plan->n_segs = n;
  plan->fused_tiles = t;
  return cudaSuccess;
}

cudaError_t launch_switch_tc_fused(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, const void* xs,
                                   float* ys) {
  if (!plan->d_segs) return cudaErrorNotSupported;
  cudaError_t e = cudaMemsetAsync(plan->d_seg_done, 0, sizeof(unsigned long long) * plan->n_segs, s);
  if (e != cudaSuccess) return e;
  // segment barriers: a CTA's share of one segment is a few tiles, so deal
  // small chunks (measured 7B: chunk 4-8 8.4 ms, 1 12.6, 16 10.7, 32 22.8)
  int chunk = 8;
  if (const char* v = getenv("LSW_TC_FUSED_CHUNK")) { int x = atoi(v); if (x >= 1) chunk = x; }
  return v1f::launch_fused_raw(&plan->maps, &plan->geom, plan->grid, plan->geom.smem_bytes, chunk, p, s,
                               plan->d_segs, plan->n_segs, plan->fused_tiles, xs, ys, plan->d_seg_done,
                               plan->trace);
}

#endif  // LSW_TC_FUSED

}  // namespace v1 / v1f
}  // namespace lsw
