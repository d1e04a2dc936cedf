// switch_tc_fc.cu -- K1-tc: the all-layer in-place switch on the 5th-gen
// tensor cores (SURVEY a-3 / a-4; the bf16 switch of every ctx).
//
// What it computes (identical to K1-simt): for every adapted matrix m of every
// layer, in ONE persistent launch (SGMM Eq. 11; "a single CUDA
// kernel operation" P:240; in place P:328):
//     W_m <- RNE( W_m + sum_j c_j * B_{m,e_j} @ A_{m,e_j} )
// with the Eq. 5/9/10 coefficient list (Eq. 9 sign corrected, R1; compacted,
// lsw_internal.cuh build_coefs).
//
// Fold mode (the default): Eq. 5 concatenates the
// selected experts along the rank dimension and folds the gate into one
// factor, so the whole update of a tile is ONE contraction of depth sum_j r_j.
// Folding c_j into a bf16 factor would round it (R13), so each folded factor is
// stored as an exact-to-2^-16 pair of bf16 parts, hi_j = bf16(c_j B_j) and
// lo_j = bf16(c_j B_j - hi_j), and the tile is
//     D = sum_j (hi_j + lo_j) @ A_j          (K = 2 * sum_j rp)
// accumulated in fp32 in ONE TMEM buffer by one chain of tcgen05.mma (M = 128,
// N = 128) and ONE commit per tile (a commit drains the tensor pipe: commits,
// not MMA work, pace the MMA warp).  The epilogue only adds D to W and rounds
// once.  Per-term modes (large k * r): raw B, one fp32 TMEM accumulator per
// term, the epilogue's running sum W + sum_j c_j acc_j in FFMA2.
//  * The fold runs once per 128-row strip (B slices are reused along the
//    strip): the operand warp bulk-copies the raw pre-swizzled B slices into
//    the strip buffer and rewrites them in place as (hi, lo) parts; the
//    element positions of the swizzled image do not change.
//  * W tiles 128 x 128 (one 4-D row-major TMA box, or two 64-column 128B-swizzled
//    3-D boxes for ragged shards), TMA loads (warp 0), TMA bulk stores (warp 2),
//    chunked sweep tile order; the fused switch + decode walks decoder order.
#include <cstdlib>
#include <cstring>

#include "switch_tc_impl.cuh"
#include "tc_common.cuh"

namespace lsw {
namespace fc {

using namespace tcx;

constexpr int kTM = 128;                    // tile rows = UMMA M = TMEM lanes
constexpr int kTN = 128;                    // tile columns = UMMA N = accumulator columns
constexpr int kSubCols = 64;                // W sub-tile columns (one 128B-swizzle TMA box)
constexpr int kSubBytes = kTM * kSubCols * 2;   // 16 KB
constexpr int kEpiWarps = 8;
constexpr int kFirstEpiWarp = 4;
constexpr int kThreads = 32 * (kFirstEpiWarp + kEpiWarps);
constexpr int kMaxStages = 8;
constexpr int kMaxAStages = 8;
constexpr int kAccBufs = 4;                 // 4 x 128 columns = all of TMEM
constexpr int kPtGroup = 2;                 // per-term mode: terms per MMA group / TMEM buffer

struct Maps {
  CUtensorMap w[LSW_NKIND];   // W [L, d_out, d_in], box {64, 128, 1}, 128B swizzle
  CUtensorMap p[LSW_NKIND];   // pristine copies (RESTORE source), same geometry
  CUtensorMap at[LSW_NKIND];  // pair mode: packed A^T as [L*col_tiles*N*128, rp] (pre-swizzled), box {rp, 64}
};

struct Geom {
  TileKinds tk;
  const __nv_bfloat16* At[LSW_NKIND];   // packed A^T [L, col_tiles, N, 128, rp], pre-swizzled
  const __nv_bfloat16* Bp[LSW_NKIND];   // packed B   [L*N, dout_pad, rp], pre-swizzled
  int64_t dout_pad[LSW_NKIND];
  int64_t d_in[LSW_NKIND], d_out[LSW_NKIND];
  int64_t tiles_total;
  int32_t n_experts, rp;
  int32_t w_stages, a_stages, b_bufs;
  uint32_t term_bytes;                  // one term's 128 x rp operand slice (A^T of a tile, or B of a strip)
  uint32_t a_stage_bytes, b_buf_bytes;  // A stage: all terms of one tile; B buffer: (hi, lo) of all terms
  uint32_t swz_mode;                    // UMMA layout type of the r-wide operands
  uint32_t smem_bytes;
  int32_t wrm;                          // 1: W tile moved row-major by one 4-D TMA op (256 B per row
                                        //    contiguous in smem and in the request stream; LSW_FC_WRM)
  int32_t pt;                           // 1: per-term mode (no fold): each term its own fp32 TMEM
                                        //    accumulator of 128 columns, kPtGroup terms per commit
  int32_t acc_bufs;                     // TMEM accumulator buffers of acc_cols columns
  uint32_t acc_cols;
  int32_t pair;                         // fold mode on CTA pairs (cta_group::2, M = 256): each CTA of a
                                        //   cluster of 2 owns one of two vertically adjacent tiles and loads
                                        //   HALF of the A^T columns; the leader issues the pair's MMAs
  TileKinds tkp;                        // pair geometry: row tiles = pairs of 128-row tiles
  int64_t tiles_pair;
  int32_t bu;                           // per-term mode with the B slices staged per unit (next to
                                        //    the unit's A^T slices) instead of per strip: the plan
                                        //    when a whole strip of 2k raw B slices does not fit
                                        //    (r = 64, k = 4: 128 KB)
  int32_t tb;                           // fold mode with the (hi, lo) B strip in TMEM (the MMA's M-side
                                        //    operand read from TMEM): the epilogue warps fold each strip
                                        //    from a raw shared-memory copy straight into one of b_bufs
                                        //    TMEM buffers of bcols columns at b_col0; A^T slices staged
                                        //    in units of unit_terms terms
  int32_t unit_terms;
  int32_t unit_commit;                  // tb: each A unit freed by its own MMA commit (default), else
                                        //    by the epilogue with its tile
  uint32_t bcols, b_col0, raw_bytes;
};

// Fused switch + decode: one segment per (layer, GEMV group),
// tiles walked in decoder order; the epilogue also accumulates
// y_seg += RNE(W_new) x_seg from the freshly rounded tile.
struct FusedSeg {
  int64_t tile_begin, tile_count;   // fused-order tiles of this segment
  int32_t layer, n_kinds;
  int32_t kinds[3];                 // kind ids in group order
  int32_t pad;
  int64_t x_off;                    // elements into xs of this segment's input
  int64_t y_off[3];                 // elements into ys of each kind's row 0
  int64_t y_rows;                   // rows of the segment's outputs (ys[y_off[0] ..+ y_rows])
};

struct TcPlan {
  Maps maps;
  Geom geom;
  FusedSeg* d_segs = nullptr;       // fused mode (tc_plan_set_fused)
  unsigned long long* d_seg_done = nullptr;
  unsigned long long* d_ys_fx = nullptr;   // fixed-point output accumulators (2^-40), [ys_rows]
  int64_t ys_rows = 0;
  int32_t n_segs = 0;
  int64_t fused_tiles = 0;
  int32_t chunk = 48;
  int32_t probe = 0;          // tuning builds only (tc_probe=1): W stream alone, W written back unchanged
  int32_t fused_probe = 0;    // tuning builds only (fc_fused_probe)
  int32_t fused_adapt = 1;    // option fc_adapt: adaptive split of the fused decode's segments
  int32_t fw_stages = 0, fa_stages = 0, fb_bufs = 0;   // the fused decode's shared-memory plan (W 3 first)
  uint32_t fsmem_bytes = 0;
  int32_t sweep_dyn = 1;      // option fc_dyn: plain sweep's chunks claimed dynamically
  uint32_t* trace = nullptr;  // tuning builds only (trace_buf: device buffer of kTraceCtas * kTraceTiles * 8 u32)
  uint32_t* seg_trace = nullptr;  // tuning builds only (seg_trace_buf: grid * 512 * 2 u32)
  void* packed_At[LSW_NKIND] = {};
  void* packed_B[LSW_NKIND] = {};
  int64_t bytes = 0;
  int grid = 0;
  int pair_grid = 0;          // CTA-pair launches (geom.pair): an even grid
};

struct Args {
  Geom g;
  int32_t chunk, probe;
  int32_t mode, top_k, n_experts;
  float scale;
  const int32_t* cur_idx;
  const float* cur_g;
  DevState* state;
  int64_t t0, t_count;        // tile range of this launch (t_count = 0: all tiles)
  // fused switch + decode only
  const FusedSeg* segs;
  int32_t n_seg;
  const __nv_bfloat16* xs;
  float* ys;
  unsigned long long* ys_fx;      // fixed-point accumulators of ys, zeroed before the launch
  unsigned long long* seg_done;   // [n_seg], zeroed before the launch
  uint32_t* trace;                // tuning builds only (option trace_buf): per-tile role timestamps
  uint32_t* seg_trace;            // tuning builds only (option seg_trace_buf): [CTA][segment][2] publish / wait-done
  int32_t adapt;                  // fused: adaptive split of the segments (DevState fused_w)
  int32_t dyn;                    // plain sweep: chunks claimed from a device counter
};

// Tuning builds only: %globaltimer (low 32 bits, ns) of pipeline events for the
// first kTraceTiles tiles of CTAs 0 .. kTraceCtas-1 (the whole pass at the BASELINE shapes), slot = role event:
// 0 W load issued, 1 A stage issued, 2 MMA saw its operands, 3 MMA committed,
// 4 epilogue saw the accumulator, 5 epilogue saw W, 6 tile handed to the store,
// 7 store has read the stage.
constexpr int kTraceCtas = 2, kTraceTiles = 8192;
#ifdef LSW_TUNING
#define FC_TRACE(slot, n)                                                                                 \
  do {                                                                                                    \
    const int n_ = (n);                                                                                   \
    if (args.trace && blockIdx.x < kTraceCtas && n_ < kTraceTiles)                                        \
      args.trace[((size_t)blockIdx.x * kTraceTiles + n_) * 8 + (slot)] = (uint32_t)globaltimer();        \
  } while (0)
#define FC_SEG_TRACE(seg, which)                                                                          \
  do {                                                                                                    \
    if (args.seg_trace && (seg) < 512)                                                                    \
      args.seg_trace[((size_t)blockIdx.x * 512 + (seg)) * 2 + (which)] = (uint32_t)globaltimer();        \
  } while (0)
#else
#define FC_TRACE(slot, n) do {} while (0)
#define FC_SEG_TRACE(seg, which) do {} while (0)
#endif

// Fused outputs are accumulated in 64-bit fixed point (2^-40 units): integer
// adds are associative, so y is bitwise reproducible whatever the order of the
// per-tile contributions (fp32 atomics are not); converted to fp32 once a
// segment is complete.  |y| < 2^23 (R24: non-finite inputs are undefined).
constexpr double kFx = 1099511627776.0;          // 2^40
constexpr double kFxInv = 1.0 / 1099511627776.0;

// Convert this CTA's slice of segment q's outputs (all epilogue threads).
__device__ __forceinline__ void fx_convert(const Args& a, int q, int t, int nthr) {
  const FusedSeg& S = a.segs[q];
  const int64_t r0 = S.y_off[0] + S.y_rows * blockIdx.x / gridDim.x;
  const int64_t r1 = S.y_off[0] + S.y_rows * (blockIdx.x + 1) / gridDim.x;
  for (int64_t r = r0 + t; r < r1; r += nthr)
    a.ys[r] = (float)((double)(long long)__ldcg(a.ys_fx + r) * kFxInv);
}

// ------------------------------------------------------------------ tile walk

// The plain pass walks tcx's (kind, layer, rb, cb) order in chunks dealt
// round-robin over the CTAs; the fused pass the decoder order: segment (layer,
// group), kind within the group, rb, cb.
struct FCursor : Cursor {
  int32_t seg, kidx;
  int64_t end;        // fused: end (exclusive) of this CTA's range in segment seg
  int64_t x_off;      // fused: xs offset of the segment's input
  int64_t y_base;     // fused: ys offset of the current kind's row 0
};

// fused order: CTA b takes, in every segment s (T_s tiles), the contiguous
// range [T_s * b / G, T_s * (b + 1) / G) -- every CTA finishes each segment at
// about the same time, so the decoder-order barrier between segments waits
// for ~one tile of imbalance, not for a whole chunk of another CTA.  The
// segment's constants are read once per segment into the cursor (not per tile).
__device__ __forceinline__ void fused_at(const TileKinds& g, const Args& a, FCursor& c, int seg, int64_t t,
                                         int64_t end) {
  const FusedSeg& S = a.segs[seg];
  int64_t off = t - S.tile_begin;
  int ki = 0, kd = S.kinds[0];
  for (; ki < S.n_kinds; ++ki) {
    kd = S.kinds[ki];
    const int64_t per = (int64_t)g.row_tiles[kd] * g.col_tiles[kd];
    if (off < per) break;
    off -= per;
  }
  c.t = t;
  c.seg = seg;
  c.kidx = ki;
  c.kd = kd;
  c.layer = S.layer;
  c.rb = (int)(off / g.col_tiles[kd]);
  c.cb = (int)(off - (int64_t)c.rb * g.col_tiles[kd]);
  c.end = end;
  c.x_off = S.x_off;
  c.y_base = S.y_off[ki];
}

// this CTA's first tile in segment >= seg (t = -1: none left)
__device__ __forceinline__ void fused_from(const TileKinds& g, const TileSeq& q, const Args& a, FCursor& c, int seg) {
  for (; seg < a.n_seg; ++seg) {
    const FusedSeg& S = a.segs[seg];
    // uniform, or the adaptive split: boundaries from the cumulative weights
    // (the same value bounds both neighbours: the ranges tile the segment)
    const int64_t lo = q.adapt ? (int64_t)(((uint64_t)S.tile_count * q.wlo) >> 24) : S.tile_count * q.b / q.G;
    const int64_t hi = q.adapt ? (int64_t)(((uint64_t)S.tile_count * q.whi) >> 24) : S.tile_count * (q.b + 1) / q.G;
    if (lo < hi) { fused_at(g, a, c, seg, S.tile_begin + lo, S.tile_begin + hi); return; }
  }
  c.t = -1;
}

template <bool kF>
__device__ __forceinline__ FCursor cur_first(const TileKinds& g, const TileSeq& q, const Args& a) {
  FCursor c;
  if constexpr (kF) {
    fused_from(g, q, a, c, 0);
  } else {
    static_cast<Cursor&>(c) = cursor_first(g, q);
  }
  return c;
}

template <bool kF>
__device__ __forceinline__ void cur_next(const TileKinds& g, const TileSeq& q, const Args& a, FCursor& c) {
  if constexpr (kF) {
    if (c.t + 1 < c.end) {
      ++c.t;
      if (++c.cb == g.col_tiles[c.kd]) {
        c.cb = 0;
        if (++c.rb == g.row_tiles[c.kd]) {
          c.rb = 0;
          ++c.kidx;
          const FusedSeg& S = a.segs[c.seg];
          c.kd = S.kinds[c.kidx];
          c.y_base = S.y_off[c.kidx];
        }
      }
      return;
    }
    fused_from(g, q, a, c, c.seg + 1);
  } else {
    cursor_next(g, q, static_cast<Cursor&>(c));
  }
}

// c -> the first tile of the next strip of this CTA's walk (t = -1: none)
template <bool kF>
__device__ __forceinline__ void strip_advance(const TileKinds& g, const TileSeq& q, const Args& a, FCursor& c) {
  const int64_t s = strip_id(c);
  do cur_next<kF>(g, q, a, c); while (c.t >= 0 && strip_id(c) == s);
}

__device__ __forceinline__ void wait_count(const unsigned long long* p, unsigned long long target) {
  unsigned long long v;
  const uint64_t t0 = globaltimer();
  for (;;) {
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (v >= target) return;
    __nanosleep(64);
    if (globaltimer() - t0 > 20000000000ull) __trap();
  }
}

// ------------------------------------------------------------------ fold

__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// Eight bf16 B elements -> (hi, lo) parts of c * b: x = fl32(c * b),
// hi = RNE_bf16(x), lo = RNE_bf16(x - hi) (x - hi is exact in fp32), so
// hi + lo = x to within 2^-16 |x| (R13: the coefficient is not rounded to bf16).
__device__ __forceinline__ void fold8(const uint4 raw, float c, uint4& hi, uint4& lo) {
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t h[4], l[4];
  const uint64_t c2 = f2_pack(c, c), m1 = f2_pack(-1.f, -1.f), z2 = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // x = c * b (packed, exact product rounded once), hi = RNE(x), lo = RNE(x - hi)
    const uint64_t x = ffma2(f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u)), c2, z2);
    h[q] = f2_to_bf16x2(x);
    const uint64_t hf = f2_pack(__uint_as_float(h[q] << 16), __uint_as_float(h[q] & 0xffff0000u));
    l[q] = f2_to_bf16x2(ffma2(hf, m1, x));
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

// Fold the strip buffer at dst in place (raw B in the lo slots -> hi, lo), the
// 16-B vectors [v0, v1) of every term, by the 32 lanes of one warp.
__device__ __forceinline__ void fold_range(uint8_t* dst, uint32_t tb, int nt, const float* c, uint32_t v0,
                                           uint32_t v1, int lane) {
  for (int j = 0; j < nt; ++j) {
    const float cj = c[j];
    uint4* phi = reinterpret_cast<uint4*>(dst + 2 * j * tb);
    uint4* plo = reinterpret_cast<uint4*>(dst + (2 * j + 1) * tb);
#pragma unroll 4
    for (uint32_t v = v0 + lane; v < v1; v += 32) {
      uint4 hi, lo;
      fold8(plo[v], cj, hi, lo);
      phi[v] = hi;
      plo[v] = lo;
    }
  }
}

// TMEM fold (tb mode): this thread's row of one raw B slice (the pre-swizzled
// [128, RP] image in shared memory) -> (hi, lo) parts of c * b written to the
// row's TMEM lane, hi at columns [taddr, taddr + RP/2), lo at the next RP/2
// (column c of a 16-wide K step = elements 2c, 2c + 1: the MMA's M-side layout).
template <int RP>
__device__ __forceinline__ void fold_row_tmem(const uint8_t* slice, int row, float c, uint32_t taddr) {
  constexpr int kChunks = RP / 8;   // 16-B chunks per row
  const int f = RP == 16 ? (row >> 2) & 1 : RP == 32 ? (row >> 1) & 3 : row & 7;   // swz_off's phase
  uint32_t h[RP / 2], l[RP / 2];
#pragma unroll
  for (int ch = 0; ch < kChunks; ++ch) {
    const uint4 raw = *reinterpret_cast<const uint4*>(slice + row * (2 * RP) + ((ch ^ f) << 4));
    uint4 hi, lo;
    fold8(raw, c, hi, lo);
    h[4 * ch] = hi.x; h[4 * ch + 1] = hi.y; h[4 * ch + 2] = hi.z; h[4 * ch + 3] = hi.w;
    l[4 * ch] = lo.x; l[4 * ch + 1] = lo.y; l[4 * ch + 2] = lo.z; l[4 * ch + 3] = lo.w;
  }
  tmem_st<RP / 2>(taddr, h);
  tmem_st<RP / 2>(taddr + RP / 2, l);
}

// ------------------------------------------------------------------ epilogue

// W (bf16, one 128-B swizzle unit: 64 columns of a row) + 16 accumulator
// columns -> RNE in place; key = the unit's swizzle phase (unit index & 7).
// flip: this lane touches the odd 16-B chunk of the pair first -- with the
// row-major tile (units 2r + h, keys 2r + h mod 8) lanes r and r + 4 share a
// key, and flipping the order for r & 4 keeps every 8 lanes of one LDS/STS.128
// on 8 distinct bank groups.
__device__ __forceinline__ void epi16(uint8_t* wrow, int key, int flip, int col16, const uint32_t* acc) {
  uint4* pa = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + flip) ^ key) << 4));
  uint4* pb = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + (flip ^ 1)) ^ key) << 4));
  const uint4 ua = *pa, ub = *pb;
  const uint4 u0 = flip ? ub : ua, u1 = flip ? ua : ub;
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint64_t v = fadd2(f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u)),
                             f2_pack(__uint_as_float(acc[2 * q]), __uint_as_float(acc[2 * q + 1])));
    o[q] = f2_to_bf16x2(v);
  }
  const uint4 o0 = make_uint4(o[0], o[1], o[2], o[3]), o1 = make_uint4(o[4], o[5], o[6], o[7]);
  *pa = flip ? o1 : o0;
  *pb = flip ? o0 : o1;
}

// per-term mode: one 16-column chunk of a W row (swizzle key / flip as epi16)
// widened to fp32 pairs, and the pairs rounded (RNE) back in place
__device__ __forceinline__ void w_load16(const uint8_t* wrow, int key, int flip, int col16, uint64_t* v) {
  const uint4 ua = *reinterpret_cast<const uint4*>(wrow + (((col16 * 2 + flip) ^ key) << 4));
  const uint4 ub = *reinterpret_cast<const uint4*>(wrow + (((col16 * 2 + (flip ^ 1)) ^ key) << 4));
  const uint4 u0 = flip ? ub : ua, u1 = flip ? ua : ub;
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u));
}

__device__ __forceinline__ void w_store16(uint8_t* wrow, int key, int flip, int col16, const uint64_t* v) {
  uint32_t o[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) o[q] = f2_to_bf16x2(v[q]);
  const uint4 o0 = make_uint4(o[0], o[1], o[2], o[3]), o1 = make_uint4(o[4], o[5], o[6], o[7]);
  *reinterpret_cast<uint4*>(wrow + (((col16 * 2 + flip) ^ key) << 4)) = flip ? o1 : o0;
  *reinterpret_cast<uint4*>(wrow + (((col16 * 2 + (flip ^ 1)) ^ key) << 4)) = flip ? o0 : o1;
}


// As epi16, keeping the 8 rounded bf16x2 words of the 16 columns for the dot
// product the fused decode computes after the tile has been handed to the store.
__device__ __forceinline__ void epi16_keep(uint8_t* wrow, int key, int flip, int col16, const uint32_t* acc,
                                           uint32_t* o) {
  uint4* pa = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + flip) ^ key) << 4));
  uint4* pb = reinterpret_cast<uint4*>(wrow + (((col16 * 2 + (flip ^ 1)) ^ key) << 4));
  const uint4 ua = *pa, ub = *pb;
  const uint4 u0 = flip ? ub : ua, u1 = flip ? ua : ub;
  const uint32_t w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint64_t v = fadd2(f2_pack(__uint_as_float(w[q] << 16), __uint_as_float(w[q] & 0xffff0000u)),
                             f2_pack(__uint_as_float(acc[2 * q]), __uint_as_float(acc[2 * q + 1])));
    o[q] = f2_to_bf16x2(v);
  }
  const uint4 o0 = make_uint4(o[0], o[1], o[2], o[3]), o1 = make_uint4(o[4], o[5], o[6], o[7]);
  *pa = flip ? o1 : o0;
  *pb = flip ? o0 : o1;
}

// y2 (fp32 pairs) += RNE(W + D) . x over 16 columns: packed FMA of the element
// pairs in column order (x: 16 bf16 of this thread's columns)
__device__ __forceinline__ uint64_t dot16(const uint32_t* o, const uint4 x0, const uint4 x1, uint64_t y2) {
  const uint32_t xw[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
  for (int q = 0; q < 8; ++q)
    y2 = ffma2(f2_pack(__uint_as_float(o[q] << 16), __uint_as_float(o[q] & 0xffff0000u)),
               f2_pack(__uint_as_float(xw[q] << 16), __uint_as_float(xw[q] & 0xffff0000u)), y2);
  return y2;
}

// ------------------------------------------------------------------ CTA pairs

__device__ __forceinline__ uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// the shared::cluster address of the same shared offset in CTA `rank`
__device__ __forceinline__ uint32_t mapa_u32(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// pair: a tensor copy into this CTA's shared memory completing on `bar`,
// which may be the leader's barrier (shared::cluster address)
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
// arrive on the mbarrier at the same shared offset in CTA `rank` of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
// the pair's MMA (leader only): D[256 x 128] += A[256 x K] . B[128 x K]^T, A = the
// two CTAs' B strips (M halves), B = their A^T halves (N halves), same offsets
__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
      ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// commit the pair's MMAs to the barrier at this offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"((uint16_t)3) : "memory");
}

// ------------------------------------------------------------------ the kernel

template <bool kF, bool kPT, bool kPair = false, bool kTB = false>
__global__ void __launch_bounds__(kThreads, 1)
switch_fc_kernel(const __grid_constant__ Maps maps, const __grid_constant__ Args args) {
  static_assert(!kPair || (!kF && !kPT), "CTA pairs: the plain fold mode only");
  static_assert(!kTB || (!kF && !kPT && !kPair), "TMEM strip: the plain fold mode only");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ Coefs cf;
  __shared__ int32_t s_parity;
  __shared__ unsigned long long s_fz_t0, s_fz_proc;   // fused: this CTA's segment processing time
  __shared__ uint32_t s_fz_n;                          //        and tiles (adaptive split)
  __shared__ int32_t s_fz_last;
  __shared__ int32_t s_claim[2 + 16];            // plain sweep, dynamic chunks: [claimed, claimer, id[16]]
  __shared__ uint32_t s_tmem_base;
  __shared__ __align__(8) uint64_t bar_wfull[kMaxStages], bar_wempty[kMaxStages], bar_wdone[kMaxStages];
  __shared__ __align__(8) uint64_t bar_afull[kMaxAStages], bar_aempty[kMaxAStages];
  __shared__ __align__(8) uint64_t bar_braw[2], bar_bfull[2], bar_bempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[kAccBufs], bar_accempty[kAccBufs];
  __shared__ __align__(8) uint64_t bar_bpeer[2];   // pair: the follower's B strip folded
  __shared__ __align__(8) uint64_t bar_rawfull, bar_rawempty;                // tb: the raw B strip copy

  const Geom& g = args.g;
  const uint32_t crank = kPair ? cta_rank_in_cluster() : 0;
  const bool leader = crank == 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // shared layout (1 KB aligned): [w_stages x W tile][a_stages x A slices][b_bufs x (hi, lo) B strip]
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* wst0 = base;
  uint8_t* ast0 = wst0 + (size_t)g.w_stages * (2 * kSubBytes);
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
    s_fz_t0 = globaltimer();
    s_fz_proc = 0;
    s_fz_n = 0;
    s_claim[0] = 0;
    s_claim[1] = 0;
    build_coefs(p, parity, cf);
    if (blockIdx.x == 0 && !cf.bad) stage_decision(p, parity);
    for (int s = 0; s < g.w_stages; ++s) {
      mbar_init(smem_u32(&bar_wfull[s]), 1);
      mbar_init(smem_u32(&bar_wempty[s]), 1);
      mbar_init(smem_u32(&bar_wdone[s]), kEpiWarps);
    }
    for (int s = 0; s < g.a_stages; ++s) {
      mbar_init(smem_u32(&bar_afull[s]), 1);
      mbar_init(smem_u32(&bar_aempty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&bar_braw[s]), 1);
      // fold: + the MMA warp's half; tb: every epilogue warp's TMEM stores
      mbar_init(smem_u32(&bar_bfull[s]), kTB ? kEpiWarps : g.b_bufs == 1 && !g.pt ? 2 : 1);
      mbar_init(smem_u32(&bar_bempty[s]), 1);
      mbar_init(smem_u32(&bar_bpeer[s]), 1);
    }
    mbar_init(smem_u32(&bar_rawfull), 1);
    mbar_init(smem_u32(&bar_rawempty), kEpiWarps);
    for (int s = 0; s < g.acc_bufs; ++s) {
      mbar_init(smem_u32(&bar_accfull[s]), 1);
      mbar_init(smem_u32(&bar_accempty[s]), kPair ? 2 * kEpiWarps : kEpiWarps);   // pair: both CTAs' epilogues
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0)
    for (int k = 0; k < LSW_NKIND; ++k) prefetch_map(args.mode == MODE_RESTORE ? &maps.p[k] : &maps.w[k]);
  if (warp == 1) {
    if constexpr (kPair) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(&s_tmem_base)), "r"(kAccBufs * kTN) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                   ::"r"(smem_u32(&s_tmem_base)), "r"(kAccBufs * kTN) : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();      // the peer's barriers exist before any remote arrive / commit
  tc_fence_after();

  const int nt = cf.bad ? 0 : cf.n;
  TileSeq seq;
  seq.T = args.t_count > 0 ? args.t_count : kPair ? g.tiles_pair : g.tiles_total;
  seq.t0 = args.t0;
  seq.chunk = args.chunk < 1 ? 1 : args.chunk;
  seq.G = kPair ? gridDim.x / 2 : gridDim.x;      // pair: both CTAs of a cluster walk the same pair tiles
  seq.b = kPair ? blockIdx.x / 2 : blockIdx.x;
  seq.adapt = 0;
  seq.wlo = seq.whi = 0;
  seq.dyn = !kF && !kPair && args.dyn && seq.chunk >= 2;
  seq.ctr = &args.state->sweep_next;
  seq.ring = s_claim;
  if constexpr (kF) {
    // adaptive split (written by the previous fused pass's last CTA; stream-ordered)
    if (args.adapt && gridDim.x <= kFusedMaxCtas &&
        *reinterpret_cast<volatile const int32_t*>(&args.state->fused_w_valid) == (int32_t)gridDim.x) {
      seq.adapt = 1;
      seq.wlo = args.state->fused_w[blockIdx.x];
      seq.whi = args.state->fused_w[blockIdx.x + 1];
    }
  }
  const TileKinds& tk = kPair ? g.tkp : g.tk;
  // pair: this CTA's 128-row tile of the pair tile's 256 rows
  auto rbr = [&](int rb) { return kPair ? 2 * rb + (int)crank : rb; };
  const uint32_t tmem_base = s_tmem_base;

  // Nothing to add (nt == 0: the new decision equals the merged one, R12, or
  // the decision was rejected): the plain pass is a no-op; the fused pass still
  // streams W (unchanged, not stored back) and computes its GEMV outputs.
  if (nt > 0 || kF) {
    if (warp == 0) {
      // ============================ W producer =============================
      if (lane == 0) {
        const uint64_t pol_stream = policy_evict_first();
        const CUtensorMap* src = args.mode == MODE_RESTORE ? maps.p : maps.w;   // RESTORE reads P
        Ring wring{0, 0, (uint32_t)g.w_stages};
        int nt_tr = 0;
        for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
          mbar_wait(smem_u32(&bar_wempty[wring.i]), wring.phase ^ 1);
          FC_TRACE(0, nt_tr++);
          const uint32_t wbar = smem_u32(&bar_wfull[wring.i]);
          mbar_expect_tx(wbar, 2 * kSubBytes);
          uint8_t* wdst = wst0 + (size_t)wring.i * (2 * kSubBytes);
          if (g.wrm)
            tma_load_4d(smem_u32(wdst), &src[c.kd], 0, c.cb * 2, rbr(c.rb) * kTM, c.layer, wbar, pol_stream);
          else
            for (int sb = 0; sb < 2; ++sb)
              tma_load_3d(smem_u32(wdst + sb * kSubBytes), &src[c.kd], c.cb * kTN + sb * kSubCols, rbr(c.rb) * kTM,
                          c.layer, wbar, pol_stream);
          wring.next();
        }
      }
    } else if (warp == 2) {
      // ============================ store warp ==============================
      if (lane == 0) {
        const uint64_t pol_stream = policy_evict_first();
        Ring wring{0, 0, (uint32_t)g.w_stages};
        int ns_tr = 0;
        for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
          mbar_wait(smem_u32(&bar_wdone[wring.i]), wring.phase);     // epilogue wrote the tile
          if (nt == 0) {                                             // fused, W unchanged: no store
            mbar_arrive(smem_u32(&bar_wempty[wring.i]));
            wring.next();
            continue;
          }
          uint8_t* wsrc = wst0 + (size_t)wring.i * (2 * kSubBytes);
          if (g.wrm)
            tma_store_4d(&maps.w[c.kd], smem_u32(wsrc), 0, c.cb * 2, rbr(c.rb) * kTM, c.layer, pol_stream);
          else
            for (int sb = 0; sb < 2; ++sb)
              tma_store_3d(&maps.w[c.kd], smem_u32(wsrc + sb * kSubBytes), c.cb * kTN + sb * kSubCols,
                           rbr(c.rb) * kTM, c.layer, pol_stream);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read -> stage reusable
          FC_TRACE(7, ns_tr++);
          mbar_arrive(smem_u32(&bar_wempty[wring.i]));
          wring.next();
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      }
    } else if (warp == 3 && nt > 0 && !(args.probe & 1)) {
      if constexpr (kPT) {
        // per-term mode: raw B slices per strip and A^T slices per (tile, term
        // group), all by bulk copies completing on the consumers' barriers
        if (lane == 0) {
          const uint64_t pol_keep = policy_evict_last();
          const size_t rpe = (size_t)g.rp;
          const uint32_t tb = g.term_bytes;
          int64_t strip_prev = -1;
          Ring bring{0, 0, (uint32_t)g.b_bufs};
          Ring aring{0, 0, (uint32_t)g.a_stages};
          for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
            if (!g.bu && strip_id(c) != strip_prev) {
              if (strip_prev >= 0) bring.next();
              strip_prev = strip_id(c);
              mbar_wait(smem_u32(&bar_bempty[bring.i]), bring.phase ^ 1);
              uint8_t* dst = bst0 + (size_t)bring.i * g.b_buf_bytes;
              const uint32_t bar = smem_u32(&bar_bfull[bring.i]);
              mbar_expect_tx(bar, nt * tb);
              for (int j = 0; j < nt; ++j)
                bulk_load(smem_u32(dst + j * tb),
                          g.Bp[c.kd] + (((size_t)c.layer * g.n_experts + cf.e[j]) * g.dout_pad[c.kd] +
                                        (size_t)c.rb * kTM) * rpe,
                          tb, bar, pol_keep);
            }
            const __nv_bfloat16* blk =
                g.At[c.kd] + (((size_t)c.layer * tk.col_tiles[c.kd] + c.cb) * g.n_experts) * (size_t)kTN * rpe;
            for (int j0 = 0; j0 < nt; j0 += kPtGroup) {
              const int n_in = nt - j0 < kPtGroup ? nt - j0 : kPtGroup;
              mbar_wait(smem_u32(&bar_aempty[aring.i]), aring.phase ^ 1);
              uint8_t* adst = ast0 + (size_t)aring.i * g.a_stage_bytes;
              const uint32_t bar = smem_u32(&bar_afull[aring.i]);
              mbar_expect_tx(bar, (g.bu ? 2 : 1) * n_in * tb);
              for (int jj = 0; jj < n_in; ++jj)
                bulk_load(smem_u32(adst + jj * tb), blk + (size_t)cf.e[j0 + jj] * kTN * rpe, tb, bar, pol_keep);
              if (g.bu)                              // the unit's B slices of this strip, after its A^T slices
                for (int jj = 0; jj < n_in; ++jj)
                  bulk_load(smem_u32(adst + (kPtGroup + jj) * tb),
                            g.Bp[c.kd] + (((size_t)c.layer * g.n_experts + cf.e[j0 + jj]) * g.dout_pad[c.kd] +
                                          (size_t)c.rb * kTM) * rpe,
                            tb, bar, pol_keep);
              aring.next();
            }
          }
        }
      } else if (kTB) {
        // tb mode: raw B strips (one or two ahead of the walk, as many as TMEM
        // buffers) for the epilogue to fold into TMEM, and per tile the A^T
        // slices in units of unit_terms terms (freed by the epilogue with the tile)
        if (lane == 0) {
          const uint64_t pol_keep = policy_evict_last();
          const size_t rpe = (size_t)g.rp;
          const uint32_t tb = g.term_bytes;
          const int U = g.unit_terms;
          FCursor rc = cur_first<kF>(tk, seq, args);
          uint32_t raw_phase = 0;
          auto load_raw = [&]() {                  // the strip at rc, then rc -> the next strip
            if (rc.t < 0) return;
            mbar_wait(smem_u32(&bar_rawempty), raw_phase ^ 1);
            const uint32_t bar = smem_u32(&bar_rawfull);
            mbar_expect_tx(bar, nt * tb);
            for (int j = 0; j < nt; ++j)
              bulk_load(smem_u32(bst0 + j * tb),
                        g.Bp[rc.kd] + (((size_t)rc.layer * g.n_experts + cf.e[j]) * g.dout_pad[rc.kd] +
                                       (size_t)rc.rb * kTM) * rpe,
                        tb, bar, pol_keep);
            raw_phase ^= 1;
            strip_advance<kF>(tk, seq, args, rc);
          };
          for (int i = 0; i < g.b_bufs; ++i) load_raw();
          Ring aring{0, 0, (uint32_t)g.a_stages};
          int64_t strip_prev = -1;
          int na_tr = 0;
          for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
            if (strip_id(c) != strip_prev) {
              if (strip_prev >= 0) load_raw();
              strip_prev = strip_id(c);
            }
            const __nv_bfloat16* blk =
                g.At[c.kd] + (((size_t)c.layer * tk.col_tiles[c.kd] + c.cb) * g.n_experts) * (size_t)kTN * rpe;
            FC_TRACE(1, na_tr++);
            for (int j0 = 0; j0 < nt; j0 += U) {
              const int n_in = nt - j0 < U ? nt - j0 : U;
              mbar_wait(smem_u32(&bar_aempty[aring.i]), aring.phase ^ 1);
              uint8_t* adst = ast0 + (size_t)aring.i * g.a_stage_bytes;
              const uint32_t bar = smem_u32(&bar_afull[aring.i]);
              mbar_expect_tx(bar, n_in * tb);
              for (int jj = 0; jj < n_in; ++jj)
                bulk_load(smem_u32(adst + jj * tb), blk + (size_t)cf.e[j0 + jj] * kTN * rpe, tb, bar, pol_keep);
              aring.next();
            }
          }
        }
      } else {
      // ============================ operand producer ========================
      // Per strip (rare): raw B slices of all terms by bulk copies into the lo
      // slots, then the whole warp folds them into (hi, lo) parts in place and
      // publishes the buffer to the MMA warp (generic -> async proxy fence).
      // Per tile: all terms' A^T slices (each one contiguous block) into one A
      // stage, released by the epilogue once the tile's accumulator is complete.
      const uint64_t pol_keep = policy_evict_last();
      const size_t rpe = (size_t)g.rp;
      const uint32_t tb = g.term_bytes;
      const uint32_t vec_per_term = tb / 16;
      int64_t strip_prev = -1;
      Ring bring{0, 0, (uint32_t)g.b_bufs};
      Ring aring{0, 0, (uint32_t)g.a_stages};
      int na_tr = 0;
      for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
        if (strip_id(c) != strip_prev) {
          if (strip_prev >= 0) bring.next();
          strip_prev = strip_id(c);
          mbar_wait(smem_u32(&bar_bempty[bring.i]), bring.phase ^ 1);
          uint8_t* dst = bst0 + (size_t)bring.i * g.b_buf_bytes;
          const uint32_t rbar = smem_u32(&bar_braw[bring.i]);
          if (lane == 0) {
            mbar_expect_tx(rbar, nt * tb);
            for (int j = 0; j < nt; ++j) {
              const __nv_bfloat16* src = g.Bp[c.kd] + (((size_t)c.layer * g.n_experts + cf.e[j]) * g.dout_pad[c.kd] +
                                                       (size_t)rbr(c.rb) * kTM) * rpe;
              bulk_load(smem_u32(dst + (2 * j + 1) * tb), src, tb, rbar, pol_keep);
            }
          }
          mbar_wait(rbar, bring.phase);
          // with a single B buffer the fold is on the MMA's critical path: the
          // MMA warp, idle until it lands, folds the second half of every term
          if (!(args.probe & 16))                    // probe 16 (tuning only): skip the fold math
            fold_range(dst, tb, nt, cf.c, 0, g.b_bufs == 1 ? vec_per_term / 2 : vec_per_term, lane);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_bfull[bring.i]));
        }
        if (lane == 0) {
          const __nv_bfloat16* blk =
              g.At[c.kd] + (((size_t)c.layer * tk.col_tiles[c.kd] + c.cb) * g.n_experts) * (size_t)kTN * rpe;
          mbar_wait(smem_u32(&bar_aempty[aring.i]), aring.phase ^ 1);
          FC_TRACE(1, na_tr);
          uint8_t* adst = ast0 + (size_t)aring.i * g.a_stage_bytes;
          const uint32_t bar = smem_u32(&bar_afull[aring.i]);
          if constexpr (kPair) {
            // this CTA's half of the tile's 128 columns (rows 64 * rank.. of
            // each A^T slice) by .cta_group::2 tensor copies completing on the
            // LEADER's barrier, which expects both halves: no relay of the
            // stage from the follower to the leader's MMA warp
            const uint32_t ta = tb / 2;
            if (leader) mbar_expect_tx(bar, 2 * nt * ta);
            const uint32_t lbar = leader ? bar : mapa_u32(bar, 0);
            const int64_t row0 = (((int64_t)c.layer * tk.col_tiles[c.kd] + c.cb) * g.n_experts) * kTN +
                                 (int64_t)crank * (kTN / 2);
            for (int j = 0; j < nt; ++j)
              tma_load_2d_cg2(smem_u32(adst + j * ta), &maps.at[c.kd], 0, (int32_t)(row0 + (int64_t)cf.e[j] * kTN),
                              lbar, pol_keep);
          } else {
            mbar_expect_tx(bar, nt * tb);
            for (int j = 0; j < nt; ++j)
              bulk_load(smem_u32(adst + j * tb), blk + (size_t)cf.e[j] * kTN * rpe, tb, bar, pol_keep);
          }
        }
        __syncwarp();
        aring.next();
        ++na_tr;
      }
      }  // !kPT
    } else if (warp == 1 && nt > 0 && !(args.probe & 1)) {
      // ============================ MMA issuer ==============================
      // One chain per tile: for every term, the hi and lo parts times the A^T
      // slice, K = rp each in steps of 16, into the tile's single accumulator;
      // ONE commit per tile.
      // instruction descriptor: D f32, A/B bf16, both K-major, N = 128, M = 128
      // (pair: M = 256 -- the two CTAs' 128-row tiles)
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTN >> 3) << 17) |
                             ((uint32_t)((kPair ? 2 : 1) * kTM >> 4) << 24);
      const uint32_t sbo = 8 * (uint32_t)g.rp * 2;
      const int ksteps = g.rp / 16;
      const uint64_t desc0 = umma_desc(0, sbo, g.swz_mode);
      const uint64_t term = g.term_bytes >> 4;
      const uint64_t aterm = (kPair ? g.term_bytes / 2 : g.term_bytes) >> 4;   // A^T slice per term in a stage
      Ring bring{0, 0, (uint32_t)g.b_bufs};
      Ring aring{0, 0, (uint32_t)g.a_stages};
      Ring acc{0, 0, (uint32_t)g.acc_bufs};
      int64_t strip_prev = -1;
      int nm_tr = 0;
      for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
        if (!g.bu && strip_id(c) != strip_prev) {
          if (strip_prev >= 0) {
            // every MMA of the previous strip is issued: its B buffer is free
            // once they complete -- released by a commit here, not after the
            // epilogue (up to kAccBufs tiles behind) has seen them, so a single
            // B buffer is refolded while the epilogue drains the accumulators
            // (pair: the leader's commit frees both CTAs' buffers)
            if constexpr (kPair) {
              if (leader && elect_one()) umma_commit_pair(smem_u32(&bar_bempty[bring.i]));
            } else {
              // (tb: the epilogue refolds a TMEM buffer only after the strip's
              // last accumulator, which completes after its MMAs)
              if (!kTB && elect_one()) umma_commit(smem_u32(&bar_bempty[bring.i]));
            }
            __syncwarp();
            bring.next();
          }
          strip_prev = strip_id(c);
          if (!kPT && !kTB && g.b_bufs == 1) {
            // single B buffer: fold the second half of every term here (the
            // operand warp folds the first half), then publish it
            uint8_t* dst = bst0 + (size_t)bring.i * g.b_buf_bytes;
            mbar_wait(smem_u32(&bar_braw[bring.i]), bring.phase);
            if (!(args.probe & 16))
              fold_range(dst, g.term_bytes, nt, cf.c, g.term_bytes / 32, g.term_bytes / 16, lane);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor core
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_bfull[bring.i]));
          }
          mbar_wait(smem_u32(&bar_bfull[bring.i]), bring.phase);
          tc_fence_after();                          // tb: the epilogue's TMEM stores -> the MMAs
          if constexpr (kPair) {
            // the leader's MMAs read both strips: the follower reports its own
            if (!leader) {
              if (lane == 0) mbar_arrive_remote(smem_u32(&bar_bpeer[bring.i]), 0);
            } else {
              mbar_wait(smem_u32(&bar_bpeer[bring.i]), bring.phase);
            }
          }
        }
        if constexpr (kPair) {
          if (!leader) {                         // follower: no MMA (its A halves land on the leader's barrier)
            aring.next();
            continue;
          }
        }
        if constexpr (kPT) {
          // per-term mode: kPtGroup terms per group, each into its own 128-column
          // accumulator of the group's TMEM buffer, one commit per group
          const uint64_t b_strip = desc0 + (smem_u32(bst0 + (size_t)bring.i * g.b_buf_bytes) >> 4);
          for (int j0 = 0; j0 < nt; j0 += kPtGroup) {
            const int n_in = nt - j0 < kPtGroup ? nt - j0 : kPtGroup;
            mbar_wait(smem_u32(&bar_afull[aring.i]), aring.phase);
            mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
            tc_fence_after();
            const uint64_t a_desc = desc0 + (smem_u32(ast0 + (size_t)aring.i * g.a_stage_bytes) >> 4);
            // B of term j0 + jj: the strip buffer, or (bu) the unit's own slices
            const uint64_t b_desc = g.bu ? a_desc + kPtGroup * term : b_strip + j0 * term;
            const uint32_t d = tmem_base + acc.i * g.acc_cols;
            if (elect_one()) {
              for (int jj = 0; jj < n_in; ++jj)
                for (int kk = 0; kk < ksteps; ++kk)
                  umma_f16(d + jj * kTN, b_desc + jj * term + kk * 2, a_desc + jj * term + kk * 2, idesc,
                           kk > 0 ? 1u : 0u);
              umma_commit(smem_u32(&bar_accfull[acc.i]));
            }
            __syncwarp();
            acc.next();
            aring.next();
          }
          continue;
        }
        if constexpr (kTB) {
          // tb: the M-side operand (the strip's (hi, lo) parts) read from TMEM;
          // the A^T slices unit by unit as they land
          mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
          tc_fence_after();
          if (lane == 0) FC_TRACE(2, nm_tr);
          const uint32_t d = tmem_base + acc.i * kTN;
          const uint32_t bt = tmem_base + g.b_col0 + bring.i * g.bcols;
          const int U = g.unit_terms;
          const uint32_t hrp = (uint32_t)g.rp / 2;
          for (int j0 = 0; j0 < nt; j0 += U) {
            const int n_in = nt - j0 < U ? nt - j0 : U;
            mbar_wait(smem_u32(&bar_afull[aring.i]), aring.phase);
            tc_fence_after();
            const uint64_t a_desc = desc0 + (smem_u32(ast0 + (size_t)aring.i * g.a_stage_bytes) >> 4);
            if (elect_one()) {
              for (int jj = 0; jj < n_in; ++jj) {
                const int j = j0 + jj;
                for (int part = 0; part < 2; ++part)
                  for (int kk = 0; kk < ksteps; ++kk)
                    umma_f16_ts(d, bt + (uint32_t)j * g.rp + part * hrp + kk * 8, a_desc + jj * term + kk * 2, idesc,
                                (j | part | kk) != 0 ? 1u : 0u);
              }
              if (g.unit_commit) umma_commit(smem_u32(&bar_aempty[aring.i]));
            }
            __syncwarp();
            aring.next();
          }
          // each unit freed by its own commit (unit_commit, the default), or,
          // with option fc_unit_commit = 0 where the ring holds two tiles'
          // units, by the epilogue with its tile (one commit per tile)
          if (elect_one()) umma_commit(smem_u32(&bar_accfull[acc.i]));
          if (lane == 0) FC_TRACE(3, nm_tr);
          ++nm_tr;
          __syncwarp();
          acc.next();
          continue;
        }
        mbar_wait(smem_u32(&bar_afull[aring.i]), aring.phase);   // (pair: both CTAs' A halves)
        if (lane == 0) FC_TRACE(2, nm_tr);
        mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
        tc_fence_after();
        const uint64_t b_desc = desc0 + (smem_u32(bst0 + (size_t)bring.i * g.b_buf_bytes) >> 4);
        const uint64_t a_desc = desc0 + (smem_u32(ast0 + (size_t)aring.i * g.a_stage_bytes) >> 4);
        const uint32_t d = tmem_base + acc.i * kTN;
        if constexpr (kPair) {
          if (elect_one()) {
            for (int j = 0; j < nt; ++j)
              for (int part = 0; part < 2; ++part)
                for (int kk = 0; kk < ksteps; ++kk)
                  umma_f16_pair(d, b_desc + (2 * j + part) * term + kk * 2, a_desc + j * aterm + kk * 2, idesc,
                                (j | part | kk) != 0 ? 1u : 0u);
            umma_commit_pair(smem_u32(&bar_aempty[aring.i]));   // both CTAs' A stages free when these complete
            umma_commit_pair(smem_u32(&bar_accfull[acc.i]));
          }
        } else if (elect_one()) {
          for (int j = 0; j < nt; ++j)
            for (int part = 0; part < 2; ++part)
              for (int kk = 0; kk < ksteps; ++kk)
                umma_f16(d, b_desc + (2 * j + part) * term + kk * 2, a_desc + j * term + kk * 2, idesc,
                         (j | part | kk) != 0 ? 1u : 0u);
          umma_commit(smem_u32(&bar_accfull[acc.i]));
        }
        if (lane == 0) FC_TRACE(3, nm_tr);
        ++nm_tr;
        __syncwarp();
        acc.next();
        aring.next();
      }
    } else if (warp >= kFirstEpiWarp) {
      // ============================ epilogue ================================
      // Warp w reads TMEM lane quarter w % 4 (rows 32*(w%4) ..) and one 64-column
      // half of the tile (= one W sub-tile): per thread one row x 64 columns.
      const int ew = warp - kFirstEpiWarp;
      const int quarter = warp & 3, half = ew >> 2;
      const int row = quarter * 32 + lane;
      const bool releaser = ew == 0 && lane == 0;   // frees A stages for the producer
      Ring wring{0, 0, (uint32_t)g.w_stages};
      Ring acc{0, 0, (uint32_t)g.acc_bufs};
      Ring aring{0, 0, (uint32_t)g.a_stages};
      int ne_tr = 0;
#ifdef LSW_TUNING
      if (kF && releaser && args.seg_trace) {     // slot 511: this CTA's SM (per-SM lateness analysis)
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        args.seg_trace[((size_t)blockIdx.x * 512 + 511) * 2 + 0] = smid + 1;
      }
#endif
      int cur_seg = -1;                            // fused: segment of the previous tile
      int conv_next = 0;                           // fused: first segment whose outputs this CTA has not converted
      unsigned long long seg_mine = 0;             // fused: tiles of cur_seg this CTA finished
      // fused: this thread's partial output of one row over the consecutive
      // column tiles of a strip (a CTA's range walks cb fastest), added to the
      // fixed-point accumulator once per strip, not per tile
      long long y_run = 0;                         // 2^-40 units: each tile's fp32 partial converted, then
                                                   // integer adds -- independent of how a strip's tiles are
                                                   // split among CTAs (the adaptive split moves them)
      int64_t y_at = -1;                           // ys_fx index y_run belongs to (-1: none)
      auto y_flush = [&]() {
        if (y_at >= 0) atomicAdd(args.ys_fx + y_at, (unsigned long long)y_run);
        y_at = -1;
        y_run = 0;
      };
      // tb: the strips are folded into TMEM here, in walk order, as many ahead as
      // there are TMEM buffers (buffer f % b_bufs for the f-th fold): the first
      // b_bufs at the start, then at the start of strip s the strip s + b_bufs - 1
      // -- its buffer last held strip s - 1, whose accumulators are all consumed.
      // (Measured: folding the next strip as soon as its raw copy lands,
      // tried at every tile, is slower.)
      const bool tbm = kTB && nt > 0 && !(args.probe & 1);
      FCursor rc = cur_first<kF>(tk, seq, args);
      int64_t ep_strip = -1;
      uint32_t nf = 0;
      auto fold_next = [&]() {
        if (rc.t < 0) return;
        const uint32_t buf = nf % (uint32_t)g.b_bufs;
        mbar_wait(smem_u32(&bar_rawfull), nf & 1);
        const uint32_t bt = tmem_base + ((uint32_t)(quarter * 32) << 16) + g.b_col0 + buf * g.bcols;
        for (int j = half; j < nt; j += 2) {
          const uint8_t* slice = bst0 + (size_t)j * g.term_bytes;
          const uint32_t ta = bt + (uint32_t)j * g.rp;
          if (g.rp == 16) fold_row_tmem<16>(slice, row, cf.c[j], ta);
          else if (g.rp == 32) fold_row_tmem<32>(slice, row, cf.c[j], ta);
          else fold_row_tmem<64>(slice, row, cf.c[j], ta);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(smem_u32(&bar_bfull[buf]));
          mbar_arrive(smem_u32(&bar_rawempty));
        }
        ++nf;
        strip_advance<kF>(tk, seq, args, rc);
      };
      for (FCursor c = cur_first<kF>(tk, seq, args); c.t >= 0; cur_next<kF>(tk, seq, args, c)) {
        uint4 xv[8];                               // fused: x of this thread's 64 columns
        if (tbm && strip_id(c) != ep_strip) {
          if (ep_strip < 0)
            for (int i = 0; i < g.b_bufs; ++i) fold_next();
          else
            fold_next();
          ep_strip = strip_id(c);
        }
        if constexpr (kF) {
          if (c.seg != cur_seg) {
            y_flush();                             // before the segment's count is published
            // decoder order: x of segment s is final only once every tile of
            // segment s-1 is done -- one thread per CTA publishes the CTA's
            // count of the segment it leaves and waits for the previous total
            __syncwarp();
            asm volatile("bar.sync 3, %0;" ::"r"(32 * kEpiWarps) : "memory");
            if (releaser && cur_seg >= 0) {
              __threadfence();
              asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(args.seg_done + cur_seg),
                           "l"(seg_mine) : "memory");
              FC_SEG_TRACE(cur_seg, 0);
              s_fz_proc += globaltimer() - s_fz_t0;
              s_fz_n += (uint32_t)seg_mine;
            }
            // every earlier segment complete (decoder order), then this CTA's
            // slice of its outputs converted from fixed point
            for (; conv_next < c.seg; ++conv_next) {
              if (releaser && !(args.probe & 4))
                wait_count(&args.seg_done[conv_next], (unsigned long long)args.segs[conv_next].tile_count);
              if (releaser) FC_SEG_TRACE(conv_next, 1);
              __syncwarp();
              asm volatile("bar.sync 3, %0;" ::"r"(32 * kEpiWarps) : "memory");
              fx_convert(args, conv_next, threadIdx.x - 32 * kFirstEpiWarp, 32 * kEpiWarps);
            }
            __syncwarp();
            asm volatile("bar.sync 3, %0;" ::"r"(32 * kEpiWarps) : "memory");
            if (releaser) s_fz_t0 = globaltimer();    // the segment's processing starts
            cur_seg = c.seg;
            seg_mine = 0;
          }
          const int64_t col0 = (int64_t)c.cb * kTN + half * kSubCols;
          const int64_t lim = g.d_in[c.kd] - col0;      // columns of this half inside d_in
          const uint4* xp = reinterpret_cast<const uint4*>(args.xs + c.x_off + col0);
#pragma unroll
          for (int v = 0; v < 8; ++v) xv[v] = 8 * v < lim ? __ldg(xp + v) : make_uint4(0, 0, 0, 0);
        }
        if (args.probe & 1) {                      // tuning: the W stream alone
          mbar_wait(smem_u32(&bar_wfull[wring.i]), wring.phase);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_wdone[wring.i]));
          wring.next();
          continue;
        }
        if constexpr (kPT) {
          // per-term mode: v = W, then v <- c_j * acc_j + v for j ascending
          // (fp32, FFMA2; the order does not depend on the grouping), term
          // group by term group as their accumulators complete; ONE RNE
          mbar_wait(smem_u32(&bar_wfull[wring.i]), wring.phase);
          const int unit = g.wrm ? 2 * row + half : half * kTM + row;
          const int key = unit & 7, flip = g.wrm ? (row >> 2) & 1 : 0;
          uint8_t* wrow = wst0 + (size_t)wring.i * (2 * kSubBytes) + unit * 128;
          uint64_t v[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q) w_load16(wrow, key, flip, q, v[q]);
          for (int j0 = 0; j0 < nt; j0 += kPtGroup) {
            const int n_in = nt - j0 < kPtGroup ? nt - j0 : kPtGroup;
            mbar_wait(smem_u32(&bar_accfull[acc.i]), acc.phase);
            if (releaser) mbar_arrive(smem_u32(&bar_aempty[aring.i]));
            aring.next();
            tc_fence_after();
            const uint32_t tm = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * g.acc_cols + half * kSubCols;
            const uint64_t c0 = f2_pack(cf.c[j0], cf.c[j0]);
            const uint64_t c1 = n_in > 1 ? f2_pack(cf.c[j0 + 1], cf.c[j0 + 1]) : 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t a0[16], a1[16];
              tmem_ld16(tm + q * 16, a0);
              if (n_in > 1) tmem_ld16(tm + kTN + q * 16, a1);
              tmem_wait_ld();
#pragma unroll
              for (int p = 0; p < 8; ++p)
                v[q][p] = ffma2(f2_pack(__uint_as_float(a0[2 * p]), __uint_as_float(a0[2 * p + 1])), c0, v[q][p]);
              if (n_in > 1) {
#pragma unroll
                for (int p = 0; p < 8; ++p)
                  v[q][p] = ffma2(f2_pack(__uint_as_float(a1[2 * p]), __uint_as_float(a1[2 * p + 1])), c1, v[q][p]);
              }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(smem_u32(&bar_accempty[acc.i]));
            acc.next();
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) w_store16(wrow, key, flip, q, v[q]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> TMA store
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_wdone[wring.i]));
          wring.next();
          continue;
        }
        uint32_t a[4][16];
        if (nt > 0) {
          mbar_wait(smem_u32(&bar_accfull[acc.i]), acc.phase);      // the tile's MMAs are complete
          if (releaser) FC_TRACE(4, ne_tr);
          // (pair: the leader's commit released both CTAs' A stages)
          if constexpr (kTB) {                     // tb: the tile's A units (unless the MMA's commits free them)
            for (int u = 0; u < nt; u += g.unit_terms) {
              if (g.unit_commit) { aring.next(); continue; }
              if (releaser) mbar_arrive(smem_u32(&bar_aempty[aring.i]));
              aring.next();
            }
          } else {
            if (releaser && !kPair) mbar_arrive(smem_u32(&bar_aempty[aring.i]));
            aring.next();
          }
          tc_fence_after();
          const uint32_t tm = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * kTN + half * kSubCols;
#pragma unroll
          for (int q = 0; q < 4; ++q) tmem_ld16(tm + q * 16, a[q]);
          tmem_wait_ld();
          tc_fence_before();                       // accumulator consumed -> MMA may reuse the buffer
          __syncwarp();
          if (lane == 0) {
            if (kPair && !leader) mbar_arrive_remote(smem_u32(&bar_accempty[acc.i]), 0);   // the leader's MMA
            else mbar_arrive(smem_u32(&bar_accempty[acc.i]));
          }
          acc.next();
        } else {                                   // fused, nothing to add: y from the unchanged W
#pragma unroll
          for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int v = 0; v < 16; ++v) a[q][v] = 0u;
        }
        mbar_wait(smem_u32(&bar_wfull[wring.i]), wring.phase);      // W tile landed
        if (releaser) FC_TRACE(5, ne_tr);
        // default: two [128 rows][64 cols] boxes; wrm: one [128 rows][2 x 64 cols] box
        const int unit = g.wrm ? 2 * row + half : half * kTM + row;
        uint8_t* wrow = wst0 + (size_t)wring.i * (2 * kSubBytes) + unit * 128;
        if (kF && !(args.probe & 8)) {
          // new W first, handed to the store at once; the dot product from the
          // rounded words in registers while the store reads the stage
          uint32_t o[4][8];
#pragma unroll
          for (int q = 0; q < 4; ++q) epi16_keep(wrow, unit & 7, g.wrm ? (row >> 2) & 1 : 0, q, a[q], o[q]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> TMA store
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_wdone[wring.i]));
          if (releaser) FC_TRACE(6, ne_tr);
          ++ne_tr;
          wring.next();
          ++seg_mine;
          const int64_t grow = (int64_t)c.rb * kTM + row;
          const int64_t at = grow < g.d_out[c.kd] ? c.y_base + grow : -1;
          if (at != y_at) {
            y_flush();
            y_at = at;
          }
          uint64_t y2 = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) y2 = dot16(o[q], xv[2 * q], xv[2 * q + 1], y2);
          float ylo, yhi;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(ylo), "=f"(yhi) : "l"(y2));
          y_run += __double2ll_rn((double)(ylo + yhi) * kFx);
          continue;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) epi16(wrow, unit & 7, g.wrm ? (row >> 2) & 1 : 0, q, a[q]);
        if constexpr (kF) ++seg_mine;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> TMA store
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_wdone[wring.i]));
        if (releaser) FC_TRACE(6, ne_tr);
        ++ne_tr;
        wring.next();
      }
      if constexpr (kF) {
        y_flush();
        if (cur_seg >= 0) {                        // publish the last segment this CTA worked on
          __syncwarp();
          asm volatile("bar.sync 3, %0;" ::"r"(32 * kEpiWarps) : "memory");
          if (releaser) {
            __threadfence();
            asm volatile("red.release.gpu.global.add.u64 [%0], %1;" ::"l"(args.seg_done + cur_seg),
                         "l"(seg_mine) : "memory");
            s_fz_proc += globaltimer() - s_fz_t0;
            s_fz_n += (uint32_t)seg_mine;
          }
        }
        if (releaser && args.adapt && blockIdx.x < kFusedMaxCtas)
          args.state->fused_perf[blockIdx.x] = s_fz_n ? (float)((double)s_fz_proc / s_fz_n) : 0.f;
        for (; conv_next < args.n_seg; ++conv_next) {   // the remaining segments' outputs
          if (releaser && !(args.probe & 4))
            wait_count(&args.seg_done[conv_next], (unsigned long long)args.segs[conv_next].tile_count);
          __syncwarp();
          asm volatile("bar.sync 3, %0;" ::"r"(32 * kEpiWarps) : "memory");
          fx_convert(args, conv_next, threadIdx.x - 32 * kFirstEpiWarp, 32 * kEpiWarps);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kPair) cluster_sync_all();      // no remote arrive / commit may target a CTA that left
  if (warp == 1) {
    tc_fence_after();
    if constexpr (kPair)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAccBufs * kTN)
                   : "memory");
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAccBufs * kTN)
                   : "memory");
  }
  if constexpr (kF) {
    // adaptive split: the pass's last CTA weighs every CTA by its measured
    // speed (1 / ns per tile), half-and-half with the current split, each
    // weight within [1/2, 2] of uniform; the cumulative bounds (2^-24 units,
    // 0 and 2^24 at the ends) are the next pass's ranges.  Results do not
    // depend on the split (tiles are independent; y is fixed-point).
    if (args.adapt && gridDim.x <= kFusedMaxCtas) {
      DevState* st = args.state;
      const int G = (int)gridDim.x;
      if (threadIdx.x == 0) {
        __threadfence();
        const uint32_t prev = atomicAdd(&st->fused_done, 1u);
        s_fz_last = prev == (uint32_t)G - 1;
      }
      __syncthreads();
      if (s_fz_last) {
        __threadfence();
        float* wsh = reinterpret_cast<float*>(smem_raw);   // the stages are idle now
        for (int b = threadIdx.x; b < G; b += blockDim.x) {
          const float pf = *reinterpret_cast<volatile const float*>(&st->fused_perf[b]);
          wsh[b] = pf > 0.f ? 1.f / pf : 0.f;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
          const bool valid = *reinterpret_cast<volatile const int32_t*>(&st->fused_w_valid) == G;
          float spd_sum = 0.f;
          int n_ok = 0;
          for (int b = 0; b < G; ++b)
            if (wsh[b] > 0.f) { spd_sum += wsh[b]; ++n_ok; }
          const float mean = n_ok ? spd_sum / n_ok : 1.f;
          float tot = 0.f;
          for (int b = 0; b < G; ++b) {
            const float meas = (wsh[b] > 0.f ? wsh[b] : mean) / (mean * G);          // measured share
            const float old = valid ? (float)(st->fused_w[b + 1] - st->fused_w[b]) * (1.f / 16777216.f)
                                    : 1.f / G;
            float w = 0.5f * old + 0.5f * meas;
            w = fminf(fmaxf(w, 0.5f / G), 2.f / G);
            wsh[b] = w;
            tot += w;
          }
          float run = 0.f;
          st->fused_w[0] = 0;
          for (int b = 0; b < G; ++b) {
            run += wsh[b];
            st->fused_w[b + 1] = b + 1 == G ? 16777216u : (uint32_t)fminf(run / tot * 16777216.f, 16777216.f);
          }
          st->fused_w_valid = G;
          st->fused_done = 0;
          __threadfence();
        }
      }
    }
  }
#ifdef LSW_TUNING
  if (threadIdx.x == 0 && args.seg_trace) {      // slot 510: this CTA's end time and SM (tail analysis)
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    args.seg_trace[((size_t)blockIdx.x * 512 + 510) * 2 + 0] = (uint32_t)globaltimer();
    args.seg_trace[((size_t)blockIdx.x * 512 + 510) * 2 + 1] = smid + 1;
  }
#endif
  if (threadIdx.x == 0) {
    SwitchParams p{};
    p.mode = args.mode;
    p.state = args.state;
    finish_pass(p, s_parity, cf);
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

static bool encode_w(CUtensorMap* m, const void* base, uint64_t d_in, uint64_t d_out, uint64_t L) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d_in, d_out, L};
  cuuint64_t strides[2] = {d_in * 2, d_in * d_out * 2};
  cuuint32_t box[3] = {(cuuint32_t)kSubCols, (cuuint32_t)kTM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Row-major 4-D view {64, d_in / 64, d_out, L}, box {64, 2, 128, 1}: one op
// moves a 128 x 128 tile with each row's 256 B requested (and laid out in
// shared memory) contiguously; needs d_in % 64 == 0.
static bool encode_w_rm(CUtensorMap* m, const void* base, uint64_t d_in, uint64_t d_out, uint64_t L) {
  auto enc = get_encode();
  if (!enc || d_in % 64) return false;
  cuuint64_t dims[4] = {64, d_in / 64, d_out, L};
  cuuint64_t strides[3] = {128, d_in * 2, d_in * d_out * 2};
  cuuint32_t box[4] = {64, 2, (cuuint32_t)kTM, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static bool encode_any(CUtensorMap* m, const void* base, uint64_t d_in, uint64_t d_out, uint64_t L, bool rm) {
  return rm ? encode_w_rm(m, base, d_in, d_out, L) : encode_w(m, base, d_in, d_out, L);
}

// bf16 [rows, rp] already laid out as an operand (pre-swizzled): box {rp,
// box_rows}, no TMA swizzle -- a plain 2-D block copy
static bool encode_rows(CUtensorMap* m, const void* base, uint64_t rows, uint32_t rp, uint32_t box_rows) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {rp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)rp * 2};
  cuuint32_t box[2] = {rp, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static uint32_t align1k(uint32_t x) { return (x + 1023) & ~1023u; }

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& sp, int num_sms, const char** why, int pt) {
  *out = nullptr;
  int dev = 0, major = 0, minor = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) { *why = "needs an sm_100 (B200) device"; return cudaErrorNotSupported; }
  const int r = sp.rank, rp = r <= 16 ? 16 : r <= 32 ? 32 : 64;
  if (r > 64) { *why = "rank > 64"; return cudaErrorNotSupported; }
  TcPlan* plan = new TcPlan();
  Geom& g = plan->geom;
  memset(&g, 0, sizeof(g));
  g.tk.n_layers = sp.n_layers;
  g.n_experts = sp.n_experts;
  g.rp = rp;
  g.swz_mode = rp == 16 ? 6u : rp == 32 ? 4u : 2u;        // SWIZZLE_32B / 64B / 128B (UMMA encoding)
  g.term_bytes = kTM * rp * 2;
  const int mt = 2 * sp.top_k;
  // per-term mode (LSW_FC_PT=1, or chosen by the dispatcher): B raw, A units of
  // kPtGroup terms, TMEM buffers of kPtGroup x 128 columns
  g.pt = pt != 0;
  g.bu = pt == 2;
  if (g.pt) {
    g.acc_cols = kPtGroup * kTN;
    g.acc_bufs = 512 / (int)g.acc_cols;
    g.a_stage_bytes = align1k((uint32_t)(g.bu ? 2 : 1) * kPtGroup * g.term_bytes);
    g.b_buf_bytes = g.bu ? 0 : align1k((uint32_t)mt * g.term_bytes);
  } else {
    g.acc_cols = kTN;
    g.acc_bufs = kAccBufs;
    g.a_stage_bytes = align1k((uint32_t)mt * g.term_bytes);
    g.b_buf_bytes = align1k((uint32_t)(2 * mt) * g.term_bytes);
  }
  const uint32_t w_stage = 2 * kSubBytes;
  const int bb_opt = (int)opt_int("fc_bbufs", 0), as_opt = (int)opt_int("fc_astages", 0),
            ws_opt = (int)opt_int("fc_stages", 0);
  // Shared-memory plan for an A stage of `asb` bytes, in order of preference
  // (measured, 7B shape: W 3 + B 2 + A 3 0.895 of the copy peak vs W 4 + B 1 +
  // A 3 0.868 -- a single B buffer drains the MMA pipeline at every strip
  // change, a 4th W stage buys nothing); what is left goes to more W stages.
  auto make_plan = [&](uint32_t asb, bool w3_first = false) -> bool {
    const int64_t budget = 227 * 1024 - 1024 /*align*/ - 2048 /*static*/;
    // A ring depth in units per tile u (fold: the whole tile's slices; per-term:
    // one unit per kPtGroup terms).  Candidates (W stages, B buffers) in order of
    // preference -- three W stages first: a fourth puts more W requests in flight
    // than the HBM stream wants (k = 1, same box: W 3 + B 2 + A 4 0.895 vs W 4 +
    // B 2 + A 3 0.85; the W-stream probe itself 0.872 with 4 stages vs 0.91 with
    // 3); for each the A stages that fit.  Pass 0 wants 2u + 1 A units
    // (a tile of lookahead), pass 1 u + 1, pass 2 any >= 2; W stays >= 3 before
    // the last resort (measured, 16-layer 7B shape: W 2 costs 7-15 %; W 3 + B 1
    // + A 3 0.860 vs W 4 + B 1 + A 2 0.846 at k = 3; per-term r = 32 k = 3:
    // W 3 + B 1 + A 5 0.656 vs W 3 + B 2 + A 2 0.626).
    // Fold mode with run-time chunk claims (r02): four W stages and one B
    // buffer first -- W 4 + B 1 + A 4 vs W 3 + B 2 + A 4, same box: 7B 0.930
    // vs 0.918 of the copy peak, Mistral 0.932 vs 0.918, r = 8 k = 2 0.926 vs
    // 0.914, r = 4 k = 1 0.937 vs 0.924 (the static deal preferred W 3, see
    // above: its tail hid the difference)
    struct Cand { int ws, bb; };
    const Cand cands_pt[] = {{3, 2}, {3, 1}, {4, 2}, {4, 1}};
    const Cand cands_fold[] = {{4, 1}, {3, 2}, {3, 1}, {4, 2}};
    const Cand* cands = g.pt || w3_first ? cands_pt : cands_fold;
    const int u = g.pt ? (mt + kPtGroup - 1) / kPtGroup : 1;
    const int bb_min = g.bu ? 0 : 1;           // bu: no strip buffer
    if (bb_opt >= bb_min && bb_opt <= 2 && as_opt >= 2 && as_opt <= kMaxAStages && ws_opt >= 2 &&
        ws_opt <= kMaxStages &&
        budget >= (int64_t)bb_opt * g.b_buf_bytes + (int64_t)as_opt * asb + (int64_t)ws_opt * w_stage) {
      g.w_stages = ws_opt;                     // variant option: an explicit plan (all three set)
      g.a_stages = as_opt;
      g.b_bufs = g.bu ? 0 : bb_opt;
      return true;
    }
    for (int pass = 0; pass < 3; ++pass) {
      const int a_min = pass == 0 ? 2 * u + 1 : pass == 1 ? u + 1 : 2;
      for (int ci = 0; ci < 4; ++ci) {
        const Cand& c = cands[ci];
        const int bb = g.bu ? 0 : c.bb;
        const int64_t rest = budget - (int64_t)c.ws * w_stage - (int64_t)bb * g.b_buf_bytes;
        if (rest < 0) continue;
        int as = (int)(rest / asb);
        if (as > kMaxAStages) as = kMaxAStages;
        if (as < a_min) continue;
        g.w_stages = c.ws;
        g.a_stages = as;
        g.b_bufs = bb;
        return true;
      }
    }
    for (int bb = g.bu ? 0 : 2; bb >= bb_min; --bb) {   // last resort: two W stages
      const int64_t rest = budget - 2 * (int64_t)w_stage - (int64_t)bb * g.b_buf_bytes;
      int as = rest > 0 ? (int)(rest / asb) : 0;
      if (as > kMaxAStages) as = kMaxAStages;
      if (as < 2) continue;
      g.w_stages = 2;
      g.a_stages = as;
      g.b_bufs = bb;
      return true;
    }
    return false;
  };
  // tb (fold mode with k >= 3, or option tc_tb = 1): the (hi, lo) B strip in TMEM --
  // b_bufs buffers of mt * rp columns next to >= 2 accumulators -- so shared
  // memory holds only the W stages, ONE raw B strip and the A^T units; the
  // strip change costs no MMA drain (measured: DESIGN.md §5)
  bool ok = false;
  if (!g.pt && opt_int("tc_tb", 0) == 1) {
    const int bcols = mt * rp;                 // (hi, lo) of a term: rp 32-bit columns
    int bb = 0, accb = 0;
    if (512 - 2 * bcols >= 2 * kTN && opt_int("tc_tb_bbufs", 2) != 1) { bb = 2; accb = (512 - 2 * bcols) / kTN; }
    else if (512 - bcols >= 2 * kTN) { bb = 1; accb = (512 - bcols) / kTN; }
    if (accb > kAccBufs) accb = kAccBufs;
    int U = (int)(16384 / g.term_bytes);
    if (U < 1) U = 1;
    if (U > mt) U = mt;
    const uint32_t unit = align1k((uint32_t)U * g.term_bytes), raw = align1k((uint32_t)mt * g.term_bytes);
    const int64_t budget = 227 * 1024 - 1024 /*align*/ - 2048 /*static*/;
    const int ws = ws_opt >= 2 && ws_opt <= kMaxStages ? ws_opt : 3;
    const int64_t rest = budget - (int64_t)ws * w_stage - raw;
    int as = rest > 0 ? (int)(rest / unit) : 0;
    if (as > kMaxAStages) as = kMaxAStages;
    if (as_opt >= 2 && as_opt <= as) as = as_opt;
    if (bb > 0 && as >= 2) {
      g.tb = 1;
      g.b_bufs = bb;
      g.acc_bufs = accb;
      g.acc_cols = kTN;
      g.w_stages = ws;
      g.a_stages = as;
      g.unit_terms = U;
      g.a_stage_bytes = unit;
      g.bcols = (uint32_t)bcols;
      g.b_col0 = (uint32_t)accb * kTN;
      g.raw_bytes = raw;
      // measured (7B, r = 16 k = 3 / 4): releasing a tile's units from the
      // epilogue (one commit per tile) is 5-10 % slower than a commit per unit
      g.unit_commit = opt_int("fc_unit_commit", 1) != 0 || as < 2 * ((mt + U - 1) / U);
      ok = true;
    }
  }
  if (!ok) ok = make_plan(g.a_stage_bytes);
  // CTA pairs (fold mode, variant option tc_pair = 1; off by default): each
  // CTA stages half of a tile's A^T columns (the same shared memory holds twice
  // the A lookahead) and the leader issues the pair's M = 256 MMAs.  Measured
  // (13B, same box): 12.6 vs 9.57 ms per switch -- the per-tile trace shows the
  // A stage cycle stretched from 1.4 to 6.5 us by the cross-CTA chain (the
  // leader's commit frees the follower's stage, the follower refills it and
  // reports it back before the leader's next MMA) and the W stages held longer
  // by the pair's lockstep.
  {
    const long pair_opt = opt_int("tc_pair", 0);
    const bool want = !g.pt && !g.tb && pair_opt == 1 && num_sms >= 2 && opt_int("tc_grid", 0) != 1;
    if (want) {
      const uint32_t half = align1k((uint32_t)mt * g.term_bytes / 2);
      const Geom keep = g;
      if (make_plan(half)) {
        g.pair = 1;
        g.a_stage_bytes = half;
        ok = true;
      } else {
        g = keep;
      }
    }
  }
  if (!ok) { delete plan; *why = "shared memory: rank * top_k too large for the folded kernel"; return cudaErrorNotSupported; }
  // sweep chunk: one q-row strip (d_model / 128 tiles) when that is 24..64,
  // else 48.  Measured (r02, same box, median of 2 x 12 passes): 13B (40-tile
  // strips) 48 -> 40: 10.04 -> 9.77 ms; 7B (32-tile strips) 48 vs 32: equal
  // within 0.3 %
  {
    const int64_t strip = ((int64_t)sp.kind[LSW_Q].d_in + kTN - 1) / kTN;
    if (strip >= 24 && strip <= 64) plan->chunk = (int)strip;
  }
  plan->chunk = (int)opt_int("tc_chunk", plan->chunk);
  if (plan->chunk < 1) plan->chunk = 1;
  plan->probe = (int)probe_int("tc_probe") & 17;
#ifdef LSW_TUNING
  { const char* v = opt_str("trace_buf"); plan->trace = v ? reinterpret_cast<uint32_t*>(strtoull(v, nullptr, 10)) : nullptr; }
  { const char* v = opt_str("seg_trace_buf"); plan->seg_trace = v ? reinterpret_cast<uint32_t*>(strtoull(v, nullptr, 10)) : nullptr; }
#endif
  plan->fused_probe = (int)probe_int("fc_fused_probe") & 29;
  plan->fused_adapt = opt_int("fc_adapt", 1) != 0;
  plan->sweep_dyn = opt_int("fc_dyn", 1) != 0;   // tuning builds only: 1 W stream only, 4 no segment wait, 8 no GEMV, 16 no fold math
  // measured (7B, same box, 3 pairs): W-stream probe 0.865 -> 0.878 of the copy
  // peak, full kernel +0.3-1.5 % with the conflict-free epilogue order
  g.wrm = opt_int("fc_wrm", 1) != 0;
  for (int k = 0; k < LSW_NKIND; ++k) if (sp.kind[k].d_in % 64) g.wrm = 0;   // ragged TP shards: 3-D boxes
  g.smem_bytes = g.w_stages * w_stage + g.a_stages * g.a_stage_bytes + (g.tb ? g.raw_bytes : g.b_bufs * g.b_buf_bytes) +
                 1024;
  // the fused decode keeps three W stages first (measured, 7B, same box: W 3
  // + B 2 + A 4 5.74-5.77 vs W 4 + B 1 + A 4 5.84 ms per token)
  if (!g.pt && !g.tb && !g.pair) {
    const Geom keep = g;
    if (make_plan(g.a_stage_bytes, true)) {
      plan->fw_stages = g.w_stages;
      plan->fa_stages = g.a_stages;
      plan->fb_bufs = g.b_bufs;
      plan->fsmem_bytes = g.w_stages * w_stage + g.a_stages * g.a_stage_bytes + g.b_bufs * g.b_buf_bytes + 1024;
    }
    g = keep;
  }
  // tiles
  int64_t t = 0;
  for (int k = 0; k < LSW_NKIND; ++k) {
    const KindGeom& kg = sp.kind[k];
    g.tk.row_tiles[k] = (int32_t)((kg.d_out + kTM - 1) / kTM);
    g.tk.col_tiles[k] = (int32_t)((kg.d_in + kTN - 1) / kTN);
    // packed B rows padded to an even number of row tiles: a pair's second
    // tile past d_out reads zeros
    g.dout_pad[k] = (int64_t)((g.tk.row_tiles[k] + 1) / 2 * 2) * kTM;
    g.d_in[k] = kg.d_in;
    g.d_out[k] = kg.d_out;
    g.tk.tile_begin[k] = t;
    t += (int64_t)sp.n_layers * g.tk.row_tiles[k] * g.tk.col_tiles[k];
  }
  g.tiles_total = t;
  // pair geometry: the row tiles of each matrix taken two by two
  g.tkp = g.tk;
  {
    int64_t tp = 0;
    for (int k = 0; k < LSW_NKIND; ++k) {
      g.tkp.row_tiles[k] = (g.tk.row_tiles[k] + 1) / 2;
      g.tkp.tile_begin[k] = tp;
      tp += (int64_t)sp.n_layers * g.tkp.row_tiles[k] * g.tkp.col_tiles[k];
    }
    g.tiles_pair = tp;
  }
  plan->grid = (int)(t < num_sms ? t : num_sms);
  { const int x = (int)opt_int("tc_grid", 0); if (x >= 1 && x < plan->grid) plan->grid = x; }
  if (plan->grid < 1) plan->grid = 1;
  if (g.pair) {                                  // clusters of 2: an even grid, <= 2 per pair tile
    int gp = num_sms / 2 * 2;
    if (gp > 2 * g.tiles_pair) gp = (int)(2 * g.tiles_pair);
    { const int x = (int)opt_int("tc_grid", 0); if (x >= 2 && x < gp) gp = x / 2 * 2; }
    plan->pair_grid = gp < 2 ? 2 : gp;
  }
  // pack operands + encode maps (same packed images as the term-group kernel,
  // with 128-column A^T blocks)
  const int64_t M = (int64_t)sp.n_layers * sp.n_experts;
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < LSW_NKIND && e == cudaSuccess; ++k) {
    const KindGeom& kg = sp.kind[k];
    const int64_t din_pad = (int64_t)g.tk.col_tiles[k] * kTN;
    const size_t at_bytes = (size_t)M * din_pad * rp * 2;
    const size_t b_bytes = (size_t)M * g.dout_pad[k] * rp * 2;
    e = cudaMalloc(&plan->packed_At[k], at_bytes);
    if (e != cudaSuccess) break;
    e = cudaMalloc(&plan->packed_B[k], b_bytes);
    if (e != cudaSuccess) break;
    plan->bytes += at_bytes + b_bytes;
    pack_At_kernel<<<2048, 256>>>((const __nv_bfloat16*)kg.A, (__nv_bfloat16*)plan->packed_At[k], sp.n_layers,
                                  sp.n_experts, r, rp, kg.d_in, g.tk.col_tiles[k], kTN);
    pack_B_kernel<<<2048, 256>>>((const __nv_bfloat16*)kg.B, (__nv_bfloat16*)plan->packed_B[k], M, r, rp,
                                 kg.d_out, g.dout_pad[k]);
    g.At[k] = (const __nv_bfloat16*)plan->packed_At[k];
    g.Bp[k] = (const __nv_bfloat16*)plan->packed_B[k];
    if (!encode_any(&plan->maps.w[k], kg.W, kg.d_in, kg.d_out, sp.n_layers, g.wrm) ||
        !encode_rows(&plan->maps.at[k], plan->packed_At[k], (uint64_t)M * din_pad, (uint32_t)rp, kTN / 2)) {
      *why = "cuTensorMapEncodeTiled failed";
      e = cudaErrorInvalidValue;
    }
  }
  if (e == cudaSuccess) e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(switch_fc_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)g.smem_bytes);
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(switch_fc_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(plan->fsmem_bytes > g.smem_bytes ? plan->fsmem_bytes : g.smem_bytes));
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(switch_fc_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)g.smem_bytes);
  if (e == cudaSuccess && g.pair)
    e = cudaFuncSetAttribute(switch_fc_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)g.smem_bytes);
  if (e == cudaSuccess && g.tb)
    e = cudaFuncSetAttribute(switch_fc_kernel<false, false, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g.smem_bytes);
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
  for (int k = 0; k < LSW_NKIND; ++k) {
    cudaFree(plan->packed_At[k]);
    cudaFree(plan->packed_B[k]);
  }
  cudaFree(plan->d_segs);
  cudaFree(plan->d_seg_done);
  cudaFree(plan->d_ys_fx);
  delete plan;
}

int64_t tc_plan_bytes(const TcPlan* plan) { return plan ? plan->bytes : 0; }
int tc_plan_grid(const TcPlan* plan) { return plan ? (plan->geom.pair ? plan->pair_grid : plan->grid) : 0; }
int tc_plan_tile_n(const TcPlan* plan) { return plan ? kTN : 0; }
int tc_plan_pair(const TcPlan* plan) { return plan ? plan->geom.pair : 0; }
int tc_plan_tb(const TcPlan* plan) { return plan ? plan->geom.tb : 0; }
int64_t tc_plan_tiles(const TcPlan* plan) { return plan ? plan->geom.tiles_total : 0; }
const void* tc_plan_packed_B(const TcPlan* plan, int kind, int64_t* dout_pad, int* rp) {
  *dout_pad = plan->geom.dout_pad[kind];
  *rp = plan->geom.rp;
  return plan->packed_B[kind];
}

cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& sp) {
  for (int k = 0; k < LSW_NKIND; ++k)
    if (!sp.kind[k].P ||
        !encode_any(&plan->maps.p[k], sp.kind[k].P, sp.kind[k].d_in, sp.kind[k].d_out, sp.n_layers, plan->geom.wrm))
      return cudaErrorInvalidValue;
  return cudaSuccess;
}

int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0) {
  const Geom& g = plan->geom;
  const int64_t per = (int64_t)g.tk.row_tiles[kind] * g.tk.col_tiles[kind];
  *t0 = g.tk.tile_begin[kind] + (int64_t)layer * per;
  return per;
}

cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0,
                             int64_t t_count) {
  Args a;
  a.t0 = t0;
  a.t_count = t_count;
  a.g = plan->geom;
  a.chunk = plan->chunk;
  a.probe = plan->probe;
  a.mode = p.mode;
  a.top_k = p.top_k;
  a.n_experts = p.n_experts;
  a.scale = p.scale;
  a.cur_idx = p.cur_idx;
  a.cur_g = p.cur_g;
  a.state = p.state;
  a.segs = nullptr;
  a.n_seg = 0;
  a.xs = nullptr;
  a.ys = nullptr;
  a.ys_fx = nullptr;
  a.seg_done = nullptr;
  a.trace = plan->trace;
  a.seg_trace = plan->seg_trace;
  a.dyn = plan->sweep_dyn;
  a.adapt = 0;
  if (plan->geom.pt) {
    switch_fc_kernel<false, true><<<plan->grid, kThreads, plan->geom.smem_bytes, s>>>(plan->maps, a);
  } else if (plan->geom.tb) {
    switch_fc_kernel<false, false, false, true><<<plan->grid, kThreads, plan->geom.smem_bytes, s>>>(plan->maps, a);
  } else if (plan->geom.pair && t_count == 0) {
    // CTA pairs (the per-matrix ablation keeps single CTAs: its tile ranges are single-CTA tiles)
    cudaLaunchConfig_t lc{};
    lc.gridDim = dim3(plan->pair_grid);
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = plan->geom.smem_bytes;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    return cudaLaunchKernelEx(&lc, switch_fc_kernel<false, false, true>, plan->maps, a);
  } else {
    switch_fc_kernel<false, false><<<plan->grid, kThreads, plan->geom.smem_bytes, s>>>(plan->maps, a);
  }
  return cudaGetLastError();
}

// Fused switch + decode: segment table in decoder order (layer, group), built
// once per ctx.
cudaError_t tc_plan_set_fused(TcPlan* plan, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]) {
  const Geom& g = plan->geom;
  if (g.pt || g.tb) return cudaErrorNotSupported;            // the fused epilogue is the shared-memory fold's
  for (int k = 0; k < LSW_NKIND; ++k) if (g.d_in[k] % 8) return cudaErrorNotSupported;   // 16-B x loads
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
        yo += g.d_out[kd];
        S.y_rows += g.d_out[kd];
        S.tile_count += (int64_t)g.tk.row_tiles[kd] * g.tk.col_tiles[kd];
      }
      t += S.tile_count;
      if (S.y_off[0] + S.y_rows > plan->ys_rows) plan->ys_rows = S.y_off[0] + S.y_rows;
    }
  cudaError_t e = cudaSuccess;
  if (!plan->d_ys_fx) e = cudaMalloc(&plan->d_ys_fx, sizeof(unsigned long long) * plan->ys_rows);
  if (e == cudaSuccess && !plan->d_segs) e = cudaMalloc(&plan->d_segs, sizeof(FusedSeg) * n);
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
  if (e == cudaSuccess) e = cudaMemsetAsync(plan->d_ys_fx, 0, sizeof(unsigned long long) * plan->ys_rows, s);
  if (e != cudaSuccess) return e;
  Args a;
  a.t0 = 0;
  a.t_count = plan->fused_tiles;
  a.g = plan->geom;
  a.chunk = 1;                     // unused: per-segment ranges (fused_from)
  a.probe = plan->fused_probe;     // tuning builds only: 1 = W stream only, 4 = no segment wait, 8 = no GEMV (results wrong)
  a.mode = p.mode;
  a.top_k = p.top_k;
  a.n_experts = p.n_experts;
  a.scale = p.scale;
  a.cur_idx = p.cur_idx;
  a.cur_g = p.cur_g;
  a.state = p.state;
  a.segs = plan->d_segs;
  a.n_seg = plan->n_segs;
  a.xs = static_cast<const __nv_bfloat16*>(xs);
  a.ys = ys;
  a.ys_fx = plan->d_ys_fx;
  a.seg_done = plan->d_seg_done;
  a.trace = plan->trace;
  a.seg_trace = plan->seg_trace;
  a.adapt = plan->fused_adapt;
  a.dyn = 0;
  uint32_t smem = plan->geom.smem_bytes;
  if (plan->fsmem_bytes) {                        // the fused decode's own stage plan (W 3 first)
    a.g.w_stages = plan->fw_stages;
    a.g.a_stages = plan->fa_stages;
    a.g.b_bufs = plan->fb_bufs;
    smem = plan->fsmem_bytes;
  }
  switch_fc_kernel<true, false><<<plan->grid, kThreads, smem, s>>>(plan->maps, a);
  return cudaGetLastError();
}

}  // namespace fc
}  // namespace lsw
