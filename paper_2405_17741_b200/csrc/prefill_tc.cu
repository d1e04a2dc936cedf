// prefill_tc.cu -- the unmerged prefill of one GEMV group for T prompt tokens
// on the 5th-gen tensor cores ("For the prefilling
// phase, we have not implemented specific optimizations"): every token t
// carries its own pre-gated decision (idx[t], gate[t]), so nothing can be
// merged and Eq. 2 is evaluated as written,
//     Y[t] = W x_t + sum_j (alpha/r) g_tj B_{e_tj} (A_{e_tj} x_t).
//
// Three launches per group, all our kernels (no library GEMM):
//  1. LoRA-down, prefill_gemm<MODE_U>: U[t][q][e*r + rho] = A_q[e][rho, :] . x_t
//     for EVERY expert e of every site q -- the bank A_q [N, r, d_in] is one
//     [N*r, d_in] K-major matrix, so this is a dense GEMM with N*r rows (N/k
//     times the products a gather would need, on tensor cores, reading A once).
//     Few row tiles, so K is split over the grid; fp32 partials per split.
//  2. prefill_zbuild: Z[t][q][e*rp + rho] = c_t(e) * sum_split U, with
//     c_t(e) = sum_j [e_tj == e] (alpha/r) g_tj (zero for experts t did not
//     select), stored as an exact-to-2^-16 pair of bf16 parts (hi, lo) --
//     the coefficient and U are not rounded to bf16 (R13) -- in the
//     pre-swizzled K-major layout of a tcgen05 operand.
//  3. prefill_gemm<MODE_Y>: one tile = 128 output rows x 128 tokens,
//        D = W_tile . X_tile^T                    (K = d_in, TMA 128B-swizzled boxes)
//          + sum_e B_e,tile . (Zhi_e + Zlo_e)^T   (K = 2 N rp, bulk copies)
//     accumulated in fp32 in TMEM by one chain of tcgen05.mma (M = 128,
//     N = 128) -- the LoRA-up term is just N*2*rp more K of the same
//     contraction -- then written to Y (fp32) by the epilogue warps.
// Single-CTA launches (no CTA pairs, top_k <= 4, not under stream capture;
// option pf_fuse_u, default on) fold 1 and 2 into 3: the launch's first tiles
// are A-bank tiles (128 bank rows x one token tile), whose epilogue forms z =
// c_t(e) u from TMEM and stores the (hi, lo) Z slots itself, then counts the
// tile in a monotonic device word; a W tile's producer waits for this launch's
// count before its first LoRA-up stage.  When the launch is one wave each bank
// tile's K is split over two CTAs (option pf_bank_split): half 0's fp32
// partial goes through U, half 1 adds it (fixed order) and builds Z.  One
// launch instead of three.
// Warp roles: 0 TMA/bulk producer, 1 MMA issuer (+ TMEM alloc), 2-5 epilogue
// (TMEM lane quarter = warp % 4).  Persistent grid, tiles dealt round-robin
// with the token tile fastest, so the CTAs that share a W strip run together
// (one HBM read of W per strip, the X tiles stay in L2).
#include <cstdlib>
#include <cstring>

#include "tc_common.cuh"

namespace lsw {
namespace pf {

using namespace tcx;

constexpr int kTM = 128;        // output rows per tile (UMMA M, TMEM lanes)
constexpr int kTTMax = 256;     // tokens per tile (UMMA N, accumulator columns): 128 or 256
constexpr int kKB = 64;         // K per dense stage: one 128-B swizzle box
constexpr int kBoxBytes = kTM * kKB * 2;       // 16 KB
constexpr int kEpiWarps = 4;
constexpr int kThreads = 32 * (2 + kEpiWarps);
constexpr int kMaxStages = 8;
constexpr int kAccBufs = 2;
constexpr int kMaxSplits = 16;  // LoRA-down K splits at most
constexpr int MODE_Y = 0, MODE_U = 1;

struct Maps {
  CUtensorMap op[3];   // MODE_Y: W of site q [L, d_out, d_in]; MODE_U: A of site q [L, N*r, d_in]
  CUtensorMap x;       // X [T, d_in]
  CUtensorMap a[3];    // MODE_Y with fuse_u: A of site q [L, N*r, d_in]
};
// CTA pairs: every operand moved by a tensor copy (so that the follower's
// copies can complete on the leader's barrier)
struct PairMaps {
  CUtensorMap op[3];   // W of site q [L, d_out, d_in], box {64, 128}, 128-B swizzle
  CUtensorMap x;       // X [T, d_in], box {64, kTT/2}, 128-B swizzle
  CUtensorMap b[3];    // packed B of site q's kind as [L*N*dout_pad, rp] (pre-swizzled), box {rp, 128}, no swizzle
  CUtensorMap z;       // Z as [rows, rp] (pre-swizzled), box {rp, kTT/2}, no swizzle
};

struct Args {
  int32_t mode, n_sites, layer, n_tt, n_kb, splits, total_tiles;
  int32_t row_tiles_total;
  int32_t tile_row0[4];          // prefix sums of the sites' row tiles
  int64_t rows_valid[3];         // output rows per site (d_out or N*r)
  int64_t col0[3];               // column of site q's row 0 in the output row
  int64_t ld;                    // output row stride (elements)
  int64_t T;
  float* out;                    // MODE_Y: Y [T, ld]; MODE_U: U [splits, T, ld]
  // MODE_Y LoRA-up stages
  int32_t n_experts, rp;
  uint32_t term_bytes;           // 128 x rp bf16 (one B slice)
  uint32_t zpart_bytes;          // kTT x rp bf16 (one Z part)
  uint32_t swz;                  // UMMA layout type of the rp-wide operands
  const __nv_bfloat16* Bp[3];    // site q: packed B of this layer [N, dout_pad, rp], pre-swizzled
  int64_t dout_pad[3];
  const __nv_bfloat16* Z;        // [n_tt][n_sites][N][2][kTT][rp], pre-swizzled
  uint32_t stage_bytes, b_off;   // stage = [A part | B part at b_off]
  int32_t stages;
  int32_t pair_row0[4];          // CTA pairs: prefix sums of the sites' row-tile PAIRS
  // MODE_Y, fuse_u: the LoRA-down products and Z built by the same launch.  The
  // first a_tiles tiles are A-bank tiles (site q's rows e*r + rho of A_q x one
  // token tile, full K); their epilogue writes the gate-scaled (hi, lo) Z slots
  // straight from TMEM and counts itself in *zdone; a W tile's producer waits
  // for *zdone == a_tiles before its first LoRA-up stage
  int32_t a_tiles;
  int32_t a_row0[4];             // prefix sums of the sites' A-bank row tiles
  int32_t k, r;
  float scale;
  uint32_t* zdone;               // monotonic count of A-bank tiles done (plan-owned word)
  uint32_t z_target;             // *zdone after this launch's A-bank tiles (mod 2^32)
  // a_split == 2: each A-bank tile's K in two halves on two CTAs (iterations
  // 2j, 2j+1): half 0 stores its fp32 partial to Pp [j][kTT][128] and counts
  // in *pdone; half 1 waits for *pdone == p_target, adds the partial (half 0
  // first: fixed order) and builds Z.  a_tiles counts iterations.
  int32_t a_split;
  uint32_t* pdone;
  uint32_t p_target;
  float* Pp;
  const int32_t* idx;            // [T, k]
  const float* gate;             // [T, k]
  __nv_bfloat16* Zw;             // = Z, written by the A-bank tiles
};

struct TileAt {
  int q, rb, tt, kb0, kb1;
  int half, j;                   // fuse_u, split bank tiles: K half (0 | 1), bank tile index
};

__device__ __forceinline__ TileAt tile_at(const Args& a, int t) {  // token tile fastest
  TileAt r;
  r.tt = t % a.n_tt;
  int rest = t / a.n_tt;
  int split = 0;
  if (a.mode == MODE_U) {
    split = rest / a.row_tiles_total;
    rest -= split * a.row_tiles_total;
  }
  r.q = (a.n_sites > 2 && rest >= a.tile_row0[2]) ? 2 : (a.n_sites > 1 && rest >= a.tile_row0[1]) ? 1 : 0;
  r.rb = rest - a.tile_row0[r.q];
  if (a.mode == MODE_U) {
    r.kb0 = (int)((int64_t)a.n_kb * split / a.splits);
    r.kb1 = (int)((int64_t)a.n_kb * (split + 1) / a.splits);
  } else {
    r.kb0 = 0;
    r.kb1 = a.n_kb;
  }
  return r;
}

__device__ __forceinline__ uint32_t ld_acquire_gpu_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Wait until the monotonic count *p reaches target (mod 2^32), with a ~20 s
// watchdog: a protocol bug traps (sticky error) instead of hanging the GPU.
__device__ __forceinline__ void wait_count(const uint32_t* p, uint32_t target) {
  if ((int32_t)(ld_acquire_gpu_u32(p) - target) >= 0) return;
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (uint32_t n = 1;; ++n) {
    __nanosleep(32);
    if ((int32_t)(ld_acquire_gpu_u32(p) - target) >= 0) return;
    if ((n & 1023) == 0) {
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();
    }
  }
}

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                            uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}

// Thread-block clusters of kC CTAs along the token-tile dimension (MODE_Y):
// the CTAs of a cluster compute the same 128-row block for kC consecutive
// token tiles in lockstep, so each loads 128/kC rows of the W box and
// multicasts them to all kC CTAs -- W crosses L2 -> SM once per cluster instead
// of once per token tile.  Every stage's MMA completion is committed to the
// `empty` barrier of every CTA of the cluster (count kC), so no CTA refills a
// stage -- its own or, by multicast, a peer's -- before all kC have consumed it.
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_count() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_3d_mc(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                               int32_t c2, uint32_t bar, uint16_t mask, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
      ".L2::cache_hint [%0], [%1, {%2, %3, %4}], [%5], %6, %7;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "h"(mask),
        "l"(policy)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mc(uint32_t bar, uint16_t mask) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"(mask) : "memory");
}

// CTA pairs: arrive on the mbarrier at the same shared offset in CTA `rank`
// of the cluster; the pair's MMA (leader only, M = 256 over both CTAs' A
// halves, N over both CTAs' B halves, same shared offsets); the pair's commit
// multicast to the barrier at this offset in both CTAs
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(bar), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ void umma_f16_pair(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}"
      ::"r"(d_tmem), "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
               ::"r"(bar), "h"((uint16_t)3) : "memory");
}

// Tile of iteration `it` of this CTA: kC == 1 -- global tile index (tile_at);
// kC > 1 -- cluster tile (row block, token-tile group), this CTA's token tile
// = group * kC + rank (may lie past the last token tile: OOB-zero operands,
// masked stores).
template <int kC>
__device__ __forceinline__ TileAt tile_for(const Args& a, int it, int crank, bool& bank) {
  bank = false;
  if constexpr (kC == 1) {
    if (it >= a.a_tiles) {
      return tile_at(a, it - a.a_tiles);
    }
    bank = true;                                 // A-bank tile (fuse_u)
    TileAt r;
    r.j = a.a_split == 2 ? it >> 1 : it;
    r.half = a.a_split == 2 ? it & 1 : 0;
    r.tt = r.j % a.n_tt;
    const int rest = r.j / a.n_tt;
    r.q = (a.n_sites > 2 && rest >= a.a_row0[2]) ? 2 : (a.n_sites > 1 && rest >= a.a_row0[1]) ? 1 : 0;
    r.rb = rest - a.a_row0[r.q];
    r.kb0 = r.half ? a.n_kb / 2 : 0;
    r.kb1 = a.a_split == 2 && !r.half ? a.n_kb / 2 : a.n_kb;
    return r;
  } else {
    const int n_ttg = (a.n_tt + kC - 1) / kC;
    const int rest = it / n_ttg;
    TileAt r;
    r.tt = (it - rest * n_ttg) * kC + crank;
    r.q = (a.n_sites > 2 && rest >= a.tile_row0[2]) ? 2 : (a.n_sites > 1 && rest >= a.tile_row0[1]) ? 1 : 0;
    r.rb = rest - a.tile_row0[r.q];
    r.kb0 = 0;
    r.kb1 = a.n_kb;
    return r;
  }
}

// A-bank tile epilogue (fuse_u): this thread's bank row is expert e, rank
// index rho; for every token t of the tile z = c_t(e) * u_t with u_t the
// full-K fp32 product in TMEM and c_t(e) = sum_j [idx_tj == e] scale * gate_tj
// (j ascending, as the Z build), stored as (hi, lo) bf16 at the pre-swizzled
// slot of Z.  Lane l fetches the decision of token l of each 32-token chunk
// (the next chunk's in flight while this one is processed) and the warp reads
// each token's K entries by shuffle -- K a template parameter, so the 16
// tokens of a TMEM load carry no branches and their shuffles overlap.
__device__ __forceinline__ int shfl_ordered(int v, int src) {
  int r;
  asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(r) : "r"(v), "r"(src));
  return r;
}

template <int K, int kTT>
__device__ __forceinline__ void bank_z(const Args& a, int tt, uint32_t tm, int e, int rho, bool okr,
                                       __nv_bfloat16* blk, int lane, const float* pp) {
  const int64_t t0 = (int64_t)tt * kTT;
  const int rp = a.rp, fmask = rp / 8 - 1, zpart = kTT * rp;
  int id[K];
  float gv[K];
  auto fetch = [&](int c32, int* idr, float* gvr) {
    const int64_t tl = t0 + c32 + lane;
    const bool in = tl < a.T;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      idr[j] = in ? __ldg(a.idx + tl * K + j) : -1;
      gvr[j] = in ? a.scale * __ldg(a.gate + tl * K + j) : 0.f;
    }
  };
  fetch(0, id, gv);
  for (int c32 = 0; c32 < kTT; c32 += 32) {
    int idn[K];
    float gvn[K];
    if (c32 + 32 < kTT) fetch(c32 + 32, idn, gvn);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      uint32_t v[16];
      tmem_ld16(tm + c32 + 16 * h, v);
      float pv[16];
      if (pp) {                                  // half 0's partial of these 16 tokens (this row)
#pragma unroll
        for (int i = 0; i < 16; ++i) pv[i] = __ldcg(pp + (c32 + 16 * h + i) * kTM);
      }
      tmem_wait_ld();
      if (pp) {
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(pv[i] + __uint_as_float(v[i]));
      }
      float c[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        c[i] = 0.f;
#pragma unroll
        for (int j = 0; j < K; ++j) {
          // volatile: the shuffles stay in token order, so their results are
          // consumed as they come instead of all being hoisted (registers)
          const int ij = shfl_ordered(id[j], 16 * h + i);
          const float gj = __int_as_float(shfl_ordered(__float_as_int(gv[j]), 16 * h + i));
          if (ij == e) c[i] += gj;
        }
      }
      if (okr) {
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int tin = c32 + 16 * h + i;
          const float z = c[i] != 0.f ? c[i] * __uint_as_float(v[i]) : 0.f;
          const __nv_bfloat16 hi = __float2bfloat16_rn(z);
          const __nv_bfloat16 lo = __float2bfloat16_rn(z - __bfloat162float(hi));
          // swz_off(tin, rho, rp) in 32-bit arithmetic
          const int off = tin * rp + ((((rho >> 3) ^ ((tin * rp) >> 6)) & fmask) << 3) + (rho & 7);
          blk[off] = hi;
          blk[zpart + off] = lo;
        }
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      id[j] = idn[j];
      gv[j] = gvn[j];
    }
  }
}

template <int kTT, int kC>
__global__ void __launch_bounds__(kThreads, 1)
prefill_gemm(const __grid_constant__ Maps maps, const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint32_t s_tmem_base;
  __shared__ __align__(8) uint64_t bar_full[kMaxStages], bar_empty[kMaxStages];
  __shared__ __align__(8) uint64_t bar_accfull[kAccBufs], bar_accempty[kAccBufs];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool lora = a.mode == MODE_Y && a.n_experts > 0;

  // MODE_U: the Z build launched next (programmatic dependent) may start at
  // once; fused MODE_Y: the next group's launch may take SMs as they free up
  if (a.mode == MODE_U || a.a_tiles) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int crank = kC > 1 ? (int)cluster_rank() : 0;
  const uint16_t cmask = (uint16_t)((1u << kC) - 1);
  const int it0 = kC > 1 ? (int)cluster_id() : blockIdx.x;
  const int istep = kC > 1 ? (int)cluster_count() : gridDim.x;
  const int n_it = kC > 1 ? a.row_tiles_total * ((a.n_tt + kC - 1) / kC) : a.total_tiles;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);
      mbar_init(smem_u32(&bar_empty[s]), kC);         // one MMA commit per CTA of the cluster
    }
    for (int s = 0; s < kAccBufs; ++s) {
      mbar_init(smem_u32(&bar_accfull[s]), 1);
      mbar_init(smem_u32(&bar_accempty[s]), kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < a.n_sites; ++q) {
      prefetch_map(&maps.op[q]);
      if (a.a_tiles) prefetch_map(&maps.a[q]);
    }
    prefetch_map(&maps.x);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&s_tmem_base)), "r"(kAccBufs * kTT) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kC > 1) cluster_sync();          // peers' barriers initialised before any multicast
  tc_fence_after();
  const uint32_t tmem_base = s_tmem_base;

  if (warp == 0) {
    // ============================ producer ==================================
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();     // W / A: streamed once per strip
      const uint64_t pol_x = policy_evict_last();      // X, B, Z: reused by many tiles
      Ring ring{0, 0, (uint32_t)a.stages};
      bool z_ready = false;
      // MODE_U is a programmatic dependent of the previous group's dense
      // launch: its setup (barriers, TMEM, tensor maps) ran already; X (and U,
      // read by the previous Z build) only after that grid has completed
      // (fused MODE_Y likewise: X, and Z / Y still read by the previous group)
      if (a.mode == MODE_U || a.a_tiles) asm volatile("griddepcontrol.wait;" ::: "memory");
      for (int it = it0; it < n_it; it += istep) {
        bool bank;
        const TileAt ta = tile_for<kC>(a, it, crank, bank);
        const CUtensorMap* opmap = bank ? &maps.a[ta.q] : &maps.op[ta.q];
        for (int kb = ta.kb0; kb < ta.kb1; ++kb) {
          mbar_wait(smem_u32(&bar_empty[ring.i]), ring.phase ^ 1);
          uint8_t* st = base + (size_t)ring.i * a.stage_bytes;
          const uint32_t bar = smem_u32(&bar_full[ring.i]);
          mbar_expect_tx(bar, kBoxBytes + kTT * kKB * 2);   // W box (all kC slices) + own X box
          if constexpr (kC > 1) {
            // this CTA's 128/kC rows of the W box, to the same offset of every CTA
            tma_load_3d_mc(smem_u32(st) + crank * (kBoxBytes / kC), &maps.op[ta.q], kb * kKB,
                           ta.rb * kTM + crank * (kTM / kC), a.layer, bar, cmask, pol_w);
          } else {
            tma_load_3d(smem_u32(st), opmap, kb * kKB, ta.rb * kTM, a.layer, bar, pol_w);
          }
          tma_load_2d(smem_u32(st + a.b_off), &maps.x, kb * kKB, ta.tt * kTT, bar, pol_x);   // box {64, kTT}
          ring.next();
        }
        if (lora && !bank) {
          if (!z_ready) {
            if (a.a_tiles) {                     // Z is written by this grid's A-bank tiles
              wait_count(a.zdone, a.z_target);
              asm volatile("fence.proxy.async.global;" ::: "memory");
            } else {                             // Z is written by the preceding (Z build) grid
              asm volatile("griddepcontrol.wait;" ::: "memory");
            }
            z_ready = true;
          }
          for (int e = 0; e < a.n_experts; ++e) {
            mbar_wait(smem_u32(&bar_empty[ring.i]), ring.phase ^ 1);
            uint8_t* st = base + (size_t)ring.i * a.stage_bytes;
            const uint32_t bar = smem_u32(&bar_full[ring.i]);
            mbar_expect_tx(bar, a.term_bytes + 2 * a.zpart_bytes);
            bulk_load(smem_u32(st), a.Bp[ta.q] + ((size_t)e * a.dout_pad[ta.q] + (size_t)ta.rb * kTM) * a.rp,
                      a.term_bytes, bar, pol_x);
            const __nv_bfloat16* z =
                a.Z + ((((size_t)ta.tt * a.n_sites + ta.q) * a.n_experts + e) * 2) * (size_t)kTT * a.rp;
            bulk_load(smem_u32(st + a.b_off), z, 2 * a.zpart_bytes, bar, pol_x);    // hi, lo: contiguous
            ring.next();
          }
        }
      }
      if constexpr (kC > 1) {
        // drain: every stage's last fill released by all kC CTAs, so no peer's
        // commit still targets this CTA's barriers when it leaves
        for (int i = 0; i < a.stages; ++i) {
          mbar_wait(smem_u32(&bar_empty[ring.i]), ring.phase ^ 1);
          ring.next();
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ================================
    // D f32, A/B bf16, both K-major, N = 128 (tokens), M = 128 (rows)
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTT >> 3) << 17) |
                           ((uint32_t)(kTM >> 4) << 24);
    const uint64_t dense0 = umma_desc(0, 1024, 2);                       // 128-B rows, SWIZZLE_128B
    const uint64_t lora0 = umma_desc(0, 8 * (uint32_t)a.rp * 2, a.swz);  // rp-wide rows
    const uint64_t zpart = a.zpart_bytes >> 4;
    Ring ring{0, 0, (uint32_t)a.stages};
    Ring acc{0, 0, kAccBufs};
    for (int it = it0; it < n_it; it += istep) {
      bool bank;
      const TileAt ta = tile_for<kC>(a, it, crank, bank);
      mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
      tc_fence_after();
      const uint32_t d = tmem_base + acc.i * kTT;
      uint32_t accum = 0;
      for (int kb = ta.kb0; kb < ta.kb1; ++kb) {
        mbar_wait(smem_u32(&bar_full[ring.i]), ring.phase);
        tc_fence_after();
        const uint32_t st = smem_u32(base + (size_t)ring.i * a.stage_bytes);
        const uint64_t da = dense0 + (st >> 4), db = dense0 + ((st + a.b_off) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < kKB / 16; ++kk) umma_f16(d, da + kk * 2, db + kk * 2, idesc, accum | kk);
          if constexpr (kC > 1) umma_commit_mc(smem_u32(&bar_empty[ring.i]), cmask);   // every CTA's copy
          else umma_commit(smem_u32(&bar_empty[ring.i]));  // stage free once these MMAs complete
        }
        __syncwarp();
        accum = 1;
        ring.next();
      }
      if (lora && !bank) {
        const int ksteps = a.rp / 16;
        for (int e = 0; e < a.n_experts; ++e) {
          mbar_wait(smem_u32(&bar_full[ring.i]), ring.phase);
          tc_fence_after();
          const uint32_t st = smem_u32(base + (size_t)ring.i * a.stage_bytes);
          const uint64_t da = lora0 + (st >> 4), db = lora0 + ((st + a.b_off) >> 4);
          if (elect_one()) {
            for (int part = 0; part < 2; ++part)
              for (int kk = 0; kk < ksteps; ++kk)
                umma_f16(d, da + kk * 2, db + part * zpart + kk * 2, idesc, 1u);
            if constexpr (kC > 1) umma_commit_mc(smem_u32(&bar_empty[ring.i]), cmask);
            else umma_commit(smem_u32(&bar_empty[ring.i]));
          }
          __syncwarp();
          ring.next();
        }
      }
      if (elect_one()) umma_commit(smem_u32(&bar_accfull[acc.i]));   // accumulator complete
      __syncwarp();
      acc.next();
    }
  } else {
    // ============================ epilogue ==================================
    // thread = one output row of the tile (TMEM lane); 16 token columns per
    // tcgen05.ld; a warp's 32 stores of one token are 128 contiguous bytes
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    Ring acc{0, 0, kAccBufs};
    for (int it = it0; it < n_it; it += istep) {
      bool bank;
      const TileAt ta = tile_for<kC>(a, it, crank, bank);
      mbar_wait(smem_u32(&bar_accfull[acc.i]), acc.phase);
      tc_fence_after();
      if (bank) {
        // Z slots of A-bank row R = e*r + rho: z = c_t(e) * u, u from TMEM
        // (full-K fp32), c_t(e) = sum_j [idx_tj == e] scale * gate_tj -- the
        // Z build's arithmetic, split into (hi, lo) bf16
        const int R = ta.rb * kTM + row;
        const int e = R / a.r, rho = R - e * a.r;
        const bool okr = e < a.n_experts;
        __nv_bfloat16* blk =
            a.Zw + ((((int64_t)ta.tt * a.n_sites + ta.q) * a.n_experts + e) * 2) * (int64_t)kTT * a.rp;
        const uint32_t tm = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * kTT;
        float* pj = a.Pp + (int64_t)ta.j * kTT * kTM + row;   // [j][token][row]
        if (a.a_split == 2 && ta.half == 0) {
          // half 0: the fp32 partial to Pp, counted in *pdone (no Z)
          for (int c0 = 0; c0 < kTT; c0 += 16) {
            uint32_t v[16];
            tmem_ld16(tm + c0, v);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) __stcg(pj + (c0 + i) * kTM, __uint_as_float(v[i]));
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&bar_accempty[acc.i]));
          asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
          if (warp == 2 && lane == 0) {
            __threadfence();
            atomicAdd(a.pdone, 1u);
          }
          acc.next();
          continue;
        }
        const float* pp = nullptr;
        if (a.a_split == 2) {                    // half 1: every half 0 of this launch stored
          if (lane == 0) wait_count(a.pdone, a.p_target);
          __syncwarp();
          pp = pj;
        }
        {
          switch (a.k) {
            case 1: bank_z<1, kTT>(a, ta.tt, tm, e, rho, okr, blk, lane, pp); break;
            case 2: bank_z<2, kTT>(a, ta.tt, tm, e, rho, okr, blk, lane, pp); break;
            case 3: bank_z<3, kTT>(a, ta.tt, tm, e, rho, okr, blk, lane, pp); break;
            case 4: bank_z<4, kTT>(a, ta.tt, tm, e, rho, okr, blk, lane, pp); break;
            default: bank_z<4, kTT>(a, ta.tt, tm, e, rho, okr, blk, lane, pp); break;   // (k <= 4: host)
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_accempty[acc.i]));
        // every epilogue thread's Z stores before the count; the W tiles read
        // Z by bulk copies (async proxy)
        asm volatile("fence.proxy.async.global;" ::: "memory");
        asm volatile("bar.sync 1, %0;" ::"r"(32 * kEpiWarps) : "memory");
        if (warp == 2 && lane == 0) {
          __threadfence();
          atomicAdd(a.zdone, 1u);
        }
        acc.next();
        continue;
      }
      const int64_t grow = (int64_t)ta.rb * kTM + row;
      const bool ok = grow < a.rows_valid[ta.q];
      const int split = a.mode == MODE_U ? it / a.n_tt / a.row_tiles_total : 0;
      float* outp = a.out + (int64_t)split * a.T * a.ld + a.col0[ta.q] + grow;
      const uint32_t tm = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * kTT;
      for (int c0 = 0; c0 < kTT; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tm + c0, v);
        tmem_wait_ld();
        const int64_t tok0 = (int64_t)ta.tt * kTT + c0;
        if (ok) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (tok0 + i < a.T) outp[(tok0 + i) * a.ld] = __uint_as_float(v[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&bar_accempty[acc.i]));
      acc.next();
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (kC > 1) cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAccBufs * kTT)
                 : "memory");
  }
}

// ---------------------------------------------------------------------------
// MODE_Y on CTA pairs (cta_group::2): a pair tile is 256 output rows (two
// row tiles of ONE site, one per CTA of a cluster of 2) x kTT tokens.  Each
// CTA loads its own 128 W rows and HALF of the tile's tokens (X box of kTT/2
// rows; for the LoRA-up stages its B slice and half of Z's hi and lo parts),
// and the leader issues tcgen05.mma.cta_group::2 (M = 256, N = kTT) reading
// both CTAs' shared memory: per CTA and 64-deep K step 32 KB of operands
// instead of 48 KB for the same MACs as a 128 x 256 tile, the dense GEMM's
// bound being the operand feed from L2.  Every copy is a tensor copy with
// .cta_group::2 completing on the LEADER's full barrier (which expects both
// CTAs' bytes), so no stage is relayed between the CTAs; the leader's commits
// are multicast to both CTAs' empty / accumulator barriers; each CTA's
// epilogue reads its own TMEM lanes (its 128 rows) and the follower's
// epilogue releases the accumulator to the leader by a remote arrive.  Pairs
// never straddle two sites: Z (the N operand of the LoRA-up stages) belongs
// to one site.
__device__ __forceinline__ void tma_load_2d_cg2(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d_cg2(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1,
                                                int32_t c2, uint32_t bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;"
      ::"r"(dst), "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}

#ifdef LSW_TUNING
// Tuning builds only (option pf_trace_buf = a device pointer): per CTA of the
// pair launch, per unit: [tile, %smid, accumulator ready, epilogue done]
// (%globaltimer low 32 bits), 16 units per CTA, slot 0 the CTA's start time.
__device__ uint32_t* g_pf_trace = nullptr;
#define PF_TRACE(unit, a0, a1, a2, a3)                                                          \
  do {                                                                                        \
    if (g_pf_trace && (unit) < 15) {                                                          \
      uint32_t* t_ = g_pf_trace + (blockIdx.x * 16 + 1 + (unit)) * 4;                         \
      t_[0] = (a0); t_[1] = (a1); t_[2] = (a2); t_[3] = (a3);                                 \
    }                                                                                         \
  } while (0)
__device__ __forceinline__ uint32_t pf_now() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return (uint32_t)t;
}
__device__ __forceinline__ uint32_t pf_smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#else
#define PF_TRACE(unit, a0, a1, a2, a3) do {} while (0)
#endif

template <int kTT>
__global__ void __launch_bounds__(kThreads, 1)
prefill_gemm_pair(const __grid_constant__ PairMaps maps, const __grid_constant__ Args a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint32_t s_tmem_base;
  __shared__ __align__(8) uint64_t bar_full[kMaxStages], bar_empty[kMaxStages];
  __shared__ __align__(8) uint64_t bar_accfull[kAccBufs], bar_accempty[kAccBufs];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool lora = a.n_experts > 0;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  constexpr int kHalf = kTT / 2;                  // tokens per CTA of a pair tile
  const int it0 = (int)cluster_id(), istep = (int)cluster_count();
  const int n_it = a.pair_row0[a.n_sites] * a.n_tt;
#ifdef LSW_TUNING
  if (g_pf_trace && threadIdx.x == 0) {
    uint32_t* t_ = g_pf_trace + blockIdx.x * 16 * 4;
    t_[0] = pf_now(); t_[1] = pf_smid(); t_[2] = (uint32_t)it0; t_[3] = (uint32_t)istep;
  }
  uint32_t tr_ready = 0, tr_unit = 0;
#endif
  const uint32_t zhalf = (uint32_t)kHalf * a.rp * 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < a.stages; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);          // leader: its producer's arrive + both CTAs' bytes
      mbar_init(smem_u32(&bar_empty[s]), 1);         // the leader's commit, multicast to both CTAs
    }
    for (int s = 0; s < kAccBufs; ++s) {
      mbar_init(smem_u32(&bar_accfull[s]), 1);
      mbar_init(smem_u32(&bar_accempty[s]), 2 * kEpiWarps);   // leader: both CTAs' epilogues
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int q = 0; q < a.n_sites; ++q) {
      prefetch_map(&maps.op[q]);
      if (lora) prefetch_map(&maps.b[q]);
    }
    prefetch_map(&maps.x);
    if (lora) prefetch_map(&maps.z);
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&s_tmem_base)), "r"(kAccBufs * kTT) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                                 // the peer's barriers exist before any copy / commit targets them
  tc_fence_after();
  const uint32_t tmem_base = s_tmem_base;
  // pair tile `it` -> this CTA's (site, row tile, token tile)
  auto tile = [&](int it) {
    TileAt r;
    r.tt = it % a.n_tt;
    const int p = it / a.n_tt;
    r.q = (a.n_sites > 2 && p >= a.pair_row0[2]) ? 2 : (a.n_sites > 1 && p >= a.pair_row0[1]) ? 1 : 0;
    r.rb = 2 * (p - a.pair_row0[r.q]) + (int)crank;
    r.kb0 = 0;
    r.kb1 = a.n_kb;
    return r;
  };

  if (warp == 0) {
    // ============================ producer ==================================
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_first();
      const uint64_t pol_x = policy_evict_last();
      Ring ring{0, 0, (uint32_t)a.stages};
      bool z_ready = false;
      const uint32_t dense_bytes = kBoxBytes + kHalf * kKB * 2, lora_bytes = a.term_bytes + 2 * zhalf;
      for (int it = it0; it < n_it; it += istep) {
        const TileAt ta = tile(it);
        const int units = a.n_kb + (lora ? a.n_experts : 0);
        for (int k = 0; k < units; ++k) {
          if (k == a.n_kb && !z_ready) {          // Z is written by the preceding (Z build) grid
            asm volatile("griddepcontrol.wait;" ::: "memory");
            z_ready = true;
          }
          mbar_wait(smem_u32(&bar_empty[ring.i]), ring.phase ^ 1);
          uint8_t* st = base + (size_t)ring.i * a.stage_bytes;
          const uint32_t fb = smem_u32(&bar_full[ring.i]);
          // the leader's barrier expects both CTAs' bytes; the follower's copies complete on it
          if (leader) mbar_expect_tx(fb, 2 * (k < a.n_kb ? dense_bytes : lora_bytes));
          const uint32_t bar = leader ? fb : mapa_rank(fb, 0);
          if (k < a.n_kb) {
            tma_load_3d_cg2(smem_u32(st), &maps.op[ta.q], k * kKB, ta.rb * kTM, a.layer, bar, pol_w);
            tma_load_2d_cg2(smem_u32(st + a.b_off), &maps.x, k * kKB, ta.tt * kTT + (int)crank * kHalf, bar, pol_x);
          } else {
            const int e = k - a.n_kb;
            tma_load_2d_cg2(smem_u32(st), &maps.b[ta.q], 0,
                            (int)(((int64_t)a.layer * a.n_experts + e) * a.dout_pad[ta.q] + (int64_t)ta.rb * kTM),
                            bar, pol_x);
            const int zr = (int)(((((int64_t)ta.tt * a.n_sites + ta.q) * a.n_experts + e) * 2) * kTT) +
                           (int)crank * kHalf;
            tma_load_2d_cg2(smem_u32(st + a.b_off), &maps.z, 0, zr, bar, pol_x);                  // hi half
            tma_load_2d_cg2(smem_u32(st + a.b_off + zhalf), &maps.z, 0, zr + kTT, bar, pol_x);    // lo half
          }
          ring.next();
        }
      }
      // drain: every stage's last fill consumed by the leader's MMAs, so no
      // commit still targets this CTA's barriers when it leaves
      for (int i = 0; i < a.stages; ++i) {
        mbar_wait(smem_u32(&bar_empty[ring.i]), ring.phase ^ 1);
        ring.next();
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer (leader) =======================
    // D f32, A/B bf16, both K-major, M = 256 (both CTAs' rows), N = kTT
    if (leader) {
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTT >> 3) << 17) |
                             ((uint32_t)((2 * kTM) >> 4) << 24);
      const uint64_t dense0 = umma_desc(0, 1024, 2);
      const uint64_t lora0 = umma_desc(0, 8 * (uint32_t)a.rp * 2, a.swz);
      const uint64_t zpart = zhalf >> 4;
      const int ksteps = a.rp / 16;
      Ring ring{0, 0, (uint32_t)a.stages};
      Ring acc{0, 0, kAccBufs};
      const int units = a.n_kb + (lora ? a.n_experts : 0);
      for (int it = it0; it < n_it; it += istep) {
        mbar_wait(smem_u32(&bar_accempty[acc.i]), acc.phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc.i * kTT;
        for (int k = 0; k < units; ++k) {
          mbar_wait(smem_u32(&bar_full[ring.i]), ring.phase);
          tc_fence_after();
          const uint32_t st = smem_u32(base + (size_t)ring.i * a.stage_bytes);
          if (elect_one()) {
            if (k < a.n_kb) {
              const uint64_t da = dense0 + (st >> 4), db = dense0 + ((st + a.b_off) >> 4);
#pragma unroll
              for (int kk = 0; kk < kKB / 16; ++kk)
                umma_f16_pair(d, da + kk * 2, db + kk * 2, idesc, (k | kk) ? 1u : 0u);
            } else {
              const uint64_t da = lora0 + (st >> 4), db = lora0 + ((st + a.b_off) >> 4);
              for (int part = 0; part < 2; ++part)
                for (int kk = 0; kk < ksteps; ++kk)
                  umma_f16_pair(d, da + kk * 2, db + part * zpart + kk * 2, idesc, 1u);
            }
            umma_commit_pair(smem_u32(&bar_empty[ring.i]));   // both CTAs' stages free when these complete
          }
          __syncwarp();
          ring.next();
        }
        if (elect_one()) umma_commit_pair(smem_u32(&bar_accfull[acc.i]));
        __syncwarp();
        acc.next();
      }
    }
  } else {
    // ============================ epilogue ==================================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    Ring acc{0, 0, kAccBufs};
    for (int it = it0; it < n_it; it += istep) {
      const TileAt ta = tile(it);
      mbar_wait(smem_u32(&bar_accfull[acc.i]), acc.phase);
      tc_fence_after();
#ifdef LSW_TUNING
      tr_ready = pf_now();
#endif
      const int64_t grow = (int64_t)ta.rb * kTM + row;
      const bool ok = grow < a.rows_valid[ta.q];
      float* outp = a.out + a.col0[ta.q] + grow;
      const uint32_t tm = tmem_base + ((uint32_t)(quarter * 32) << 16) + acc.i * kTT;
      for (int c0 = 0; c0 < kTT; c0 += 16) {
        uint32_t v[16];
        tmem_ld16(tm + c0, v);
        tmem_wait_ld();
        const int64_t tok0 = (int64_t)ta.tt * kTT + c0;
        if (ok) {
#pragma unroll
          for (int i = 0; i < 16; ++i)
            if (tok0 + i < a.T) outp[(tok0 + i) * a.ld] = __uint_as_float(v[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(smem_u32(&bar_accempty[acc.i]));
        else mbar_arrive_remote(smem_u32(&bar_accempty[acc.i]), 0);
      }
#ifdef LSW_TUNING
      if (warp == 2 && lane == 0) PF_TRACE(tr_unit, (uint32_t)it, pf_smid(), tr_ready, pf_now());
      ++tr_unit;
#endif
      acc.next();
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();                                 // no copy / commit / remote arrive may target a CTA that left
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kAccBufs * kTT)
                 : "memory");
  }
}

// Z (hi, lo) parts from the split-K LoRA-down partials: one thread per
// (token tile, site, expert, token in tile, rho < rp).
__global__ void prefill_zbuild(const float* __restrict__ U, int splits, int64_t T, int64_t ldu, int n_sites, int N,
                               int r, int rp, int k, float scale, const int32_t* __restrict__ idx,
                               const float* __restrict__ gate, __nv_bfloat16* __restrict__ Z, int n_tt, int kTT) {
  // programmatic dependent of the LoRA-down grid, and primary of the dense
  // grid: let that one start its K loop at once, then wait for U
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const int64_t total = (int64_t)n_tt * n_sites * N * kTT * rp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int rho = (int)(i % rp);
    int64_t rest = i / rp;
    const int tin = (int)(rest % kTT);
    rest /= kTT;
    const int e = (int)(rest % N);
    rest /= N;
    const int q = (int)(rest % n_sites);
    const int tt = (int)(rest / n_sites);
    const int64_t t = (int64_t)tt * kTT + tin;
    float z = 0.f;
    if (t < T && rho < r) {
      float c = 0.f;
      for (int j = 0; j < k; ++j)
        if (idx[t * k + j] == e) c += scale * gate[t * k + j];
      if (c != 0.f) {
        const int64_t col = (int64_t)q * N * r + (int64_t)e * r + rho;
        float us[kMaxSplits];             // every split's partial in flight at once
#pragma unroll
        for (int s = 0; s < kMaxSplits; ++s) us[s] = s < splits ? __ldcg(U + ((int64_t)s * T + t) * ldu + col) : 0.f;
        float u = 0.f;
#pragma unroll
        for (int s = 0; s < kMaxSplits; ++s)
          if (s < splits) u += us[s];      // split order: deterministic
        z = c * u;
      }
    }
    const __nv_bfloat16 hi = __float2bfloat16_rn(z);
    const __nv_bfloat16 lo = __float2bfloat16_rn(z - __bfloat162float(hi));    // z - hi exact in fp32
    __nv_bfloat16* blk = Z + ((((int64_t)tt * n_sites + q) * N + e) * 2) * (int64_t)kTT * rp;
    const int64_t off = swz_off(tin, rho, rp);
    blk[off] = hi;
    blk[(int64_t)kTT * rp + off] = lo;
  }
}

}  // namespace pf

// ------------------------------------------------------------------ host side

struct PfPlan {
  CUtensorMap w[LSW_NKIND], a[LSW_NKIND];
  CUtensorMap w2[LSW_NKIND], w4[LSW_NKIND];   // W boxes of 64 / 32 rows: one CTA's slice in a cluster of 2 / 4
  const __nv_bfloat16* Bp[LSW_NKIND];
  int64_t dout_pad[LSW_NKIND], d_out[LSW_NKIND], d_in[LSW_NKIND];
  int n_layers, n_experts, r, rp, num_sms;
  int tt_opt;                    // variant option pf_tt (128 | 256), 0: chosen per launch
  int cl_opt;                    // variant option pf_cluster (1 | 2 | 4), 0: chosen per launch
  int pair_opt;                  // variant option pf_pair: 0 never, 1 (default) for groups with a wave of
                                 // 256-token tiles, 2 whenever the sites' row tiles pair up: dense + LoRA-up
                                 // on CTA pairs
  CUtensorMap bmap[LSW_NKIND];   // pairs: the packed B of every kind as [L*N*dout_pad, rp]
  uint32_t* zdone;               // device words: [0] A-bank tiles done, [1] split-K half-0 partials
                                 // stored -- monotonic over the plan's launches
  mutable uint32_t z_count;      // host copy of zdone[0] once every launch so far has completed
  mutable uint32_t p_count;      // host copy of zdone[1]
  int split_opt;                 // variant option pf_bank_split: 1 (default) A-bank tiles split in two K
                                 // halves when the launch is one wave; 0 never
  int fuse_opt;                  // variant option pf_fuse_u: 1 (default) the single-CTA dense launch also
                                 // computes the LoRA-down and builds Z (A-bank tiles); 0 three launches
};

// shared-memory plan of one token-tile width: stage = [128 x 64 A box | B
// part], the B part a TT x 64 X box (dense) or the (hi, lo) pair of one
// expert's TT x rp Z slice (LoRA-up)
struct PfGeom {
  uint32_t stage_bytes, b_off, smem;
  int stages;
};
static constexpr uint32_t kPfBudget = 220 * 1024;

static PfGeom pf_geom(int tt, int rp) {
  PfGeom g;
  g.b_off = pf::kBoxBytes;
  const uint32_t dense_b = (uint32_t)tt * pf::kKB * 2, lora_b = 2u * tt * rp * 2;
  g.stage_bytes = g.b_off + (dense_b > lora_b ? dense_b : lora_b);
  g.stages = (int)(kPfBudget / g.stage_bytes);
  if (g.stages > pf::kMaxStages) g.stages = pf::kMaxStages;
  g.smem = g.stages * g.stage_bytes + 1024;
  return g;
}

// CTA pairs: stage = [128 x 64 W box | kTT/2 x 64 X box], or [B slice | the
// hi and lo halves of the token half of one expert's Z slice]
static PfGeom pf_geom_pair(int tt, int rp) {
  PfGeom g;
  g.b_off = pf::kBoxBytes;
  const uint32_t dense_b = (uint32_t)(tt / 2) * pf::kKB * 2, lora_b = 2u * (tt / 2) * rp * 2;
  g.stage_bytes = g.b_off + (dense_b > lora_b ? dense_b : lora_b);
  g.stages = (int)(kPfBudget / g.stage_bytes);
  if (g.stages > pf::kMaxStages) g.stages = pf::kMaxStages;
  g.smem = g.stages * g.stage_bytes + 1024;
  return g;
}

static PFN_cuTensorMapEncodeTiled_v12000 pf_encode();
// bf16 [rows, rp] row-major, already laid out as the operand (pre-swizzled):
// box {rp, box_rows}, no TMA swizzle -- a plain 2-D block copy
static bool pf_map_rows(CUtensorMap* m, const void* base, uint64_t rows, uint32_t rp, uint32_t box_rows) {
  auto enc = pf_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {rp, rows};
  cuuint64_t strides[1] = {(cuuint64_t)rp * 2};
  cuuint32_t box[2] = {rp, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static PFN_cuTensorMapEncodeTiled_v12000 pf_encode() {
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

// bf16 [.., rows, cols] row-major, box {64, box_rows(, 1)}, 128-B swizzle, zero OOB fill
static bool pf_map(CUtensorMap* m, const void* base, uint64_t cols, uint64_t rows, uint64_t L,
                   uint32_t box_rows = 128) {
  auto enc = pf_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {cols, rows, L};
  cuuint64_t strides[2] = {cols * 2, cols * rows * 2};
  cuuint32_t box[3] = {(cuuint32_t)pf::kKB, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, L ? 3 : 2, const_cast<void*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t pf_plan_create(PfPlan** out, const SwitchParams& sp, const TcPlan* tc, int num_sms) {
  *out = nullptr;
  PfPlan* p = new PfPlan();
  memset(p, 0, sizeof(*p));
  p->n_layers = sp.n_layers;
  p->n_experts = sp.n_experts;
  p->r = sp.rank;
  p->num_sms = num_sms;
  for (int k = 0; k < LSW_NKIND; ++k) {
    const KindGeom& g = sp.kind[k];
    int rp = 0;
    p->Bp[k] = static_cast<const __nv_bfloat16*>(tc_plan_packed_B(tc, k, &p->dout_pad[k], &rp));
    p->rp = rp;
    p->d_out[k] = g.d_out;
    p->d_in[k] = g.d_in;
    if (!p->Bp[k] || !pf_map(&p->w[k], g.W, g.d_in, g.d_out, sp.n_layers) ||
        !pf_map(&p->w2[k], g.W, g.d_in, g.d_out, sp.n_layers, 64) ||
        !pf_map(&p->w4[k], g.W, g.d_in, g.d_out, sp.n_layers, 32) ||
        !pf_map(&p->a[k], g.A, g.d_in, (uint64_t)sp.n_experts * sp.rank, sp.n_layers) ||
        !pf_map_rows(&p->bmap[k], p->Bp[k], (uint64_t)sp.n_layers * sp.n_experts * p->dout_pad[k], (uint32_t)rp, 128)) {
      delete p;
      return cudaErrorInvalidValue;
    }
  }
  p->tt_opt = (int)opt_int("pf_tt", 0);
  if (p->tt_opt != 128 && p->tt_opt != 256) p->tt_opt = 0;
  p->cl_opt = (int)opt_int("pf_cluster", 0);
  p->pair_opt = (int)opt_int("pf_pair", 1);
#ifdef LSW_TUNING
  {
    const char* v = opt_str("pf_trace_buf");
    uint32_t* buf = v ? reinterpret_cast<uint32_t*>(strtoull(v, nullptr, 10)) : nullptr;
    cudaMemcpyToSymbol(pf::g_pf_trace, &buf, sizeof(buf));
  }
#endif
  p->fuse_opt = (int)opt_int("pf_fuse_u", 1);
  p->split_opt = (int)opt_int("pf_bank_split", 1);
  if (p->cl_opt != 1 && p->cl_opt != 2 && p->cl_opt != 4) p->cl_opt = 0;
  if (pf_geom(128, p->rp).stages < 3) { delete p; return cudaErrorNotSupported; }
  const int smem = (int)(kPfBudget + 1024);
  cudaError_t e = cudaSuccess;
  for (auto fn : {pf::prefill_gemm<128, 1>, pf::prefill_gemm<128, 2>, pf::prefill_gemm<128, 4>,
                  pf::prefill_gemm<256, 1>, pf::prefill_gemm<256, 2>, pf::prefill_gemm<256, 4>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  for (auto fn : {pf::prefill_gemm_pair<128>, pf::prefill_gemm_pair<256>})
    if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaMalloc(&p->zdone, 2 * sizeof(uint32_t));
  if (e == cudaSuccess) e = cudaMemset(p->zdone, 0, 2 * sizeof(uint32_t));
  if (e != cudaSuccess) { cudaFree(p->zdone); delete p; return e; }
  *out = p;
  return cudaSuccess;
}

void pf_plan_destroy(PfPlan* p) {
  if (p) cudaFree(p->zdone);
  delete p;
}

// cluster size of the dense launch (variant option pf_cluster; default 1).
// Measured (7B, 512 tokens, same box): clusters of 4 token tiles sharing each
// W block by multicast 0.41 ms per layer vs 0.34 without -- the lockstep the
// multicast protocol imposes on the cluster's CTAs costs more than the L2
// traffic it saves.
static int pf_cluster(const PfPlan* p, int64_t n_tt) {
  (void)n_tt;
  return p->cl_opt ? p->cl_opt : 1;
}

// token-tile width of a group's launches (rt: the dense launch's row tiles).
// A 256-token tile moves 2/3 of the operand bytes per MAC of a 128-token one
// (48 vs 32 KB per 64-deep stage for twice the MACs), so it takes ~1/0.65 of
// the 128-token tile's time for twice the work -- but the dense launch is
// persistent over ONE wave of num_sms CTAs, and with few row tiles the
// 256-token tiles leave SMs idle (7B o / down at 512 tokens: 64 tiles on 148
// SMs).  Chosen by rounds x relative tile time; 256 needs >= 3 stages (rp <=
// 32) and T a multiple of 256 (no half-empty tiles).  Measured (7B, 512
// tokens): o 38.3 vs 43.9 us, down 67.8 vs 81.3 with 128; q|k|v 73.1 vs 84.5,
// gate|up 99.2 vs 122.8 with 256.
static int pf_tt(const PfPlan* p, int64_t T, int64_t rt, bool pair) {
  const bool ok256 = T % 256 == 0 && pf_geom(256, p->rp).stages >= 3;
  if (p->tt_opt) return p->tt_opt == 256 && pf_geom(256, p->rp).stages >= 3 ? 256 : 128;
  if (!ok256) return 128;
  const int64_t G = p->num_sms;
  const int64_t r128 = (rt * ((T + 127) / 128) + G - 1) / G, r256 = (rt * (T / 256) + G - 1) / G;
  // pairs: 32 vs 24 KB per CTA and K step (256- vs 128-token tile) -> 0.75
  return 100 * r256 <= (pair ? 75 : 65) * r128 + 5 ? 256 : 128;
}

// the dense + LoRA-up launch runs on CTA pairs: option on, no multicast
// cluster, every site's row tiles pair up within the site, and at least a
// wave of 256-token tiles (measured, 7B at 512 tokens: q|k|v 68.8 vs 70.5
// us, gate|up 90.6 vs 98.7 on pairs; o / down -- 64 tiles of 256 tokens, the
// LoRA chain their bound -- 40.6 vs 35.3 and 73.9 vs 64.6: single CTAs)
static bool pf_pair(const PfPlan* p, int n_sites, const int kinds[3], int64_t T, int64_t rt) {
  if (!p->pair_opt || pf_cluster(p, 0) != 1) return false;
  if (p->pair_opt == 1 && rt * ((T + 255) / 256) < p->num_sms) return false;   // (pf_pair=2: always)
  for (int q = 0; q < n_sites; ++q)
    if (((p->d_out[kinds[q]] + pf::kTM - 1) / pf::kTM) % 2) return false;
  return true;
}


// scratch sizes (elements) a launch with T tokens needs (either token tile)
void pf_scratch(const PfPlan* p, int n_sites, int64_t T, int64_t* u_elems, int64_t* z_elems) {
  const int64_t nr = (int64_t)p->n_experts * p->r;
  *u_elems = (int64_t)pf::kMaxSplits * T * n_sites * nr;
  *z_elems = 0;
  for (int64_t tt : {128, 256}) {
    const int64_t n_tt = (T + tt - 1) / tt, c = pf_cluster(p, n_tt);
    // fused, split bank tiles: one fp32 [tt, 128] partial per bank tile
    const int64_t bank = n_sites * ((nr + pf::kTM - 1) / pf::kTM) * n_tt * tt * pf::kTM;
    if (bank > *u_elems) *u_elems = bank;
    const int64_t n_tt_pad = (n_tt + c - 1) / c * c;             // Z of padded token tiles: zeros
    const int64_t z = n_tt_pad * n_sites * p->n_experts * 2 * tt * p->rp;
    if (z > *z_elems) *z_elems = z;
  }
}

template <int kTT>
static cudaError_t prefill_tc_tt(const PfPlan* p, const PrefillParams& P, int layer, const int kinds[3],
                                 cudaStream_t s, bool pair) {
  using namespace pf;
  const PfGeom geo = pf_geom(kTT, p->rp);
  Maps maps;
  memset(&maps, 0, sizeof(maps));
  if (!pf_map(&maps.x, P.X, P.d_in, P.T, 0, kTT)) return cudaErrorInvalidValue;
  const int n_tt = (int)((P.T + kTT - 1) / kTT);
  const int n_kb = (int)((P.d_in + kKB - 1) / kKB);
  const int64_t nr = (int64_t)p->n_experts * p->r;
  // ---- 1. LoRA-down (every expert), K split over the grid
  Args a;
  memset(&a, 0, sizeof(a));
  a.mode = MODE_U;
  a.n_sites = P.n_sites;
  a.layer = layer;
  a.n_tt = n_tt;
  a.n_kb = n_kb;
  a.T = P.T;
  int rt = 0;
  for (int q = 0; q < P.n_sites; ++q) {
    maps.op[q] = p->a[kinds[q]];
    a.tile_row0[q] = rt;
    rt += (int)((nr + kTM - 1) / kTM);
    a.rows_valid[q] = nr;
    a.col0[q] = q * nr;
  }
  a.tile_row0[P.n_sites] = rt;
  a.row_tiles_total = rt;
  // K split over the grid, at most kMaxSplits ways: the Z build sums the
  // splits' fp32 partials per element (and they cross L2), so a 74-way split
  // (7B o at 512 tokens: every SM a 64-deep slice) made the Z build, not the
  // products, the LoRA chain's cost
  int splits = p->num_sms / (rt * n_tt);
  if (splits > kMaxSplits) splits = kMaxSplits;
  if (splits < 1) splits = 1;
  if (splits > n_kb) splits = n_kb;
  a.splits = splits;
  a.total_tiles = rt * n_tt * splits;
  a.ld = P.n_sites * nr;
  a.out = P.U;
  a.stages = geo.stages;
  a.stage_bytes = geo.stage_bytes;
  a.b_off = geo.b_off;
  a.rp = p->rp;
  int grid = a.total_tiles < p->num_sms ? a.total_tiles : p->num_sms;
  cudaError_t e;
  const int C = pf_cluster(p, n_tt);
  const int n_tt_pad = (n_tt + C - 1) / C * C;
  // fused LoRA-down (single CTAs, no pairs): the A-bank tiles lead the dense
  // launch's tile order, so every CTA runs its A-bank tiles before any W
  // tile and no W tile's wait on them can block one
  // (not under stream capture: the count target is baked into the launch)
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cap) != cudaSuccess) return cudaGetLastError();
  const bool fuse = p->fuse_opt && C == 1 && !pair && P.k <= 4 && cap == cudaStreamCaptureStatusNone;
  const int a_tiles = rt * n_tt;                 // A-bank tiles (full K)
  if (!fuse) {
    cudaLaunchConfig_t uc{};
    uc.gridDim = dim3(grid);
    uc.blockDim = dim3(kThreads);
    uc.dynamicSmemBytes = geo.smem;
    uc.stream = s;
    cudaLaunchAttribute ua[1];
    ua[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    ua[0].val.programmaticStreamSerializationAllowed = 1;
    uc.attrs = ua;
    uc.numAttrs = 1;
    e = cudaLaunchKernelEx(&uc, prefill_gemm<kTT, 1>, maps, a);
    if (e != cudaSuccess) return e;
  }
  // ---- 2. gate-scaled (hi, lo) LoRA-down products of the selected experts
  if (!fuse) {
    const int64_t n = (int64_t)n_tt_pad * P.n_sites * p->n_experts * kTT * p->rp;
    int blocks = (int)((n + 255) / 256);
    if (blocks > 4 * p->num_sms) blocks = 4 * p->num_sms;
    cudaLaunchConfig_t zc{};
    zc.gridDim = dim3(blocks);
    zc.blockDim = dim3(256);
    zc.stream = s;
    cudaLaunchAttribute za[1];
    za[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    za[0].val.programmaticStreamSerializationAllowed = 1;
    zc.attrs = za;
    zc.numAttrs = 1;
    e = cudaLaunchKernelEx(&zc, prefill_zbuild, (const float*)P.U, splits, (int64_t)P.T, (int64_t)a.ld, P.n_sites,
                           p->n_experts, p->r, p->rp, P.k, P.scale, P.idx, P.gate,
                           reinterpret_cast<__nv_bfloat16*>(P.Z), n_tt_pad, kTT);
    if (e != cudaSuccess) return e;
  }
  // ---- 3. dense part + LoRA-up in one contraction per tile
  Args y = a;
  y.mode = MODE_Y;
  y.splits = 1;
  if (fuse) {
    for (int q = 0; q <= P.n_sites; ++q) y.a_row0[q] = a.tile_row0[q];
    for (int q = 0; q < P.n_sites; ++q) maps.a[q] = p->a[kinds[q]];
    y.a_tiles = a_tiles;
    y.k = P.k;
    y.r = p->r;
    y.scale = P.scale;
    y.idx = P.idx;
    y.gate = P.gate;
    y.Zw = reinterpret_cast<__nv_bfloat16*>(P.Z);
    y.zdone = p->zdone;
    y.z_target = p->z_count + (uint32_t)a_tiles;
    // each bank tile's K in two halves on two CTAs when the whole launch is
    // one wave (every half 0 then runs beside its half 1, so the wait for the
    // launch's half-0 count cannot block), and the partials fit in U
    const int64_t w_tiles = (int64_t)n_tt * [&] {
      int64_t t = 0;
      for (int q = 0; q < P.n_sites; ++q) t += (p->d_out[kinds[q]] + kTM - 1) / kTM;
      return t;
    }();
    if (p->split_opt && n_kb >= 2 && 2 * (int64_t)a_tiles + w_tiles <= p->num_sms &&
        (int64_t)a_tiles * kTT * kTM <= P.u_elems) {
      y.a_split = 2;
      y.a_tiles = 2 * a_tiles;
      y.pdone = p->zdone + 1;
      y.p_target = p->p_count + (uint32_t)a_tiles;
      y.Pp = P.U;
    }
  }
  rt = 0;
  for (int q = 0; q < P.n_sites; ++q) {
    const int kd = kinds[q];
    maps.op[q] = C == 4 ? p->w4[kd] : C == 2 ? p->w2[kd] : p->w[kd];
    y.tile_row0[q] = rt;
    rt += (int)((p->d_out[kd] + kTM - 1) / kTM);
    y.rows_valid[q] = p->d_out[kd];
    y.col0[q] = P.row_begin[q];
    y.Bp[q] = p->Bp[kd] + (size_t)layer * p->n_experts * p->dout_pad[kd] * p->rp;
    y.dout_pad[q] = p->dout_pad[kd];
  }
  y.tile_row0[P.n_sites] = rt;
  y.row_tiles_total = rt;
  y.total_tiles = y.a_tiles + rt * n_tt;
  y.ld = P.rows;
  y.out = P.Y;
  y.n_experts = p->n_experts;
  y.term_bytes = (uint32_t)kTM * p->rp * 2;
  y.zpart_bytes = (uint32_t)kTT * p->rp * 2;
  y.swz = p->rp == 16 ? 6u : p->rp == 32 ? 4u : 2u;     // SWIZZLE_32B / 64B / 128B
  y.Z = reinterpret_cast<const __nv_bfloat16*>(P.Z);
  // programmatic dependent of the Z build: its CTAs take the SMs the
  // LoRA-down grid leaves and run the dense K loop while Z is built; the
  // producer waits for the Z build only before the first LoRA-up stage
  cudaLaunchConfig_t lc{};
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = geo.smem;
  lc.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (C == 1 && pair) {
    const PfGeom gp = pf_geom_pair(kTT, p->rp);
    PairMaps mp;
    memset(&mp, 0, sizeof(mp));
    for (int q = 0; q < P.n_sites; ++q) {
      mp.op[q] = maps.op[q];
      mp.b[q] = p->bmap[kinds[q]];
    }
    const int64_t z_rows = (int64_t)n_tt_pad * P.n_sites * p->n_experts * 2 * kTT;
    if (!pf_map(&mp.x, P.X, P.d_in, P.T, 0, kTT / 2) ||                                  // token halves
        !pf_map_rows(&mp.z, P.Z, (uint64_t)z_rows, (uint32_t)p->rp, kTT / 2))
      return cudaErrorInvalidValue;
    int pr = 0;
    for (int q = 0; q < P.n_sites; ++q) {
      y.pair_row0[q] = pr;
      pr += (int)((p->d_out[kinds[q]] + kTM - 1) / kTM) / 2;
    }
    y.pair_row0[P.n_sites] = pr;
    y.stages = gp.stages;
    y.stage_bytes = gp.stage_bytes;
    y.b_off = gp.b_off;
    const int n_pt = pr * n_tt;                               // pair tiles
    const int n_cl = n_pt < p->num_sms / 2 ? n_pt : p->num_sms / 2;
    lc.gridDim = dim3(2 * n_cl);
    lc.dynamicSmemBytes = gp.smem;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = 2;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    lc.numAttrs = 2;
    return cudaLaunchKernelEx(&lc, prefill_gemm_pair<kTT>, mp, y);
  }
  if (C == 1) {
    lc.gridDim = dim3(y.total_tiles < p->num_sms ? y.total_tiles : p->num_sms);
    e = cudaLaunchKernelEx(&lc, prefill_gemm<kTT, 1>, maps, y);
    if (e == cudaSuccess && fuse) {
      p->z_count = y.z_target;
      if (y.a_split == 2) p->p_count = y.p_target;
    }
    return e;
  }
  const int n_ct = rt * (n_tt_pad / C);                      // cluster tiles
  const int n_cl = n_ct < p->num_sms / C ? n_ct : p->num_sms / C;
  lc.gridDim = dim3(n_cl * C);
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = C;
  at[1].val.clusterDim.y = 1;
  at[1].val.clusterDim.z = 1;
  lc.numAttrs = 2;
  return C == 4 ? cudaLaunchKernelEx(&lc, prefill_gemm<kTT, 4>, maps, y)
                : cudaLaunchKernelEx(&lc, prefill_gemm<kTT, 2>, maps, y);
}

cudaError_t launch_prefill_tc(const PfPlan* p, const PrefillParams& P, int layer, const int kinds[3],
                              cudaStream_t s) {
  int64_t rt = 0;                          // row tiles of the dense launch
  for (int q = 0; q < P.n_sites; ++q) rt += (p->d_out[kinds[q]] + pf::kTM - 1) / pf::kTM;
  const bool pair = pf_pair(p, P.n_sites, kinds, P.T, rt);
  return pf_tt(p, P.T, rt, pair) == 256 ? prefill_tc_tt<256>(p, P, layer, kinds, s, pair)
                                        : prefill_tc_tt<128>(p, P, layer, kinds, s, pair);
}

}  // namespace lsw
