// switch_tc.cu -- K1-tc: the all-layer in-place switch on the 5th-gen tensor cores.
//
// What it computes (identical to K1-simt): for every adapted matrix m of every
// layer, in ONE persistent launch (SGMM Eq. 11; in place P:328):
//     W_m <- RNE( W_m + sum_j c_j * B_{m,e_j} @ A_{m,e_j} )
// with the Eq. 5/9/10 coefficient list (Eq. 9 sign corrected, R1; compacted,
// lsw_internal.cuh build_coefs).
//
// How:
//  * Tile = 128 rows (UMMA M, one row per TMEM lane) x TN=64 columns of W.
//    The tile sequence (kind, layer, row block, column block) is split into
//    equal contiguous ranges, one per persistent CTA (grid = #SMs), so a CTA
//    walks ALONG a 128-row strip: the strip's B slices (UMMA operand A,
//    128 x r per expert, K-major) stay resident in shared memory while the W
//    tile and the A slices (UMMA operand B: A^T, TN x r per expert, K-major,
//    packed at create) stream through a multi-stage TMA/mbarrier ring.
//  * One tcgen05.mma (kind::f16, bf16 in, fp32 accumulate) per expert per 16
//    of r, each expert into ITS OWN TMEM accumulator: the gate coefficients
//    c_j are then applied in fp32 in the epilogue (R13: exact fp32
//    coefficients, not Eq. 5's bf16-rounded g*DOWN).  Accumulators are
//    double-buffered in TMEM when 2 * terms * TN <= 512 columns, so the MMAs
//    of tile i+1 overlap the epilogue of tile i.
//  * Epilogue (8 warps, 2 per TMEM lane quarter): tcgen05.ld the accumulators,
//    delta = sum_j c_j acc_j, read the W tile from shared memory (128B-swizzled,
//    conflict-free), W + delta in fp32, RNE to bf16, write back to the same
//    shared buffer, then ONE TMA bulk tensor store writes the tile back in place
//    (3-D tensor map [L, d_out, d_in]: ragged row/column tails are zero-filled
//    on load and clipped on store, never spilling into the next layer).
//  * Warp roles: warp 0 = TMA producer, warp 1 = TMEM allocator + MMA issuer,
//    warps 2..9 = epilogue.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>

#include "lsw_internal.cuh"

namespace lsw {

constexpr int kTcTM = 128;
constexpr int kTcTN = 64;                 // tile columns = UMMA N
constexpr int kTcEpiWarps = 8;
constexpr int kTcThreads = 64 + 32 * kTcEpiWarps;
constexpr int kTcMaxStages = 8;
constexpr int kWTileBytes = kTcTM * kTcTN * 2;   // 16 KB

struct TcMaps {
  CUtensorMap w[LSW_NKIND];   // W   [L, d_out, d_in]      box {64, 128, 1}, 128B swizzle
  CUtensorMap a[LSW_NKIND];   // A^T [L*N, d_in, rp]       box {rp, 64, 1}
  CUtensorMap b[LSW_NKIND];   // B   [L*N, d_out, rp]      box {rp, 128, 1}
};

struct TcKind {
  int64_t tile_begin;
  int32_t row_tiles, col_tiles;
};

struct TcGeom {
  TcKind kind[LSW_NKIND];
  int64_t tiles_total;
  int32_t n_layers, n_experts, rp;        // rp: rank padded to a multiple of 16
  int32_t stages;                         // W+A ring depth
  int32_t acc_bufs;                       // TMEM accumulator buffers (1 or 2)
  int32_t b_bufs;                         // B-strip buffers (1 or 2)
  int32_t max_terms;                      // 2k
  uint32_t tmem_cols;
  uint32_t a_bytes_per_term;              // TN * rp * 2
  uint32_t b_bytes_per_term;              // 128 * rp * 2
  uint32_t swz_mode;                      // UMMA layout type of the r-wide operands
  uint32_t smem_bytes;
};

struct TcPlan {
  TcMaps maps;
  TcGeom geom;
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

struct TileCoord {
  int kd, layer, rb, cb;
};

__device__ __forceinline__ TileCoord tile_coord(const TcGeom& g, int64_t t) {
  TileCoord c;
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
  return c;
}

// ------------------------------------------------------------------ the kernel

struct TcArgs {
  TcGeom g;
  // coefficient inputs (same as SwitchParams)
  int32_t mode, top_k, n_experts;
  float scale;
  const int32_t* cur_idx;
  const float* cur_g;
  DevState* state;
};

__global__ void __launch_bounds__(kTcThreads, 1)
switch_tc_kernel(const __grid_constant__ TcMaps maps, const __grid_constant__ TcArgs args) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ Coefs cf;
  __shared__ int32_t s_parity;
  __shared__ uint32_t s_tmem_base;
  __shared__ __align__(8) uint64_t bar_full[kTcMaxStages], bar_empty[kTcMaxStages];
  __shared__ __align__(8) uint64_t bar_bfull[2], bar_bempty[2];
  __shared__ __align__(8) uint64_t bar_accfull[2], bar_accempty[2];

  const TcGeom& g = args.g;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // shared layout: [stages x (W tile 16 KB | A slices)] [2 x B strip slices], 1 KB aligned
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t a_bytes = g.max_terms * g.a_bytes_per_term;
  const uint32_t stage_bytes = (kWTileBytes + a_bytes + 1023) & ~1023u;
  const uint32_t b_bytes = (g.max_terms * g.b_bytes_per_term + 1023) & ~1023u;
  uint8_t* stage0 = base;
  uint8_t* bstrip0 = base + (size_t)g.stages * stage_bytes;

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
    for (int s = 0; s < g.stages; ++s) {
      mbar_init(smem_u32(&bar_full[s]), 1);
      mbar_init(smem_u32(&bar_empty[s]), 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(smem_u32(&bar_bfull[s]), 1);
      mbar_init(smem_u32(&bar_bempty[s]), 1);
      mbar_init(smem_u32(&bar_accfull[s]), 1);
      mbar_init(smem_u32(&bar_accempty[s]), kTcEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0 && lane == 0) {
    for (int k = 0; k < LSW_NKIND; ++k) {
      prefetch_map(&maps.w[k]);
      prefetch_map(&maps.a[k]);
      prefetch_map(&maps.b[k]);
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                 ::"r"(smem_u32(&s_tmem_base)), "r"(g.tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();

  const int nt = cf.bad ? 0 : cf.n;
  const int64_t T = g.tiles_total;
  const int64_t t_begin = T * blockIdx.x / gridDim.x;
  const int64_t t_end = T * (blockIdx.x + 1) / gridDim.x;
  const uint32_t tmem_base = s_tmem_base;

  if (nt > 0 && t_begin < t_end) {
    if (warp == 0) {
      // ============================ TMA producer ============================
      if (lane == 0) {
        const uint64_t pol_stream = policy_evict_first();
        const uint64_t pol_keep = policy_evict_last();
        int64_t strip_prev = -1;
        uint32_t nstrip = 0;
        uint32_t it = 0;
        for (int64_t t = t_begin; t < t_end; ++t, ++it) {
          const TileCoord c = tile_coord(g, t);
          const int64_t strip = t - c.cb;            // unique id of the 128-row strip
          if (strip != strip_prev) {
            strip_prev = strip;
            const uint32_t bs = nstrip % g.b_bufs, round = nstrip / g.b_bufs;
            mbar_wait(smem_u32(&bar_bempty[bs]), (round & 1) ^ 1);
            const uint32_t bar = smem_u32(&bar_bfull[bs]);
            mbar_expect_tx(bar, nt * g.b_bytes_per_term);
            uint8_t* dst = bstrip0 + (size_t)bs * b_bytes;
            for (int j = 0; j < nt; ++j)
              tma_load_3d(smem_u32(dst + j * g.b_bytes_per_term), &maps.b[c.kd], 0, c.rb * kTcTM,
                          c.layer * g.n_experts + cf.e[j], bar, pol_keep);
            ++nstrip;
          }
          const uint32_t s = it % g.stages, round = it / g.stages;
          mbar_wait(smem_u32(&bar_empty[s]), (round & 1) ^ 1);
          const uint32_t bar = smem_u32(&bar_full[s]);
          mbar_expect_tx(bar, kWTileBytes + nt * g.a_bytes_per_term);
          uint8_t* st = stage0 + (size_t)s * stage_bytes;
          tma_load_3d(smem_u32(st), &maps.w[c.kd], c.cb * kTcTN, c.rb * kTcTM, c.layer, bar, pol_stream);
          for (int j = 0; j < nt; ++j)
            tma_load_3d(smem_u32(st + kWTileBytes + j * g.a_bytes_per_term), &maps.a[c.kd], 0, c.cb * kTcTN,
                        c.layer * g.n_experts + cf.e[j], bar, pol_keep);
        }
      }
    } else if (warp == 1) {
      // ============================ MMA issuer ==============================
      if (lane == 0) {
        // instruction descriptor: D f32, A/B bf16, both K-major, N = 64, M = 128
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kTcTN >> 3) << 17) |
                               ((uint32_t)(kTcTM >> 4) << 24);
        const uint32_t row_bytes = g.rp * 2;
        const uint32_t sbo = 8 * row_bytes;
        int64_t strip_prev = -1;
        uint32_t nstrip = 0, bs = 0;
        uint32_t it = 0;
        for (int64_t t = t_begin; t < t_end; ++t, ++it) {
          const TileCoord c = tile_coord(g, t);
          const int64_t strip = t - c.cb;
          if (strip != strip_prev) {
            strip_prev = strip;
            bs = nstrip % g.b_bufs;
            mbar_wait(smem_u32(&bar_bfull[bs]), (nstrip / g.b_bufs) & 1);
            ++nstrip;
          }
          const uint32_t s = it % g.stages;
          mbar_wait(smem_u32(&bar_full[s]), (it / g.stages) & 1);
          const uint32_t ab = it % g.acc_bufs;
          mbar_wait(smem_u32(&bar_accempty[ab]), ((it / g.acc_bufs) & 1) ^ 1);
          tc_fence_after();
          const uint32_t a_stage = smem_u32(stage0 + (size_t)s * stage_bytes + kWTileBytes);
          const uint32_t b_strip = smem_u32(bstrip0 + (size_t)bs * b_bytes);
          for (int j = 0; j < nt; ++j) {
            const uint32_t d_tmem = tmem_base + (ab * g.max_terms + j) * kTcTN;
            for (int kk = 0; kk < g.rp / 16; ++kk) {
              const uint64_t adesc = umma_desc(b_strip + j * g.b_bytes_per_term + kk * 32, sbo, g.swz_mode);
              const uint64_t bdesc = umma_desc(a_stage + j * g.a_bytes_per_term + kk * 32, sbo, g.swz_mode);
              umma_f16(d_tmem, adesc, bdesc, idesc, kk > 0 ? 1u : 0u);
            }
          }
          umma_commit(smem_u32(&bar_accfull[ab]));
          // B strip no longer needed after the last tile of the strip
          const bool strip_ends = (t + 1 == t_end) || (c.cb + 1 == g.kind[c.kd].col_tiles);
          if (strip_ends) umma_commit(smem_u32(&bar_bempty[bs]));
        }
      }
    } else {
      // ============================ epilogue ================================
      const int ew = warp - 2;                     // 0..7
      const int quarter = warp & 3;                // TMEM lane quarter this warp may access
      const int half = ew >> 2;                    // which 32 of the 64 columns
      const int row = quarter * 32 + lane;         // tile-local row == TMEM lane
      const bool store_thread = (ew == 0 && lane == 0);
      const uint64_t pol_stream = policy_evict_first();
      float cj[kMaxTerms];
#pragma unroll
      for (int j = 0; j < kMaxTerms; ++j) cj[j] = j < nt ? cf.c[j] : 0.f;
      uint32_t it = 0;
      int32_t prev_stage = -1;
      for (int64_t t = t_begin; t < t_end; ++t, ++it) {
        const uint32_t s = it % g.stages;
        const uint32_t ab = it % g.acc_bufs;
        mbar_wait(smem_u32(&bar_full[s]), (it / g.stages) & 1);       // W tile landed (acquire)
        mbar_wait(smem_u32(&bar_accfull[ab]), (it / g.acc_bufs) & 1);  // accumulators ready
        tc_fence_after();
        uint8_t* wt = stage0 + (size_t)s * stage_bytes;
        const uint32_t tm_row = tmem_base + ((uint32_t)(quarter * 32) << 16) + ab * g.max_terms * kTcTN;
#pragma unroll
        for (int q2 = 0; q2 < 2; ++q2) {
          const int col16 = half * 2 + q2;         // 16-column chunk 0..3
          float d[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) d[i] = 0.f;
          for (int j0 = 0; j0 < nt; j0 += 4) {
            uint32_t acc[4][16];
            const int nj = nt - j0 < 4 ? nt - j0 : 4;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              if (jj < nj) tmem_ld16(tm_row + (j0 + jj) * kTcTN + col16 * 16, acc[jj]);
            tmem_wait_ld();
#pragma unroll
            for (int jj = 0; jj < 4; ++jj)
              if (jj < nj) {
                const float c = cj[j0 + jj];
#pragma unroll
                for (int i = 0; i < 16; ++i) d[i] = fmaf(c, __uint_as_float(acc[jj][i]), d[i]);
              }
          }
          // W row chunk: two 16-B swizzled chunks (8 bf16 each) of this row's 128-B line
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int chunk = col16 * 2 + h;
            uint4* p = reinterpret_cast<uint4*>(wt + row * 128 + ((chunk ^ (row & 7)) << 4));
            uint4 u = *p;
            uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float lo = __uint_as_float(w[i] << 16) + d[h * 8 + 2 * i];
              const float hi = __uint_as_float(w[i] & 0xffff0000u) + d[h * 8 + 2 * i + 1];
              __nv_bfloat162 b2 = __floats2bfloat162_rn(lo, hi);
              w[i] = *reinterpret_cast<uint32_t*>(&b2);
            }
            *p = make_uint4(w[0], w[1], w[2], w[3]);
          }
        }
        // accumulators consumed -> MMA may reuse this TMEM buffer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&bar_accempty[ab]));
        // make generic-proxy smem writes visible to the TMA (async proxy), then store
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        named_bar(1, 32 * kTcEpiWarps);
        if (store_thread) {
          const TileCoord c = tile_coord(g, t);
          tma_store_3d(&maps.w[c.kd], smem_u32(wt), c.cb * kTcTN, c.rb * kTcTM, c.layer, pol_stream);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          // the previous tile's store has finished reading smem -> free its stage
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          if (prev_stage >= 0) mbar_arrive(smem_u32(&bar_empty[prev_stage]));
          prev_stage = (int32_t)s;
        }
      }
      if (store_thread) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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

// ------------------------------------------------------------------ packing

// A [L*N, r, d_in] -> A^T [L*N, d_in, rp] (zero-padded rank)
__global__ void pack_At_kernel(const __nv_bfloat16* __restrict__ A, __nv_bfloat16* __restrict__ At, int64_t LN,
                               int r, int rp, int64_t d_in) {
  const int64_t total = LN * d_in * rp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int rho = (int)(i % rp);
    const int64_t c = (i / rp) % d_in;
    const int64_t m = i / ((int64_t)rp * d_in);
    At[i] = rho < r ? A[(m * r + rho) * d_in + c] : __float2bfloat16(0.f);
  }
}

// B [L*N, d_out, r] -> [L*N, d_out, rp] (zero-padded rank), only when r % 16 != 0
__global__ void pack_B_kernel(const __nv_bfloat16* __restrict__ B, __nv_bfloat16* __restrict__ Bp, int64_t rows,
                              int r, int rp) {
  const int64_t total = rows * rp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int rho = (int)(i % rp);
    const int64_t row = i / rp;
    Bp[i] = rho < r ? B[row * r + rho] : __float2bfloat16(0.f);
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

static bool encode3d(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2, uint32_t b0,
                     uint32_t b1, CUtensorMapSwizzle swz) {
  auto enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {d0 * 2, d0 * d1 * 2};
  cuuint32_t box[3] = {b0, b1, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& sp, int num_sms, const char** why) {
  *out = nullptr;
  int dev = 0, major = 0, minor = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (major != 10 || minor != 0) { *why = "needs an sm_100 (B200) device"; return cudaErrorNotSupported; }
  const int r = sp.rank, rp = (r + 15) / 16 * 16;
  if (rp > 64) { *why = "rank > 64"; return cudaErrorNotSupported; }
  TcPlan* plan = new TcPlan();
  TcGeom& g = plan->geom;
  memset(&g, 0, sizeof(g));
  g.n_layers = sp.n_layers;
  g.n_experts = sp.n_experts;
  g.rp = rp;
  g.max_terms = 2 * sp.top_k;
  g.a_bytes_per_term = kTcTN * rp * 2;
  g.b_bytes_per_term = kTcTM * rp * 2;
  g.swz_mode = rp == 16 ? 6u : rp == 32 ? 4u : 2u;        // SWIZZLE_32B / 64B / 128B (UMMA encoding)
  const CUtensorMapSwizzle tswz = rp == 16 ? CU_TENSOR_MAP_SWIZZLE_32B
                                  : rp == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B;
  const uint32_t cols1 = (uint32_t)g.max_terms * kTcTN;
  if (cols1 > 512) { delete plan; *why = "2*top_k*64 TMEM columns exceed 512"; return cudaErrorNotSupported; }
  g.acc_bufs = cols1 * 2 <= 512 ? 2 : 1;
  uint32_t need = cols1 * g.acc_bufs, cols = 32;
  while (cols < need) cols <<= 1;
  g.tmem_cols = cols;
  const uint32_t stage_bytes = (kWTileBytes + g.max_terms * g.a_bytes_per_term + 1023) & ~1023u;
  const uint32_t b_bytes = (g.max_terms * g.b_bytes_per_term + 1023) & ~1023u;
  const uint32_t budget = 227 * 1024 - 1024 /*align*/ - 2048 /*static*/;
  int stages = kTcMaxStages, bbufs = 2;
  while (stages > 2 && (uint32_t)stages * stage_bytes + bbufs * b_bytes > budget) --stages;
  if ((uint32_t)stages * stage_bytes + bbufs * b_bytes > budget) bbufs = 1;
  if ((uint32_t)stages * stage_bytes + bbufs * b_bytes > budget) {
    delete plan; *why = "shared memory: rank * top_k too large"; return cudaErrorNotSupported;
  }
  g.stages = stages;
  g.b_bufs = bbufs;
  g.smem_bytes = stages * stage_bytes + bbufs * b_bytes + 1024;
  // tiles
  int64_t t = 0;
  for (int k = 0; k < LSW_NKIND; ++k) {
    const KindGeom& kg = sp.kind[k];
    g.kind[k].row_tiles = (int32_t)((kg.d_out + kTcTM - 1) / kTcTM);
    g.kind[k].col_tiles = (int32_t)((kg.d_in + kTcTN - 1) / kTcTN);
    g.kind[k].tile_begin = t;
    t += (int64_t)sp.n_layers * g.kind[k].row_tiles * g.kind[k].col_tiles;
  }
  g.tiles_total = t;
  plan->grid = (int)(t < num_sms ? t : num_sms);
  if (plan->grid < 1) plan->grid = 1;
  // pack operands + encode maps
  const int64_t LN = (int64_t)sp.n_layers * sp.n_experts;
  cudaError_t e = cudaSuccess;
  for (int k = 0; k < LSW_NKIND && e == cudaSuccess; ++k) {
    const KindGeom& kg = sp.kind[k];
    const size_t at_bytes = (size_t)LN * kg.d_in * rp * 2;
    e = cudaMalloc(&plan->packed_At[k], at_bytes);
    if (e != cudaSuccess) break;
    plan->bytes += at_bytes;
    pack_At_kernel<<<1024, 256>>>((const __nv_bfloat16*)kg.A, (__nv_bfloat16*)plan->packed_At[k], LN, r, rp, kg.d_in);
    const void* Bsrc = kg.B;
    if (rp != r) {
      const size_t b_bytes_k = (size_t)LN * kg.d_out * rp * 2;
      e = cudaMalloc(&plan->packed_B[k], b_bytes_k);
      if (e != cudaSuccess) break;
      plan->bytes += b_bytes_k;
      pack_B_kernel<<<1024, 256>>>((const __nv_bfloat16*)kg.B, (__nv_bfloat16*)plan->packed_B[k], LN * kg.d_out, r, rp);
      Bsrc = plan->packed_B[k];
    }
    if (!encode3d(&plan->maps.w[k], kg.W, kg.d_in, kg.d_out, sp.n_layers, kTcTN, kTcTM, CU_TENSOR_MAP_SWIZZLE_128B) ||
        !encode3d(&plan->maps.a[k], plan->packed_At[k], rp, kg.d_in, LN, rp, kTcTN, tswz) ||
        !encode3d(&plan->maps.b[k], Bsrc, rp, kg.d_out, LN, rp, kTcTM, tswz)) {
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
  for (int k = 0; k < LSW_NKIND; ++k) {
    cudaFree(plan->packed_At[k]);
    cudaFree(plan->packed_B[k]);
  }
  delete plan;
}

int64_t tc_plan_bytes(const TcPlan* plan) { return plan ? plan->bytes : 0; }
int tc_plan_grid(const TcPlan* plan) { return plan ? plan->grid : 0; }
int tc_plan_tile_n(const TcPlan*) { return kTcTN; }
int64_t tc_plan_tiles(const TcPlan* plan) { return plan ? plan->geom.tiles_total : 0; }

cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s) {
  TcArgs a;
  a.g = plan->geom;
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

}  // namespace lsw
