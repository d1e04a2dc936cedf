// switch_tc_impl.cuh -- the three tensor-core switch kernels behind
// lsw::tc_plan_* (switch_tc_dispatch.cu picks one per ctx at create time):
//
//   v1 (switch_tc.cu): every term of a 64-column sub-tile in its own TMEM
//      accumulator, two buffers of 2k x 64 columns -- needs 2k <= 4 and one
//      tile's A slices for all terms in shared memory (7B: 0.83 of the copy
//      peak; superseded by fc, kept for the fused decode of tg ctxs and tests).
//   tg (switch_tc_tg.cu): a tile's terms stream through TMEM tg at a time
//      with an fp32 running sum in the epilogue, A slices staged per
//      (sub-tile, term group): any k <= 4, any r <= 64.
//   fc (switch_tc_fc.cu, the default): the coefficients folded into the B
//      factors as exact (hi, lo) bf16 pairs, ONE accumulator and one commit per
//      128 x 128 tile (Eq. 5's concatenation, K = 2 * sum_j rp): twice the
//      tensor-core work, a fraction of the epilogue's TMEM reads and FMAs and
//      of the commits (7B: 0.90 of the copy peak); its per-term mode (raw B,
//      one accumulator per term, N = 128) for r = 64 and r = 32 with k >= 3.
#pragma once

#include "lsw_internal.cuh"

namespace lsw {
namespace v1 {
struct TcPlan;
// strict: refuse (cudaErrorNotSupported) a degraded plan (64-column tiles,
// single TMEM buffer, split mode) instead of building it
cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why, bool strict);
void tc_plan_destroy(TcPlan* plan);
int64_t tc_plan_bytes(const TcPlan* plan);
int tc_plan_grid(const TcPlan* plan);
int tc_plan_tile_n(const TcPlan* plan);
int64_t tc_plan_tiles(const TcPlan* plan);
cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0 = 0,
                             int64_t t_count = 0);
int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0);
int64_t tc_plan_trace(const TcPlan* plan, uint64_t* host, int64_t n);
cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& geom);
// fused switch + decode: decoder-order segment table, then launches
cudaError_t tc_plan_set_fused(TcPlan* plan, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]);
cudaError_t launch_switch_tc_fused(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, const void* xs,
                                   float* ys);
}  // namespace v1

// the v1 kernel compiled with the fused epilogue (switch_tc_fused.cu)
namespace v1f {
cudaError_t launch_fused_raw(const void* maps, const void* geom, int grid, uint32_t smem, int32_t order_chunk,
                             const SwitchParams& p, cudaStream_t s, const void* segs, int32_t n_seg, int64_t tiles,
                             const void* xs, float* ys, unsigned long long* seg_done, uint64_t* trace);
}  // namespace v1f

namespace tg {
struct TcPlan;
cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why);
void tc_plan_destroy(TcPlan* plan);
int64_t tc_plan_bytes(const TcPlan* plan);
int tc_plan_grid(const TcPlan* plan);
int tc_plan_tile_n(const TcPlan* plan);
int64_t tc_plan_tiles(const TcPlan* plan);
cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0 = 0,
                             int64_t t_count = 0);
int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0);
int64_t tc_plan_trace(const TcPlan* plan, uint64_t* host, int64_t n);
cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& geom);
}  // namespace tg

namespace fc {
struct TcPlan;
// tcgen05.mma instructions (128 x 128 x 16) per tile at 2k terms
int fc_mmas_per_tile(const SwitchParams& geom);
// pt: per-term mode (no fold, one fp32 TMEM accumulator per term; for large k*r)
cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why, int pt);
void tc_plan_destroy(TcPlan* plan);
int64_t tc_plan_bytes(const TcPlan* plan);
int tc_plan_grid(const TcPlan* plan);
int tc_plan_tile_n(const TcPlan* plan);
int64_t tc_plan_tiles(const TcPlan* plan);
cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0 = 0,
                             int64_t t_count = 0);
int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0);
cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& geom);
// fused switch + decode: decoder-order segment table, then launches
cudaError_t tc_plan_set_fused(TcPlan* plan, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]);
cudaError_t launch_switch_tc_fused(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, const void* xs,
                                   float* ys);
}  // namespace fc

// the fc kernel is the default from kFcMinMmas MMAs per tile on, wherever its
// shared-memory plan fits (measured: with three W stages it is
// ahead of tg at k = 1 too, 0.895 vs 0.856)
constexpr int kFcMinMmas = 0;
}  // namespace lsw
