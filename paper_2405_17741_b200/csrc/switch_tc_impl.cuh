// switch_tc_impl.cuh -- the tensor-core switch kernel behind lsw::tc_plan_*
// (switch_tc_dispatch.cu picks its mode per ctx at create time).  fc
// (switch_tc_fc.cu): the coefficients folded into the B factors as exact
// (hi, lo) bf16 pairs, ONE accumulator and one commit per 128 x 128 tile
// (Eq. 5's concatenation, K = 2 * sum_j rp), the folded strip held in TMEM
// as the MMA's M-side operand where it fits (2k * rp <= 256); its
// per-term mode (raw B, one accumulator per term, N = 128) for r = 64 and r =
// 32 with k >= 3, with the B slices staged per unit where a whole strip does
// not fit (r = 64, k = 4).
#pragma once

#include "lsw_internal.cuh"

namespace lsw {
namespace fc {
struct TcPlan;
// pt: 0 fold; 1 per-term (no fold, one fp32 TMEM accumulator per term; for
// large k*r); 2 per-term with the B slices staged per unit (no strip buffer)
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
const void* tc_plan_packed_B(const TcPlan* plan, int kind, int64_t* dout_pad, int* rp);
int tc_plan_pair(const TcPlan* plan);   // 1: the plain switch runs on CTA pairs
int tc_plan_tb(const TcPlan* plan);     // 1: the fold with its (hi, lo) B strip in TMEM
}  // namespace fc

}  // namespace lsw
