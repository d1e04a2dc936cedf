// switch_tc_dispatch.cu -- lsw::tc_plan_*: one tensor-core switch kernel per
// ctx, chosen at create time (switch_tc_impl.cuh): v1 for 2k = 4 terms when
// it has a double-buffered 128-column plan, else the term-group kernel.
// LSW_TC_KERNEL=v1|tg forces one (tuning and tests).
#include <cstdlib>
#include <cstring>

#include "switch_tc_impl.cuh"

namespace lsw {

struct TcPlan {
  v1::TcPlan* a = nullptr;
  tg::TcPlan* b = nullptr;
};

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why) {
  *out = nullptr;
  const char* k = getenv("LSW_TC_KERNEL");
  const bool force_v1 = k && strcmp(k, "v1") == 0, force_tg = k && strcmp(k, "tg") == 0;
  TcPlan* p = new TcPlan();
  cudaError_t e = cudaErrorNotSupported;
  // measured (scripts/sweep_bench.py, 7B shape): k = 1 (2 terms) tg 0.89 vs v1
  // 0.83 of the copy peak; k = 2 (4 terms) v1 0.82 vs tg 0.73; k >= 3 only tg
  const bool prefer_tg = 2 * geom.top_k <= 2;
  if (!force_tg && (force_v1 || !prefer_tg)) {
    e = v1::tc_plan_create(&p->a, geom, num_sms, why, /*strict=*/!force_v1);
    if (e != cudaSuccess && e != cudaErrorNotSupported) { delete p; return e; }
    if (e != cudaSuccess) (void)cudaGetLastError();
  }
  if (e != cudaSuccess && !force_v1) {
    *why = "";
    e = tg::tc_plan_create(&p->b, geom, num_sms, why);
  }
  if (e != cudaSuccess) { delete p; return e; }
  *out = p;
  return cudaSuccess;
}

void tc_plan_destroy(TcPlan* plan) {
  if (!plan) return;
  if (plan->a) v1::tc_plan_destroy(plan->a);
  if (plan->b) tg::tc_plan_destroy(plan->b);
  delete plan;
}

int64_t tc_plan_bytes(const TcPlan* p) { return p->a ? v1::tc_plan_bytes(p->a) : tg::tc_plan_bytes(p->b); }
int tc_plan_grid(const TcPlan* p) { return p->a ? v1::tc_plan_grid(p->a) : tg::tc_plan_grid(p->b); }
int tc_plan_tile_n(const TcPlan* p) { return p->a ? v1::tc_plan_tile_n(p->a) : tg::tc_plan_tile_n(p->b); }
int64_t tc_plan_tiles(const TcPlan* p) { return p->a ? v1::tc_plan_tiles(p->a) : tg::tc_plan_tiles(p->b); }
int tc_plan_kernel(const TcPlan* p) { return p->a ? 1 : 2; }

cudaError_t launch_switch_tc(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, int64_t t0, int64_t t_count) {
  return p->a ? v1::launch_switch_tc(p->a, sp, s, t0, t_count) : tg::launch_switch_tc(p->b, sp, s, t0, t_count);
}

int64_t tc_plan_matrix_tiles(const TcPlan* p, int kind, int layer, int64_t* t0) {
  return p->a ? v1::tc_plan_matrix_tiles(p->a, kind, layer, t0) : tg::tc_plan_matrix_tiles(p->b, kind, layer, t0);
}

cudaError_t tc_plan_set_pristine(TcPlan* p, const SwitchParams& geom) {
  return p->a ? v1::tc_plan_set_pristine(p->a, geom) : tg::tc_plan_set_pristine(p->b, geom);
}

cudaError_t tc_plan_set_fused(TcPlan* p, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]) {
  if (!p->a) return cudaErrorNotSupported;          // the term-group kernel has no fused mode
  return v1::tc_plan_set_fused(p->a, n_layers, x_off, y_off, x_per_layer, y_per_layer, kinds, nk);
}

cudaError_t launch_switch_tc_fused(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, const void* xs, float* ys) {
  if (!p->a) return cudaErrorNotSupported;
  return v1::launch_switch_tc_fused(p->a, sp, s, xs, ys);
}

int64_t tc_plan_trace(const TcPlan* p, uint64_t* host, int64_t n) {
  return p->a ? v1::tc_plan_trace(p->a, host, n) : tg::tc_plan_trace(p->b, host, n);
}

}  // namespace lsw
