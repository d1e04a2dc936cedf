// switch_tc_dispatch.cu -- lsw::tc_plan_*: one tensor-core switch kernel per
// ctx, chosen at create time (switch_tc_impl.cuh): the folded-coefficient
// kernel (fc) where its tensor-core work per tile stays small, else v1 for
// 2k = 4 terms when it has a double-buffered 128-column plan, else the
// term-group kernel.  LSW_TC_KERNEL=v1|tg|fc forces one (tuning and tests).
#include <cstdlib>
#include <cstring>

#include "switch_tc_impl.cuh"

namespace lsw {

struct TcPlan {
  int which = 0;                 // 1: v1, 2: tg, 3: fc -- the kernel every switch call launches
  v1::TcPlan* a = nullptr;       // v1 plan (primary when which == 1; else built on demand for the fused decode)
  tg::TcPlan* b = nullptr;
  fc::TcPlan* c = nullptr;
  SwitchParams geom{};
  int num_sms = 0;
};

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why) {
  *out = nullptr;
  const char* k = getenv("LSW_TC_KERNEL");
  const bool force_v1 = k && strcmp(k, "v1") == 0, force_tg = k && strcmp(k, "tg") == 0,
             force_fc = k && strcmp(k, "fc") == 0;
  TcPlan* p = new TcPlan();
  p->geom = geom;
  p->num_sms = num_sms;
  cudaError_t e = cudaErrorNotSupported;
  // measured (scripts/sweep_bench.py, 7B shape): see DESIGN.md §5 -- the
  // folded-coefficient kernel wherever its tensor-core work per tile stays well
  // under the tile's HBM time; else v1 at 2k = 4 and tg elsewhere
  const bool prefer_fc = fc::fc_mmas_per_tile(geom) >= kFcMinMmas;
  const bool prefer_tg = 2 * geom.top_k <= 2;
  if (force_fc || (!force_v1 && !force_tg && prefer_fc)) {
    // fc's two modes (measured): the folded one up to 2k * rp =
    // 128 at r <= 32 (the BASELINE configs), the per-term one for r = 64 and
    // for r = 32 with k >= 3; either falls back to the other if its shared-
    // memory plan does not fit (LSW_FC_PT forces one inside fc)
    const int rp = geom.rank <= 16 ? 16 : geom.rank <= 32 ? 32 : 64;
    const int pt_first = (rp == 64 || (rp == 32 && geom.top_k >= 3)) ? 1 : 0;
    for (int m = 0; m < 2 && e != cudaSuccess; ++m) {
      e = fc::tc_plan_create(&p->c, geom, num_sms, why, m == 0 ? pt_first : 1 - pt_first);
      if (e != cudaSuccess && e != cudaErrorNotSupported) { delete p; return e; }
      if (e != cudaSuccess) { (void)cudaGetLastError(); p->c = nullptr; }
    }
    if (e == cudaSuccess) p->which = 3;
    else if (force_fc) { delete p; return e; }
    else *why = "";
  }
  if (e != cudaSuccess && !force_tg && (force_v1 || !prefer_tg)) {
    e = v1::tc_plan_create(&p->a, geom, num_sms, why, /*strict=*/!force_v1);
    if (e != cudaSuccess && e != cudaErrorNotSupported) { delete p; return e; }
    if (e == cudaSuccess) p->which = 1;
    else (void)cudaGetLastError();
  }
  if (e != cudaSuccess && !force_v1) {
    *why = "";
    e = tg::tc_plan_create(&p->b, geom, num_sms, why);
    if (e == cudaSuccess) p->which = 2;
  }
  if (e != cudaSuccess) { delete p; return e; }
  *out = p;
  return cudaSuccess;
}

void tc_plan_destroy(TcPlan* plan) {
  if (!plan) return;
  if (plan->a) v1::tc_plan_destroy(plan->a);
  if (plan->b) tg::tc_plan_destroy(plan->b);
  if (plan->c) fc::tc_plan_destroy(plan->c);
  delete plan;
}

#define LSW_TC_DISPATCH(call_v1, call_tg, call_fc) \
  (p->which == 1 ? (call_v1) : p->which == 2 ? (call_tg) : (call_fc))

int64_t tc_plan_bytes(const TcPlan* p) {
  return (p->a ? v1::tc_plan_bytes(p->a) : 0) + (p->b ? tg::tc_plan_bytes(p->b) : 0) +
         (p->c ? fc::tc_plan_bytes(p->c) : 0);
}
int tc_plan_grid(const TcPlan* p) {
  return LSW_TC_DISPATCH(v1::tc_plan_grid(p->a), tg::tc_plan_grid(p->b), fc::tc_plan_grid(p->c));
}
int tc_plan_tile_n(const TcPlan* p) {
  return LSW_TC_DISPATCH(v1::tc_plan_tile_n(p->a), tg::tc_plan_tile_n(p->b), fc::tc_plan_tile_n(p->c));
}
int64_t tc_plan_tiles(const TcPlan* p) {
  return LSW_TC_DISPATCH(v1::tc_plan_tiles(p->a), tg::tc_plan_tiles(p->b), fc::tc_plan_tiles(p->c));
}
int tc_plan_kernel(const TcPlan* p) { return p->which; }

cudaError_t launch_switch_tc(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, int64_t t0, int64_t t_count) {
  return LSW_TC_DISPATCH(v1::launch_switch_tc(p->a, sp, s, t0, t_count), tg::launch_switch_tc(p->b, sp, s, t0, t_count),
                         fc::launch_switch_tc(p->c, sp, s, t0, t_count));
}

int64_t tc_plan_matrix_tiles(const TcPlan* p, int kind, int layer, int64_t* t0) {
  return LSW_TC_DISPATCH(v1::tc_plan_matrix_tiles(p->a, kind, layer, t0),
                         tg::tc_plan_matrix_tiles(p->b, kind, layer, t0),
                         fc::tc_plan_matrix_tiles(p->c, kind, layer, t0));
}

cudaError_t tc_plan_set_pristine(TcPlan* p, const SwitchParams& geom) {
  return LSW_TC_DISPATCH(v1::tc_plan_set_pristine(p->a, geom), tg::tc_plan_set_pristine(p->b, geom),
                         fc::tc_plan_set_pristine(p->c, geom));
}

// The fused switch + decode: the fc kernel's own fused build when the ctx
// switches with fc (W after a fused token is bitwise what its plain switch
// stores); else the v1 kernel's -- a ctx switching with tg builds a v1 plan
// (its own packed operands) on first use.
cudaError_t tc_plan_set_fused(TcPlan* p, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]) {
  if (p->which == 3) {
    const cudaError_t e = fc::tc_plan_set_fused(p->c, n_layers, x_off, y_off, x_per_layer, y_per_layer, kinds, nk);
    if (e != cudaErrorNotSupported) return e;
  }
  if (!p->a) {
    const char* why = "";
    cudaError_t e = v1::tc_plan_create(&p->a, p->geom, p->num_sms, &why, /*strict=*/true);
    if (e != cudaSuccess) { (void)cudaGetLastError(); p->a = nullptr; return cudaErrorNotSupported; }
  }
  return v1::tc_plan_set_fused(p->a, n_layers, x_off, y_off, x_per_layer, y_per_layer, kinds, nk);
}

cudaError_t launch_switch_tc_fused(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, const void* xs, float* ys) {
  if (p->which == 3) {
    const cudaError_t e = fc::launch_switch_tc_fused(p->c, sp, s, xs, ys);
    if (e != cudaErrorNotSupported) return e;
  }
  if (!p->a) return cudaErrorNotSupported;
  return v1::launch_switch_tc_fused(p->a, sp, s, xs, ys);
}

int64_t tc_plan_trace(const TcPlan* p, uint64_t* host, int64_t n) {
  return LSW_TC_DISPATCH(v1::tc_plan_trace(p->a, host, n), tg::tc_plan_trace(p->b, host, n), (int64_t)0);
}

}  // namespace lsw
