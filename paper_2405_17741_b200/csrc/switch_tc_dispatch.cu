// switch_tc_dispatch.cu -- lsw::tc_plan_*: the tensor-core switch of a ctx is
// the fc kernel (switch_tc_fc.cu) in one of its three modes, chosen at
// lsw_create:
//   3 fold      coefficients folded into B as exact (hi, lo) bf16 pairs, ONE
//               accumulator per tile -- every BASELINE config; r <= 32, 2k*rp
//               small enough for a double-buffered strip
//   4 per-term  raw B strip, one fp32 TMEM accumulator per term (r = 64, and
//               r = 32 with k >= 3)
//   5 per-term, B per unit: the B slices staged with each unit's A^T slices
//               when a whole strip of 2k raw B slices does not fit (r = 64, k = 4)
//   6 the fold on CTA pairs (cta_group::2; option tc_pair = 1, off by
//               default: measured slower)
//   7 the fold with the (hi, lo) B strip in TMEM (the MMA's M-side operand
//               read from TMEM, folded there by the epilogue warps; shared
//               memory keeps only a raw strip; option tc_tb = 1 where
//               2k * rp <= 256; off by default: measured slower)
// The variant option "tc_kernel" (lsw_debug.h) = fold | pt | bu forces one.
#include <cstring>

#include "switch_tc_impl.cuh"

namespace lsw {

struct TcPlan {
  int which = 0;                 // 3 fold, 4 per-term, 5 per-term with B per unit
  fc::TcPlan* c = nullptr;
};

cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why) {
  *out = nullptr;
  const char* k = opt_str("tc_kernel");
  int order[3];
  int n = 0;
  if (k && strcmp(k, "fold") == 0) order[n++] = 0;
  else if (k && strcmp(k, "pt") == 0) order[n++] = 1;
  else if (k && strcmp(k, "bu") == 0) order[n++] = 2;
  else {
    // measured: the fold up to 2k * rp = 128 at r <= 32, the
    // per-term mode for r = 64 and for r = 32 with k >= 3; each falls back to
    // the other, then to B per unit, if its shared-memory plan does not fit
    const int rp = geom.rank <= 16 ? 16 : geom.rank <= 32 ? 32 : 64;
    // measured: the fold up to 2k * rp = 128 at r <= 32, the
    // per-term mode for r = 64 and for r = 32 with k >= 3; each falls back to
    // the other, then to B per unit, if its shared-memory plan does not fit
    const bool pt_first = rp == 64 || (rp == 32 && geom.top_k >= 3);
    order[n++] = pt_first ? 1 : 0;
    order[n++] = pt_first ? 0 : 1;
    order[n++] = 2;
  }
  TcPlan* p = new TcPlan();
  cudaError_t e = cudaErrorNotSupported;
  for (int m = 0; m < n && e != cudaSuccess; ++m) {
    *why = "";
    e = fc::tc_plan_create(&p->c, geom, num_sms, why, order[m]);
    if (e == cudaSuccess) p->which = 3 + order[m];
    else if (e != cudaErrorNotSupported) break;
    else { (void)cudaGetLastError(); p->c = nullptr; }
  }
  if (e != cudaSuccess) { delete p; return e; }
  *out = p;
  return cudaSuccess;
}

void tc_plan_destroy(TcPlan* plan) {
  if (!plan) return;
  if (plan->c) fc::tc_plan_destroy(plan->c);
  delete plan;
}

int64_t tc_plan_bytes(const TcPlan* p) { return fc::tc_plan_bytes(p->c); }
int tc_plan_grid(const TcPlan* p) { return fc::tc_plan_grid(p->c); }
int tc_plan_tile_n(const TcPlan* p) { return fc::tc_plan_tile_n(p->c); }
int64_t tc_plan_tiles(const TcPlan* p) { return fc::tc_plan_tiles(p->c); }
int tc_plan_kernel(const TcPlan* p) {
  if (p->which == 3 && fc::tc_plan_pair(p->c)) return 6;
  if (p->which == 3 && fc::tc_plan_tb(p->c)) return 7;
  return p->which;
}
const void* tc_plan_packed_B(const TcPlan* p, int kind, int64_t* dout_pad, int* rp) {
  return fc::tc_plan_packed_B(p->c, kind, dout_pad, rp);
}

cudaError_t launch_switch_tc(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, int64_t t0, int64_t t_count) {
  return fc::launch_switch_tc(p->c, sp, s, t0, t_count);
}

int64_t tc_plan_matrix_tiles(const TcPlan* p, int kind, int layer, int64_t* t0) {
  return fc::tc_plan_matrix_tiles(p->c, kind, layer, t0);
}

cudaError_t tc_plan_set_pristine(TcPlan* p, const SwitchParams& geom) { return fc::tc_plan_set_pristine(p->c, geom); }

// The fused switch + decode is the fold mode's own build (W after a fused
// token is bitwise what its plain switch stores); the per-term modes have none.
cudaError_t tc_plan_set_fused(TcPlan* p, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]) {
  return fc::tc_plan_set_fused(p->c, n_layers, x_off, y_off, x_per_layer, y_per_layer, kinds, nk);
}

cudaError_t launch_switch_tc_fused(const TcPlan* p, const SwitchParams& sp, cudaStream_t s, const void* xs, float* ys) {
  return fc::launch_switch_tc_fused(p->c, sp, s, xs, ys);
}

}  // namespace lsw
