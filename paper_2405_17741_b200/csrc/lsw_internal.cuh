// lsw_internal.cuh -- internal declarations shared by the csrc/ translation units.
// Nothing here is part of the ABI (include/lsw.h is).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>

#include "../../include/lsw.h"

namespace lsw {

// Variant and tuning options (include/lsw_debug.h lsw_debug_set_option): set
// explicitly by the caller, read when a ctx is created; the library never
// reads the environment.  Options that produce wrong results on purpose
// (measurement probes) take effect only in a -DLSW_TUNING build.
const char* opt_str(const char* key);      // nullptr if unset
long opt_int(const char* key, long dflt);  // dflt if unset
long probe_int(const char* key);           // 0 unless built with LSW_TUNING

constexpr int kMaxTerms = 2 * LSW_MAX_TOPK;   // |S_t u S_{t-1}| <= 2k

// Switch modes (K1).  MERGE: Eq. 6; SWITCH: Eq. 10; UNMERGE: Eq. 7;
// RESTORE: W <- RNE(P + Delta(cur)) from a pristine copy P --
// the MERGE coefficient list, read from P instead of W.
enum SwitchMode : int32_t { MODE_MERGE = 0, MODE_SWITCH = 1, MODE_UNMERGE = 2, MODE_RESTORE = 3 };

// Ctx-owned device state.  slot[parity] holds the merged decision; a switch
// pass writes the new decision into slot[parity^1] and the LAST CTA to finish
// flips parity (every CTA has read slot[parity] before it counts itself done).
// `merged` is the device's own record of the state machine: set by
// a merge / switch / restore pass that ran, cleared by an unmerge; a pass whose
// decision was rejected (latched error) leaves it unchanged.  SWITCH and
// UNMERGE subtract the slot's decision only while it is set, so a rejected
// merge can never make a later pass subtract a decision W does not contain.
constexpr int kFusedMaxCtas = 256;

struct DevState {
  int32_t parity;
  uint32_t done;
  int32_t err;        // first latched LSW_DEV_* code
  int32_t merged;     // 1: slot[parity] is merged into W
  int32_t idx[2][LSW_MAX_TOPK];
  float g[2][LSW_MAX_TOPK];
  uint32_t lora_arrive;          // unmerged GEMV: LoRA-down products published in this launch
  uint32_t lora_depart;          // unmerged GEMV: CTAs done (the last one resets both)
  // fused decode's adaptive split (fc kernel): CTA b takes, in every segment
  // of T tiles, [T * fused_w[b], T * fused_w[b + 1]) >> 24; fused_perf[b] its
  // last pass's ns per tile (segment processing only, waits excluded); the
  // pass's last CTA turns them into the next pass's split
  uint32_t sweep_next;            // plain sweep, dynamic chunks: chunks claimed in this pass (the last CTA resets)
  int32_t fused_w_valid;          // 0: uniform split (b / G)
  uint32_t fused_done;            // CTAs done with the pass (the last one updates and resets)
  uint32_t fused_w[kFusedMaxCtas + 1];
  float fused_perf[kFusedMaxCtas];
};

// One kind's stacked tensors, as the kernels see them.
struct KindGeom {
  void* W;            // [L, d_out, d_in]
  const void* A;      // [L, N, r, d_in]
  const void* B;      // [L, N, d_out, r]
  const void* P;      // pristine copy of W (RESTORE source), or null
  int64_t d_out, d_in;
  int64_t tile_begin; // first tile index of this kind (prefix sum)
  int32_t row_tiles, col_tiles;
};

struct SwitchParams {
  KindGeom kind[LSW_NKIND];
  int64_t tiles_total;
  int32_t n_layers, n_experts, rank, top_k;
  float scale;        // alpha / r
  int32_t mode;
  const int32_t* cur_idx;
  const float* cur_g;
  DevState* state;
};

// The compacted coefficient list of one pass (SURVEY a-2), identical in every
// CTA: n terms (expert e[j], fp32 coefficient c[j]).
struct Coefs {
  int32_t n;
  int32_t bad;        // LSW_DEV_* if the inputs are invalid (pass becomes a no-op)
  int32_t e[kMaxTerms];
  float c[kMaxTerms];
};

// Build the coefficient list from (mode, cur, slot[parity]).  Run by ONE thread.
__device__ __forceinline__ void build_coefs(const SwitchParams& p, int32_t parity, Coefs& out) {
  out.n = 0;
  out.bad = 0;
  const int k = p.top_k, N = p.n_experts;
  int32_t ci[LSW_MAX_TOPK], pi[LSW_MAX_TOPK];
  float cg[LSW_MAX_TOPK], pg[LSW_MAX_TOPK];
  const bool has_cur = p.mode != MODE_UNMERGE;
  const bool has_prev = (p.mode == MODE_SWITCH || p.mode == MODE_UNMERGE) &&
                        *reinterpret_cast<volatile const int32_t*>(&p.state->merged) != 0;
  for (int j = 0; j < k; ++j) {
    if (has_cur) {
      ci[j] = p.cur_idx[j];
      cg[j] = p.cur_g[j];
      if (ci[j] < 0 || ci[j] >= N) out.bad = LSW_DEV_BAD_INDEX;
      if (!isfinite(cg[j])) out.bad = out.bad ? out.bad : LSW_DEV_BAD_GATE;
      for (int i = 0; i < j; ++i) if (ci[i] == ci[j]) out.bad = LSW_DEV_BAD_INDEX;
    }
    if (has_prev) {
      pi[j] = p.state->idx[parity][j];
      pg[j] = p.state->g[parity][j];
    }
  }
  if (out.bad) return;
  // current experts: c = scale * (g_cur - g_prev[e])  (g_prev = 0 if absent)
  if (has_cur) {
    for (int j = 0; j < k; ++j) {
      float gp = 0.f;
      if (has_prev)
        for (int i = 0; i < k; ++i) if (pi[i] == ci[j]) gp = pg[i];
      const float c = p.scale * (cg[j] - gp);
      if (c != 0.f) { out.e[out.n] = ci[j]; out.c[out.n] = c; ++out.n; }
    }
  }
  // previous-only experts: c = -scale * g_prev
  if (has_prev) {
    for (int i = 0; i < k; ++i) {
      bool in_cur = false;
      if (has_cur)
        for (int j = 0; j < k; ++j) in_cur |= (ci[j] == pi[i]);
      if (in_cur) continue;
      const float c = -p.scale * pg[i];
      if (c != 0.f) { out.e[out.n] = pi[i]; out.c[out.n] = c; ++out.n; }
    }
  }
}

// Epilogue of every switch kernel: record the decision and flip parity once
// all CTAs are done (thread 0 of each CTA, after the CTA's last tile).
__device__ __forceinline__ void finish_pass(const SwitchParams& p, int32_t parity, const Coefs& cf) {
  __threadfence();
  const uint32_t prev = atomicAdd(&p.state->done, 1u);
  if (prev == gridDim.x - 1) {
    volatile DevState* s = p.state;
    if (cf.bad) {
      atomicCAS(&p.state->err, 0, cf.bad);       // state unchanged
    } else if (p.mode != MODE_UNMERGE) {
      s->parity = parity ^ 1;
      s->merged = 1;
    } else {
      s->merged = 0;                             // state none: the slot is stale
    }
    p.state->done = 0;
    p.state->sweep_next = 0;                       // every CTA has run out of chunks
    __threadfence();
  }
}

// Write the current decision into the free slot (CTA 0, thread 0, at start).
__device__ __forceinline__ void stage_decision(const SwitchParams& p, int32_t parity) {
  if (p.mode == MODE_UNMERGE) return;
  for (int j = 0; j < p.top_k; ++j) {
    p.state->idx[parity ^ 1][j] = p.cur_idx[j];
    p.state->g[parity ^ 1][j] = p.cur_g[j];
  }
}

// Launchers (return cudaError_t of the launch).
cudaError_t launch_router(const void* Wg, const void* x1, int32_t n_experts, int64_t d_model,
                          int32_t top_k, int32_t dtype, int32_t* idx, float* gate,
                          DevState* state, cudaStream_t s);

cudaError_t launch_switch_simt(const SwitchParams& p, int32_t dtype, int grid, cudaStream_t s);

struct GemvSite {
  const void* W;      // [d_out, d_in] of this (layer, kind)
  int64_t d_out;
  int64_t row_begin;  // offset of this site's rows in the group output
};
struct GemvParams {
  GemvSite site[3];
  int32_t n_sites;
  int64_t rows_total;
  int64_t d_in;
  const void* x;
  float* y;
};
// Unmerged decode (Eq. 2 at P:228 without merging):
// y = W x + sum_j scale * g_j * B_{e_j} (A_{e_j} x) for every site of a group,
// W being the un-merged (pristine) weight.  ONE launch per group: the GEMV's
// CTAs compute the k*r LoRA-down products per site (dealt over the grid,
// published through a device counter) before streaming their W rows, and add
// the LoRA-up term to their rows at the end of the stream (gemv.cu).
struct GemvLora {
  const void* A[3];          // site q: A_kind of this layer [N, r, d_in]
  const void* B[3];          // site q: B_kind of this layer [N, d_out_q, r]
  const int32_t* idx;        // [k] device
  const float* gate;         // [k] device
  float scale;               // alpha / r
  int32_t k, r, n_experts;
  float* u;                  // scratch [n_sites * k * r] fp32
  int32_t* err;              // DevState::err: an invalid decision latches LSW_DEV_* and drops the LoRA terms
  uint32_t* arrive;          // DevState::lora_arrive / lora_depart (zero between launches)
  uint32_t* depart;
  int32_t flags;             // tuning builds only (probe unmerged_flags): 4 = no LoRA-up term (results wrong)
};
// Launch plan of the decode GEMV (gemv.cu), fixed per ctx at lsw_create.
struct GemvTune {
  int grid_cap = 148;               // CTAs at most (the SM count)
  uint32_t op_bytes = 32768;        // bytes per bulk copy at most (R rows per op, see launch_gemv)
  uint32_t op_min = 24576;          // ... and at least, unless one row is larger
  size_t budget = 176 * 1024;       // ring + x staging, merged-weight GEMV
  size_t budget_lora = 208 * 1024;  // same, unmerged form
  int probe = 0;                    // tuning builds only: 1 = stream W without the dot products
  bool ldg = false;                 // variant option gemv=ldg: the warp-per-row LDG kernel
  int split_rows = 1;               // option gemv_split: 1 rows over 24 KB reduced by two warps, 0 never, 2 always
};
// early_w: the previous launch on `s` was a GEMV (W may be prefetched before
// griddepcontrol.wait; see gemv.cu).  lora: null for the merged-weight GEMV,
// else the unmerged form (LoRA-down and LoRA-up inside the same launch).
cudaError_t launch_gemv(const GemvParams& p, int32_t dtype, const GemvTune& t, cudaStream_t s, bool early_w = false,
                        GemvLora* lora = nullptr);

// Unmerged prefill of one group for T tokens: prefill_tc.cu
// (bf16 with a tensor-core plan: tcgen05 LoRA-down GEMM, Z build, one tcgen05
// GEMM for the dense part + LoRA-up), prefill.cu (SIMT, fp32 storage or the
// SIMT switch).
struct PrefillParams {
  const void* W[3];          // site q: W [d_out_q, d_in] of this layer (pristine)
  const void* A[3];          // site q: A [N, r, d_in] of this layer
  const void* B[3];          // site q: B [N, d_out_q, r] of this layer
  int64_t d_out[3], row_begin[3];
  int32_t n_sites, k, r, n_experts;
  int64_t d_in, rows, T;
  float scale;               // alpha / r
  const void* X;             // [T, d_in]
  const int32_t* idx;        // [T, k]
  const float* gate;         // [T, k]
  float* U;                  // scratch: LoRA-down products (tc: per K split; fused: split-K bank partials)
  int64_t u_elems;           // its size (elements)
  void* Z;                   // scratch (tc): gate-scaled (hi, lo) bf16 operand of the LoRA-up step
  float* Y;                  // [T, rows]
};
cudaError_t launch_prefill_simt(const PrefillParams& P, int32_t dtype, cudaStream_t s);
struct PfPlan;               // prefill_tc.cu: TMA maps + launch geometry
struct TcPlan;
cudaError_t pf_plan_create(PfPlan** out, const SwitchParams& geom, const TcPlan* tc, int num_sms);
void pf_plan_destroy(PfPlan* plan);
void pf_scratch(const PfPlan* plan, int n_sites, int64_t T, int64_t* u_elems, int64_t* z_elems);
cudaError_t launch_prefill_tc(const PfPlan* plan, const PrefillParams& P, int layer, const int kinds[3],
                              cudaStream_t s);

// Tensor-core switch (switch_tc_dispatch.cu / switch_tc_fc.cu).
struct TcPlan;   // opaque: packed operands + TMA descriptors
cudaError_t tc_plan_create(TcPlan** out, const SwitchParams& geom, int num_sms, const char** why);
void tc_plan_destroy(TcPlan* plan);
int64_t tc_plan_bytes(const TcPlan* plan);
int tc_plan_grid(const TcPlan* plan);
int tc_plan_tile_n(const TcPlan* plan);
int64_t tc_plan_tiles(const TcPlan* plan);
// t_count > 0: only tiles [t0, t0 + t_count) (the launch-count ablation)
cudaError_t launch_switch_tc(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, int64_t t0 = 0,
                             int64_t t_count = 0);
int64_t tc_plan_matrix_tiles(const TcPlan* plan, int kind, int layer, int64_t* t0);   // tiles of one matrix
// Fused switch + decode (the fold mode only, else cudaErrorNotSupported)
cudaError_t tc_plan_set_fused(TcPlan* plan, int n_layers, const int64_t x_off[4], const int64_t y_off[4],
                              int64_t x_per_layer, int64_t y_per_layer, const int kinds[4][3], const int nk[4]);
cudaError_t launch_switch_tc_fused(const TcPlan* plan, const SwitchParams& p, cudaStream_t s, const void* xs,
                                   float* ys);
int tc_plan_kernel(const TcPlan* plan);   // 3: fc fold, 4: fc per-term, 5: fc per-term with B per unit
// packed, pre-swizzled B of one kind [L*N, dout_pad, rp] (also the prefill's LoRA-up operand)
const void* tc_plan_packed_B(const TcPlan* plan, int kind, int64_t* dout_pad, int* rp);
// RESTORE source: encode tensor maps over geom.kind[k].P (lsw_attach_pristine)
cudaError_t tc_plan_set_pristine(TcPlan* plan, const SwitchParams& geom);

}  // namespace lsw
