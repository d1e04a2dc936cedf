/*
 * lsw_debug.h -- variant selection, tuning and ablation hooks of liblsw.so.
 * Not part of the hot path and not needed by users.
 */
#ifndef LSW_DEBUG_H_
#define LSW_DEBUG_H_

#include "lsw.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Variant / tuning options, process-wide, read when a ctx is created
 * (lsw_create): the library never reads the environment.  key NULL clears
 * every option; value NULL unsets `key`.  Unknown keys are ignored.  Always
 * LSW_OK.  Keys (defaults in brackets; results are identical for every value
 * unless marked "probe"):
 *   tc_kernel      fold | pt | bu   force a mode of the tensor-core switch
 *                                   [chosen from r, k: DESIGN.md §5]
 *   tc_grid        N      switch grid (CTAs) below the SM count      [#SMs]
 *   tc_pair        0 | 1  the fold mode on CTA pairs (cta_group::2, M = 256;
 *                         each CTA stages half of the A^T columns)     [0]
 *   tc_chunk       N      tiles per CTA chunk of the sweep order     [48]
 *   fc_dyn         0|1    sweep chunks claimed at run time (1) or      [1]
 *                         dealt c -> CTA c mod G (0)
 *   fc_adapt       0|1    fused decode: segments split by measured CTA  [1]
 *                         speed (1) or evenly (0)
 *   fc_stages / fc_astages / fc_bbufs   explicit shared-memory plan (all three)
 *   fc_wrm         0 | 1  W tile moved by one 4-D TMA op             [1]
 *   gemv           ldg    the warp-per-row LDG GEMV instead of the bulk ring
 *   gemv_grid      N      GEMV grid cap                               [#SMs]
 *   gemv_op_kb     N      bytes per bulk copy, KB                     [32]
 *   gemv_smem_kb   N      ring budget, KB                             [176 / 208]
 *   gemv_split     0|1|2  rows over 24 KB reduced by two warps (1);    [1]
 *                         never (0); every row (2, tests)
 *   host_graph     0|1    lsw_decode_token_host replayed as a CUDA graph [1]
 *   Prefill (lsw_prefill_group, read at its first call; results may differ
 *   in fp32 summation order between values, each deterministic):
 *   pf_tt          128|256  token tile                       [per group]
 *   pf_cluster     1|2|4  dense launch on W-multicast clusters          [1]
 *   pf_pair        0|1|2  dense + LoRA-up on CTA pairs: never / groups  [1]
 *                         with a wave of 256-token tiles / always
 *   pf_fuse_u      0|1    single-CTA groups: LoRA-down and Z built in   [1]
 *                         the dense launch (1) or by two launches (0)
 *   pf_bank_split  0|1    fused: each A-bank tile's K in two halves on  [1]
 *                         two CTAs when the launch is one wave
 *   nccl_path      file   libnccl.so.2 to dlopen when none is loaded yet
 *                         (read at the first NCCL call, lsw_nccl_version)
 * Probes (deliberately WRONG results; only in a build with -DLSW_TUNING,
 * ignored otherwise): tc_probe (1: W stream only; 16: no fold math),
 * fc_fused_probe (4: no segment wait; 8: no GEMV), gemv_probe (stream only),
 * unmerged_flags (4: no LoRA-up term); timing traces into a caller's device
 * buffer (value = its address): gemv_trace_buf, pf_trace_buf. */
LSW_API lsw_status lsw_debug_set_option(const char* key, const char* value);

/* Launch-count ablation (the paper's "simple merge" row of
 * Tab. 6): the Eq. 6 merge of lsw_merge_all_layers, but ONE launch
 * of the same tensor-core kernel per adapted matrix (7 x L launches, each over
 * that matrix's tiles).  Same result (bitwise) as the single launch.  State
 * must be `none` (LSW_E_STATE otherwise) and becomes merged(idx, gate);
 * LSW_E_UNSUPPORTED for the SIMT switch.  Enqueue-only (graph-capturable). */
LSW_API lsw_status lsw_debug_merge_per_matrix(lsw_ctx* ctx, const int32_t* idx, const float* gate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LSW_DEBUG_H_ */
